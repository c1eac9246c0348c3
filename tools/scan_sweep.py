"""Scan-kernel timing vs the L2 prefetch distance (SW_PREFETCH), C2 (diagnostic)."""
import os, subprocess, sys
code = r'''
import os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_2603_05800_b200 as sw
from swgen import make_config
pb = make_config("C2")
plan = sw.Plan(pb)
for it in range(4):
    plan.reset(); plan.eval(0, plan.n); plan.select_batch(pb.queries); plan.pareto()
n0, ms0, b0 = plan.kernel_time(sw.SW_KERNEL_SCAN)
for it in range(6):
    plan.reset(); plan.eval(0, plan.n); plan.select_batch(pb.queries); plan.pareto()
n1, ms1, b1 = plan.kernel_time(sw.SW_KERNEL_SCAN)
print("prefetch %s: scan %.3f ms/step, %.0f GB/s" % (os.environ.get("SW_PREFETCH"), (ms1-ms0)/6, (b1-b0)/((ms1-ms0)/1e3)/1e9), flush=True)
'''
for pf in sys.argv[1:] or ["0", "1", "2", "3", "4", "6", "8"]:
    env = dict(os.environ, SW_PREFETCH=pf)
    subprocess.run([sys.executable, "-c", code], env=env)
