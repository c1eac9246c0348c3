"""Write profiles/traffic.json from ncu --set full raw CSV exports (tools/gpu_round2.sh cap):
per config and kernel, DRAM bytes (read + write) of the captured launch, its algorithmic
bytes (32 B x records written / read by that launch, given here from the launch's record
count) and issue-active %.  usage: python tools/traffic_from_ncu.py TAG"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
# (config, kernel, capture, records of the captured launch, what they are)
CAPS = [
    ("C2", "eval_kernel", "eval_C2", 429981696, "all C2 candidates (one eval launch)"),
    ("C2", "scan_kernel", "scan_C2", 376233984, "the big strided fold pass (pass 3) of C2"),
    ("C3", "eval_kernel", "eval_C3", 191102976, "all C3 candidates (one eval launch)"),
    ("C3", "scan_kernel", "scan_C3", 167215104, "the big strided fold pass (pass 3) of C3"),
    ("C5", "eval_kernel", "eval_C5", 1 << 28, "one 2^28-candidate C5 chunk (tools/one_step_c5.py)"),
    ("C5", "scan_kernel", "scan_C5", 234823680, "the big fold pass of that chunk"),
]


def metric(path, name):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    i = hdr.index(name)
    units = rows[1]
    v = float(rows[2][i].replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "%": 1}.get(units[i], 1)


out = {"how": "ncu --set full --clock-control none: dram__bytes_read.sum + dram__bytes_write.sum of one "
              "captured launch; bench scales the ratio dram/algorithmic to its own per-launch algorithmic "
              "bytes; issue_active_pct = smsp__issue_active.avg.pct_of_peak_sustained_active of the same "
              "capture", "round": "r2 (%s session)" % tag, "configs": {}}
for cfg, kern, cap, recs, what in CAPS:
    p = os.path.join(ROOT, "gpurun_out", "%s_%s_raw.csv" % (tag, cap))
    if not os.path.exists(p):
        continue
    d = metric(p, "dram__bytes_read.sum") + metric(p, "dram__bytes_write.sum")
    ia = metric(p, "smsp__issue_active.avg.pct_of_peak_sustained_active")
    out["configs"].setdefault(cfg, {"kernels": {}})["kernels"][kern] = {
        "dram_bytes": int(d), "algorithmic_bytes": 32 * recs, "ratio": d / (32 * recs),
        "records": recs, "launch": what, "issue_active_pct": round(ia, 2),
        "report": "gpurun_out/%s_%s (profiles/round2/%s_ncu_%s.txt)" % (tag, cap, tag, cap)}
json.dump(out, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
for cfg, v in out["configs"].items():
    for k, x in v["kernels"].items():
        print(cfg, k, "%.4f" % x["ratio"], x["issue_active_pct"])
