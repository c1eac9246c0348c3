"""Dump a uniform sample of a config's records (t_eff, cost, quality as int64) for offline
filter experiments.  usage: python tools/dump_records.py C3 out.npy [blocks] [block_len]"""
import os
import random
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_05800_b200 as sw  # noqa: E402
from swgen import make_config  # noqa: E402

cfg, out = sys.argv[1], sys.argv[2]
blocks = int(sys.argv[3]) if len(sys.argv) > 3 else 256
blen = int(sys.argv[4]) if len(sys.argv) > 4 else 4096
pb = make_config(cfg)
rng = random.Random(7)
with sw.Plan(pb) as plan:
    plan.eval(0, plan.n)
    rows = []
    for _ in range(blocks):
        b = rng.randrange(plan.n - blen)
        buf = plan.copy_records(b, blen)
        a = np.frombuffer(buf, dtype=np.uint64).reshape(blen, -1)
        rows.append(a.copy())
    a = np.concatenate(rows)
    np.save(out, a)
    print(cfg, a.shape, sw.__name__)
