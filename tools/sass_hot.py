"""Hot basic blocks of one kernel from `ncu --page source --csv --print-source sass` (diagnostic).

Consecutive SASS instructions with the same 'Instructions Executed' count form one block;
prints blocks by executed warp-instructions and by stall samples, with their opcodes."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, isamp, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
ins = []
for r in rows[2:]:
    if len(r) <= iex:
        continue
    try:
        ins.append((r[ia], r[isrc], int(r[isamp] or 0), int(r[iex] or 0)))
    except ValueError:
        pass
blocks, cur = [], []
for x in ins:
    if cur and x[3] != cur[-1][3]:
        blocks.append(cur)
        cur = []
    cur.append(x)
blocks.append(cur)
tot_ex = sum(x[3] for x in ins)
tot_s = sum(x[2] for x in ins)
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print("total warp-instr %.3e samples %d blocks %d" % (tot_ex, tot_s, len(blocks)))
for key, name in ((lambda b: sum(x[3] for x in b), "executed"), (lambda b: sum(x[2] for x in b), "samples")):
    print("== top blocks by", name)
    for b in sorted(blocks, key=key, reverse=True)[:top]:
        ex = sum(x[3] for x in b)
        s = sum(x[2] for x in b)
        ops = " ".join(x[1].split()[0] if not x[1].startswith("@") else x[1].split()[1] for x in b[:14])
        print("%s n=%3d count=%.2e ex=%5.1f%% samp=%5.1f%%  %s" % (b[0][0], len(b), b[0][3], 100 * ex / tot_ex, 100 * s / max(tot_s, 1), ops))
