"""Per-kernel SASS hot spots and stall reasons from an `ncu --page source --csv` dump.
    ncu -i X.ncu-rep --page source --csv > src.csv; python scripts/ncu_hotspots.py src.csv [kernel_index] [n]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
kidx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
hdr = [r for r in rows if r and r[0] == "Address"][0]
ci = {h: i for i, h in enumerate(hdr)}
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], []]
        blocks.append(cur)
    elif r and r[0] != "Address" and cur is not None and len(r) > 3:
        cur[1].append(r)
name, body = blocks[kidx]
stall = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[2]) for r in body)
print(name, "samples", tot)
agg = {h: sum(int(r[ci[h]]) for r in body if r[ci[h]] not in ("", "-")) for h in stall}
print("stalls:", [(k, round(v / tot, 3)) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]])
ops = collections.Counter()
for r in body:
    t = r[1].split()
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    ops[op] += int(r[2])
print("by opcode:", [(k, round(v / tot, 3)) for k, v in ops.most_common(12)])
for r in sorted(body, key=lambda r: -int(r[2]))[:n]:
    rs = sorted([(h[6:], int(r[ci[h]])) for h in stall if r[ci[h]] not in ("", "-", "0")], key=lambda x: -x[1])[:3]
    print(r[2].rjust(7), r[0][-5:], r[1].strip()[:64].ljust(64), rs)
