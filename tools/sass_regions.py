"""Aggregate an ncu source-page SASS csv (first kernel section) by address blocks:
instruction share and stall share per block, plus the top stall reasons.
usage: python tools/sass_regions.py sass.csv [block_bytes]"""
import csv
import sys


def num(x):
    try:
        return int(float(x))
    except Exception:
        return 0


rows = list(csv.reader(open(sys.argv[1])))
blk = int(sys.argv[2], 0) if len(sys.argv) > 2 else 0x200
hdr = rows[1]
data = []
for r in rows[2:]:
    if len(r) != len(hdr) or r[0] == "Address":
        break
    data.append(r)
ia, isrc, ie = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
iss = hdr.index("Warp Stall Sampling (All Samples)")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(num(r[ie]) for r in data)
totS = sum(num(r[iss]) for r in data)
print("instructions", tot, "samples", totS)
agg = {}
for r in data:
    k = int(r[ia], 16) // blk
    a = agg.setdefault(k, [0, 0, r[isrc]])
    a[0] += num(r[ie])
    a[1] += num(r[iss])
for k in sorted(agg):
    e, s, src = agg[k]
    if e > tot * 0.01 or s > totS * 0.01:
        print("%6s %5.1f%% instr %5.1f%% stall  %s" % (hex(k * blk), 100 * e / tot, 100 * s / totS, src[:70]))
st = {h: sum(num(r[hdr.index(h)]) for r in data) for h in stalls}
print(" ".join("%s=%.1f%%" % (h[6:], 100 * v / totS) for h, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
