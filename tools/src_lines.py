"""Per CUDA source line: warp instructions, stall samples and excessive shared / global
wavefronts (bank conflicts, uncoalesced sectors) from an ncu `--page source --csv
--print-source cuda,sass` export (lines of one kernel).
usage: python tools/src_lines.py src.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg, cur, text = {}, None, {}
fname = None
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] in ("Function Name",):
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not r:
        continue
    if r[0]:  # a CUDA source line
        cur = (fname, r[0])
        text[cur] = r[1]
        continue
    if len(r) > 7 and cur:
        a = agg.setdefault(cur, [0.0, 0.0, 0.0])
        try:
            a[0] += float(r[7] or 0)
            a[1] += float(r[4] or 0)
        except ValueError:
            pass
        if hdr:
            for i, h in enumerate(hdr):
                if "Excessive" in h and i < len(r):
                    try:
                        a[2] += float(r[i] or 0)
                    except ValueError:
                        pass
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
tx = sum(v[2] for v in agg.values()) or 1
print("instructions %.0f  samples %.0f  excessive wavefronts/sectors %.0f" % (ti, ts, tx))
if hdr:
    print("columns:", "; ".join(h for h in hdr if h))
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print("%-10s %5s %5.1f%% instr %5.1f%% stall %5.1f%% excess  %s" % (k[0][:10], k[1], 100 * v[0] / ti, 100 * v[1] / ts,
                                                                    100 * v[2] / tx, text[k].strip()[:80]))
print("-- by excessive wavefronts")
for k, v in sorted(agg.items(), key=lambda x: -x[1][2])[:12]:
    print("%-10s %5s %5.1f%% excess  %s" % (k[0][:10], k[1], 100 * v[2] / tx, text[k].strip()[:80]))
