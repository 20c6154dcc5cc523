"""Summarise an ncu capture's SASS by basic block: executions x length, stall share."""
import csv, subprocess, sys
rep = sys.argv[1]; kre = sys.argv[2] if len(sys.argv) > 2 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kre: cmd += ["-k", "regex:" + kre]
rows = list(csv.reader(subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()))
kern = []; cur = None
for r in rows:
    if r and r[0] == 'Kernel Name': cur = [r[1], None, []]; kern.append(cur); continue
    if r and r[0] == 'Address': cur[1] = r; continue
    if cur and cur[1]: cur[2].append(r)
seen = set()
for name, h, data in kern:
    if name in seen: continue
    seen.add(name)
    ie = h.index('Instructions Executed'); src = h.index('Source'); st = h.index('Warp Stall Sampling (All Samples)')
    tot = sum(int(r[ie] or 0) for r in data); stot = sum(int(r[st] or 0) for r in data) or 1
    print(name, "%.3fG warp-instr" % (tot / 1e9))
    blocks = []
    for r in data:
        n = int(r[ie] or 0); s = int(r[st] or 0)
        if blocks and blocks[-1][0] == n: blocks[-1][1] += 1; blocks[-1][2] += s; blocks[-1][3].append(r[src].strip())
        else: blocks.append([n, 1, s, [r[src].strip()]])
    for n, c, s, ins in sorted(blocks, key=lambda b: -b[0] * b[1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 12]:
        print(f"  {n/1e6:7.1f}M x {c:3d} = {n*c/1e9:5.2f}G  stall {100*s/stot:4.1f}%  | {' ; '.join(ins[:5])[:140]}")
