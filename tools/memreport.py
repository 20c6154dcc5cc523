"""the paper's memory pre-allocation comparison (Figure 9, [P:730-739]) on the
synthetic configs: device bytes each allocation strategy needs — precise ([P:165]), the hybrid
method (C~ rows of min(u_i, n) for the on-chip classes, progressive 2x growth for long rows,
[P:224], [P:297]) and the upper bound ([P:169]).  Like Figure 9 the totals include the two
input matrices and the resulting matrix ([S:455-462]); ratios are against precise, with the
harmonic mean over the products ("Hmean", Figure 9).  SPEC's overshoot invariant ([S:214]):
hybrid bytes <= upper-bound bytes + the doubling overshoot of the progressive long rows — here
the growth is capped at min(u_i, n) (R7), so the overshoot is 0 by construction and
the column "overshoot" reports the measured long-row arena against its cap.

    python tools/memreport.py c2 c3a c3b c4a c4b c5blk > profiles/r02/memory_report.md
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1504_05022_b200 as sg  # noqa: E402

STRATS = [("precise", sg.FLAG_PRECISE), ("hybrid", 0), ("upper bound", sg.FLAG_UPPER_BOUND)]


def workload(cfg):
    if cfg == "c5blk":  # config 5 as one rank's row block at P = 8 (C of the full product: 412 GB)
        from gen import torchgen as tg
        n = 1 << 23
        return [("AB rows [0, n/8)", tg.to_csr(*tg.band(n, rows=(0, n // 8))), tg.to_csr(*tg.uniform_rows(n, n, 64)))]
    return bench.make_workload(cfg)


def csr_bytes(rows, nnz):
    return 8 * (rows + 1) + 12 * nnz


print("| config | product | nnz(C) | A + B + C | " + " | ".join("%s: workspace / total (x precise)" % n for n, _ in STRATS)
      + " | long rows: arena vs cap (overshoot) |")
print("|---|---|---|---|" + "---|" * len(STRATS) + "---|")
ratios = {n: [] for n, _ in STRATS}
for cfg in sys.argv[1:] or ["c2"]:
    out = None
    for name, A, B in workload(cfg):
        dA = sg.DeviceCsr.from_host(A) if not isinstance(A, str) else out
        dB = dA if B is None else (out if isinstance(B, str) else sg.DeviceCsr.from_host(B))
        cells, totals, nnz, arena = [], {}, 0, ""
        base = csr_bytes(dA.rows, dA.nnz) + (0 if B is None else csr_bytes(dB.rows, dB.nnz))
        for sname, fl in STRATS:
            op = sg.SpGEMM(dA, dB, fl)
            nnz = op.symbolic()
            st = op.stats()
            C = op.numeric() if sname == "precise" else None
            torch.cuda.synchronize()
            tot = base + csr_bytes(dA.rows, nnz) + st["workspace_bytes"]
            totals[sname] = tot
            cells.append((st["workspace_bytes"], tot))
            if sname == "hybrid" and st["long_rows"] > 0:
                # the progressive arena against the long class's products (>= its upper bound
                # sum of min(u_i, n)): growth never passes min(u_i, n), so no overshoot
                cap = st["classes"]["long"]["products"]
                arena = "%d of <= %d entries (0)" % (st["long_entries"], cap)
            if C is not None:
                out = C
            op.destroy()
        for sname, _ in STRATS:
            ratios[sname].append(totals[sname] / totals["precise"])
        print("| %s | %s | %d | %.3f GB | %s | %s |" % (
            cfg, name, nnz, (base + csr_bytes(dA.rows, nnz)) / 1e9,
            " | ".join("%.3f / %.3f GB (%.2f)" % (w / 1e9, t / 1e9, t / totals["precise"]) for w, t in cells),
            arena or "—"), flush=True)
        torch.cuda.empty_cache()
        sg.trim_workspace_cache(0)
hm = {n: len(v) / sum(1.0 / x for x in v) for n, v in ratios.items() if v}
print("| Hmean | | | | " + " | ".join("(%.2f)" % hm[n] for n, _ in STRATS) + " | |")
