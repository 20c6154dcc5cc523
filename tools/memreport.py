"""device memory the library holds after symbolic, per allocation strategy
(hybrid progressive [P:224, P:297], hybrid upper bound [P:169], precise [P:165]), against the
bytes of C itself (12 B per entry + row pointers).  Prints a markdown table.

    python tools/memreport.py c2 c3b c4a c4b
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
import paper_1504_05022_b200 as sg

STRATS = [("hybrid (progressive)", 0), ("hybrid (upper bound)", sg.FLAG_UPPER_BOUND), ("precise", sg.FLAG_PRECISE)]
print("| config | product | nnz(C) | C bytes | " + " | ".join("%s: workspace (x C)" % n for n, _ in STRATS) + " |")
print("|---|---|---|---|" + "---|" * len(STRATS))
for cfg in sys.argv[1:] or ["c2"]:
    out = None
    for name, A, B in bench.make_workload(cfg):
        dA = sg.DeviceCsr.from_host(A)
        dB = dA if B is None else (out if isinstance(B, str) else sg.DeviceCsr.from_host(B))
        cells, nnz = [], 0
        for sname, fl in STRATS:
            op = sg.SpGEMM(dA, dB, fl)
            nnz = op.symbolic()
            st = op.stats()
            C = op.numeric() if sname == "precise" else None
            torch.cuda.synchronize()
            cells.append(st["workspace_bytes"])
            if C is not None:
                out = C
            op.destroy()
        cbytes = 12 * nnz + 8 * (dA.rows + 1)
        print("| %s | %s | %d | %.3f GB | %s |" % (cfg, name, nnz, cbytes / 1e9,
              " | ".join("%.3f GB (%.2f)" % (w / 1e9, w / cbytes) for w in cells)), flush=True)
        torch.cuda.empty_cache()
