"""Per-class stage-3 times of one config, symbolic and numeric (development aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
import paper_1504_05022_b200 as sg
for cfg in sys.argv[1:]:
    scale = None
    if ":" in cfg:
        cfg, scale = cfg.split(":"); scale = int(scale)
    for name, A, B in bench.make_workload(cfg, scale):
        if isinstance(B, str) or isinstance(A, str):
            continue
        dA = sg.DeviceCsr.from_host(A); dB = dA if B is None else sg.DeviceCsr.from_host(B)
        for rep in range(2):
            op = sg.SpGEMM(dA, dB, sg.FLAG_PRECISE); nnz = op.symbolic(); torch.cuda.synchronize()
            s1 = op.stats(); C = op.numeric(); torch.cuda.synchronize(); s2 = op.stats(); op.destroy()
        fmt = lambda st: {k: (v["rows"], v["products"], round(v["ms"], 2)) for k, v in st["classes"].items()}
        print(cfg, name, "stage_ms", [round(x, 2) for x in s2["stage_ms"]], "long", s2["long_rows"], flush=True)
        print("   symbolic:", fmt(s1), flush=True)
        print("   numeric :", fmt(s2), flush=True)
        del dA, dB, C
        torch.cuda.empty_cache()
