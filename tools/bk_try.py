"""c3b long rows: rank kernel (default) vs the bucket path (set_debug_long_bucket) — time and
bit-equality of the two results.  usage: python tools/bk_try.py [cfg] [min_window ...]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
import paper_1504_05022_b200 as sg
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3b"
mws = [int(x) for x in sys.argv[2:]] or [0, 4096]
name, A, B = bench.make_workload(cfg)[0]
dA = sg.DeviceCsr.from_host(A)
stream = torch.cuda.Stream()
ref = None
for mw in mws:
    sg.set_debug_long_bucket(mw)
    ts = []
    for rep in range(4):
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            s.record(stream)
            op = sg.SpGEMM(dA, dA, sg.FLAG_PRECISE, stream)
            op.symbolic()
            C = op.numeric()
            st = op.stats()
            op.destroy()
            e.record(stream)
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    same = None
    if ref is None:
        ref = C
    else:
        same = bool(torch.equal(ref.rp, C.rp) and torch.equal(ref.ci, C.ci) and
                    torch.equal(ref.val.view(torch.int64), C.val.view(torch.int64)))
    print("min_window", mw, "ms", ["%.2f" % t for t in ts], "long ms", st.get("tier_ms", {}).get("long"),
          "bit-equal to first", same, flush=True)
sg.set_debug_long_bucket(0)
