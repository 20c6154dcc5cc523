"""Host-side timeline of one step (create / symbolic / numeric / destroy).
usage: python tools/steptime.py [cfg] [hybrid|precise]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
import paper_1504_05022_b200 as sg
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
flags = 0 if (len(sys.argv) > 2 and sys.argv[2] == "hybrid") else sg.FLAG_PRECISE
name, A, B = bench.make_workload(cfg)[0]
dA = sg.DeviceCsr.from_host(A)
stream = torch.cuda.Stream()
for rep in range(4):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(stream)
    with torch.cuda.stream(stream):
        op = sg.SpGEMM(dA, dA, flags, stream); t.append(time.perf_counter())
        nnz = op.symbolic(); t.append(time.perf_counter())
        C = op.numeric(); t.append(time.perf_counter())
        op.destroy(); t.append(time.perf_counter())
    e.record(stream); torch.cuda.synchronize(); t.append(time.perf_counter())
    st = None
    print("rep", rep, "gpu ms %.3f" % s.elapsed_time(e), "host ms:", ["%.3f" % (1e3 * (b - a)) for a, b in zip(t, t[1:])], flush=True)
