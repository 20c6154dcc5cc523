"""Quick timing of one config through the C ABI (development aid, not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
import paper_1504_05022_b200 as sg

def run(name, A, B=None, flags=0, reps=5):
    t0 = time.time()
    dA = sg.DeviceCsr.from_host(A); dB = dA if B is None else sg.DeviceCsr.from_host(B)
    torch.cuda.synchronize()
    times = []
    for r in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        op = sg.SpGEMM(dA, dB, flags); nnz = op.symbolic(); C = op.numeric()
        e.record(); torch.cuda.synchronize()
        times.append(s.elapsed_time(e)); st = op.stats(); op.destroy()
    t = min(times)
    flops = 2 * st["sum_u"]
    cb = 8*(A.shape[0]+1)*2 + 8*(dB.rows+1) + 12*(A.nnz + dB.nnz + nnz)
    print("%-12s flags=%d ms=%.3f (all %s) GFlop/s=%.1f CB GB/s=%.1f nnzC=%d sum_u=%d stage_ms=%s tiers=%s long=%d growth=%d" % (
        name, flags, t, ["%.2f" % x for x in times], flops / t / 1e6, cb / t / 1e6, nnz, st["sum_u"],
        ["%.3f" % x for x in st["stage_ms"]], st["tier_rows"], st["long_rows"], st["growth_rounds"]), flush=True)
    print("    classes:", {k: round(v["ms"], 3) for k, v in st["classes"].items()}, flush=True)

if __name__ == "__main__":
    which = sys.argv[1:] or ["c2"]
    if "c1" in which: run("c1", gen.stencil("2d5", 32))
    if "c2" in which:
        A = gen.stencil("3d27", 128); run("c2", A); run("c2", A, flags=sg.FLAG_PRECISE)
    if "c2s" in which:
        A = gen.stencil("3d27", 64); run("c2s", A); run("c2s", A, flags=sg.FLAG_PRECISE)
    if "r16" in which:
        A = gen.rmat(16, 16, (0.45, 0.15, 0.15, 0.25)); run("rmat16", A); run("rmat16", A, flags=sg.FLAG_PRECISE)
    if "g16" in which:
        A = gen.rmat(16, 16, (0.57, 0.19, 0.19, 0.05)); run("g500s16", A); run("g500s16", A, flags=sg.FLAG_PRECISE)
