"""Run one config a few times (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen, bench
import paper_1504_05022_b200 as sg
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
flags = sg.FLAG_PRECISE if "precise" in sys.argv else 0
scale = [int(x.split("=")[1]) for x in sys.argv if x.startswith("scale=")]
reps = 3
work = bench.make_workload(cfg, scale[0] if scale else None)
name, A, B = work[0]
dA = sg.DeviceCsr.from_host(A); dB = dA if B is None else sg.DeviceCsr.from_host(B)
for _ in range(reps):
    op = sg.SpGEMM(dA, dB, flags); op.symbolic(); op.numeric(); torch.cuda.synchronize(); op.destroy()
print("done")
