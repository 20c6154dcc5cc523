#!/usr/bin/env python
"""bench.py — SpGEMM GFlop/s (2×products/s) and HBM roofline fraction on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--strategy hybrid|precise]
    python bench.py --impl reference ...      # the CPU oracle on a bounded sample (baseline arm)

One step = one pass of the whole hot path (stages 1-4: spgemm_symbolic + spgemm_numeric)
over the workload's A and B, which are resident in HBM before timing starts.  L2 is
flushed (a 512 MiB memset) before every timed step, outside the timed window.  Each step
is bracketed by CUDA events on the library's stream; the K step times are summed.  For
N > 1 (torchrun) every rank runs its row block through the dist_* ABI and the step time
is the max over ranks.  Rank 0 prints one JSON line.

metric = 2·Σu / t  (flops = 2·nnz(Ĉ) [P:433]); the compulsory-byte HBM fraction of the
step and the roofline of the dominant kernel are reported next to it.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "SpGEMM GFlop/s (2x products/s) and HBM GB/s vs roofline at 1/2/4/8 B200"
CONFIGS = {
    "c1": "C = A·A, A = 2D 5-point Laplacian on a 32×32 grid (1024 rows, fp64 CSR)",
    "c2": "C = A·A, A = 3D 27-point stencil on a 128³ grid (2.1M rows, FEM-like)",
    "c3a": "C = A·A, A = R-MAT scale 22, edge factor 16, (0.45,0.15,0.15,0.25), permuted",
    "c3b": "C = A·A, A = R-MAT Graph500 skew (0.57,0.19,0.19,0.05), scale 18, edge factor 16",
    "c4a": "Galerkin R·(A·P), A = 3D 7-point 256³, tentative 2×2×2 aggregation P",
    "c4b": "Galerkin R·(A·P), A = 3D 7-point 256³, Jacobi-smoothed aggregation P (ω=3/4)",
    "c5": "C = A·B, A = band(64) n=2^23, B = 64 uniform columns per row",
    # the paper's Galerkin set ([P:393-397]): AMG hierarchies (3 levels) of
    # smoothed aggregation with a Jacobi smoother; every level's P^T(AP) (suffix _ptap: (P^T A)P)
    "g2d5": "Galerkin P^T(AP), 3-level AMG, 2D 5-point Poisson 1024x1024",
    "g2d9": "Galerkin P^T(AP), 3-level AMG, 2D 9-point Poisson 1024x1024",
    "g3d7": "Galerkin P^T(AP), 3-level AMG, 3D 7-point Poisson 101^3",
    "g3d27": "Galerkin P^T(AP), 3-level AMG, 3D 27-point Poisson 101^3",
    "g2d5_ptap": "Galerkin (P^T A)P, 3-level AMG, 2D 5-point Poisson 1024x1024",
    "g2d9_ptap": "Galerkin (P^T A)P, 3-level AMG, 2D 9-point Poisson 1024x1024",
    "g3d7_ptap": "Galerkin (P^T A)P, 3-level AMG, 3D 7-point Poisson 101^3",
    "g3d27_ptap": "Galerkin (P^T A)P, 3-level AMG, 3D 27-point Poisson 101^3",
}
SMI_REASONS = ["gpu_idle", "applications_clocks_setting", "sw_power_cap", "hw_slowdown", "sync_boost",
               "sw_thermal_slowdown", "hw_thermal_slowdown", "hw_power_brake_slowdown", "display_clock_setting"]
BAD_REASONS = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}


# ----------------------------------------------------------------------------- inputs
def _device_gen():
    """Torch generators on the GPU when one is present (bit-identical to gen/'s numpy)."""
    try:
        import torch
        if torch.cuda.is_available():
            from gen import torchgen
            return torchgen
    except Exception:
        pass
    return None


def make_workload(cfg: str, scale: int | None = None):
    """Returns a list of (name, A, B) products; B None means B = A, "prev" = previous output."""
    import gen
    tg = _device_gen()
    if cfg == "c1":
        return [("A2", gen.stencil("2d5", 32), None)]
    if cfg == "c2":
        return [("A2", gen.stencil("3d27", scale or 128), None)]
    if cfg in ("c3a", "c3b"):
        sc = scale or (22 if cfg == "c3a" else 18)
        abcd = (0.45, 0.15, 0.15, 0.25) if cfg == "c3a" else (0.57, 0.19, 0.19, 0.05)
        if tg is not None:
            return [("A2", tg.to_csr(*tg.rmat(sc, 16, abcd, seed=gen.SEED, mode="real")), None)]
        return [("A2", gen.rmat(sc, 16, abcd, seed=gen.SEED, mode="real"), None)]
    if cfg in ("c4a", "c4b"):
        n = scale or 256
        A = gen.stencil("3d7", n)
        P = gen.aggregation_P(n, smoothed=(cfg == "c4b"))
        R = gen.transpose(P)
        return [("AP", A, P), ("R(AP)", R, "prev")]
    if cfg.startswith("g"):
        kind = cfg[1:].split("_")[0]
        n = scale or (1024 if kind.startswith("2d") else 101)
        prods = []
        for lvl, (A, P, R) in enumerate(gen.amg_levels(kind, n, 3)):
            if cfg.endswith("_ptap"):   # (P^T A) P
                prods += [("RA%d" % lvl, R, A), ("(RA)P%d" % lvl, "prev", P)]
            else:                       # P^T (A P)
                prods += [("AP%d" % lvl, A, P), ("R(AP)%d" % lvl, R, "prev")]
        return prods
    if cfg == "c5":
        n = 1 << (scale or 23)
        if tg is not None:
            return [("AB", tg.to_csr(*tg.band(n)), tg.to_csr(*tg.uniform_rows(n, n, 64)))]
        return [("AB", gen.band(n), gen.uniform_rows(n, n, 64))]
    raise SystemExit("unknown config %s" % cfg)


def csr_bytes(rows, nnz):
    return 8 * (rows + 1) + 12 * nnz


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int = 0):
        self.samples = []
        self.proc = None
        self.index = index

    def __enter__(self):
        q = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,power.draw,utilization.gpu"
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 5:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16),
                                         float(parts[3]), float(parts[4])))
                except ValueError:
                    pass

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        load = [s for s in self.samples if s[4] > 0] or self.samples
        sm = sorted(s[0] for s in load)
        mask = 0
        for s in load:
            mask |= s[2]
        reasons = [n for b, n in enumerate(SMI_REASONS) if mask & (1 << b) and n != "gpu_idle"]
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(s[1] for s in load), "reasons": reasons,
                "samples": len(load)}


# ----------------------------------------------------------------------------- GPU arm
def gpu_context(args):
    import torch
    import torch.distributed as dist

    import paper_1504_05022_b200 as sg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit("--gpus %d but WORLD_SIZE=%d" % (args.gpus, world))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = dict(torch=torch, dist=dist, sg=sg, world=world, rank=rank, local=local,
               stream=torch.cuda.Stream(), flush=torch.empty(512 << 20, dtype=torch.uint8, device="cuda"))
    sg.load()
    uid = None
    if world > 1:
        obj = [sg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    ctx["uid"] = uid
    return ctx


def c5_rank_inputs(ctx, scale):
    """Config 5 at N > 1, generated where it is used (SURVEY §8(e) variant (ii)): this rank's
    row block of the band A (a balanced split: every interior row has u = 4096) and its row
    slice of B; the library all-gathers B (spgemm_dist_create_sharded)."""
    from gen import torchgen as tg
    world, rank = ctx["world"], ctx["rank"]
    n = 1 << (scale or 23)
    r0, r1 = (rank * n) // world, ((rank + 1) * n) // world
    (arp, aci, aval), _ = tg.band(n, rows=(r0, r1))
    (brp, bci, bval), _ = tg.uniform_rows(r1 - r0, n, 64, first_row=r0)
    sg = ctx["sg"]
    return n, (r0, r1), sg.DeviceCsr(r1 - r0, n, arp, aci, aval), sg.DeviceCsr(r1 - r0, n, brp, bci, bval)


def measure(args, ctx, cfg, strategy, steps, warmup, clocks_on=True, variant="i"):
    """Time `steps` whole-hot-path steps of workload `cfg` (after `warmup`); returns the
    bench-line fields (value, ms, hbm, roofline, clocks, ...) plus the inputs for e2e.
    N > 1: variant "i" = inputs replicated on every rank (only the nnz allgather crosses
    NVLink), "ii" = inputs on rank 0 (partition, A scatter and B broadcast timed inside the
    step); config 5 at N > 1 always runs as sharded inputs generated per rank."""
    torch, dist, sg = ctx["torch"], ctx["dist"], ctx["sg"]
    world, rank, local = ctx["world"], ctx["rank"], ctx["local"]
    stream, flush, uid = ctx["stream"], ctx["flush"], ctx["uid"]
    flags = sg.FLAG_PRECISE if strategy == "precise" else 0
    c5_dist = cfg == "c5" and world > 1
    if c5_dist:
        n5, rows5, dAb5, dBs5 = c5_rank_inputs(ctx, args.scale if cfg == args.config else None)
        work = [("AB", None, None)]
        dev_inputs = [("AB", None, None, dAb5, dBs5)]
    else:
        work = make_workload(cfg, args.scale if cfg == args.config else None)
        # inputs resident in HBM
        dev_inputs = []
        for name, A, B in work:
            dA = "prev" if isinstance(A, str) else sg.DeviceCsr.from_host(A)
            dB = None if B is None else ("prev" if isinstance(B, str) else sg.DeviceCsr.from_host(B))
            dev_inputs.append((name, A, B, dA, dB))
    torch.cuda.synchronize()

    dist_ops = {}

    # Row blocks per product.  c5's C (412 GB at n = 2^23) cannot be resident: rows run in
    # waves (C of a wave is freed before the next) under --wave-gb.  Other configs: one block.
    def plan_blocks(A, Bm):
        if cfg != "c5" or isinstance(A, str) or Bm is None or isinstance(Bm, str):
            return [(0, None)]  # one block: the whole product
        m = A.shape[0]
        est = 16 * 4096 * m  # C (12 B) + workspace (~4 B) per product, u = 4096 per row
        waves = max(1, -(-est // int(args.wave_gb * (1 << 30))))
        cuts = [(m * w) // waves for w in range(waves + 1)]
        return list(zip(cuts[:-1], cuts[1:]))

    blocks_of = {}
    if c5_dist:
        m_loc = rows5[1] - rows5[0]
        est = 16 * 4096 * m_loc
        waves = torch.tensor([max(1, -(-est // int(args.wave_gb * (1 << 30))))], dtype=torch.int64, device="cuda")
        dist.all_reduce(waves, op=dist.ReduceOp.MAX)  # every rank runs the same number of collectives
        W = int(waves.item())
        cuts = [(m_loc * w) // W for w in range(W + 1)]
        blocks_of["AB"] = list(zip(cuts[:-1], cuts[1:]))
    else:
        for (name, A, B, dA, dB) in dev_inputs:
            blocks_of[name] = plan_blocks(A, A if B is None else B)

    def one_step(collect=False):
        """Whole hot path once: every product of the workload, symbolic + numeric."""
        out = None
        info = []
        for (name, A, B, dA, dB) in dev_inputs:
            if c5_dist:
                # sharded inputs: per wave, this rank's A rows and its B slice; the library
                # all-gathers B, multiplies and stitches the global row offsets
                for wi, (w0, w1) in enumerate(blocks_of[name]):
                    blk = sg.DeviceCsr(w1 - w0, dA.cols, dA.rp[w0:w1 + 1], dA.ci, dA.val)
                    key = ("c5", wi)
                    op = dist_ops.get(key)
                    if op is None:
                        op = sg.DistSpGEMM(rank, world, uid, n5, n5, n5, blk, dB, flags, stream,
                                           a_rows=(rows5[0] + w0, rows5[0] + w1), b_rows=rows5)
                        dist_ops[key] = op
                    rb, re_, ln, gn = op.symbolic()
                    out = op.numeric()
                    if collect:
                        info.append((name, op.stats(), ln, blk, dB))
                    if len(blocks_of[name]) > 1:
                        out = None
                continue
            if isinstance(dA, str):
                dA = out  # chained product: the previous C is this A
            Bm = dA if dB is None else (out if isinstance(dB, str) else dB)
            if world == 1:
                blocks = blocks_of[name]
                for (r0, r1) in blocks:
                    dAb = dA if r1 is None or (r0, r1) == (0, dA.rows) else \
                        sg.DeviceCsr(r1 - r0, dA.cols, dA.rp[r0:r1 + 1], dA.ci, dA.val)
                    op = sg.SpGEMM(dAb, Bm, flags, stream)
                    nnz = op.symbolic()
                    out = op.numeric()
                    if collect:
                        info.append((name, op.stats(), nnz, dAb, Bm))
                    op.destroy()
                    if len(blocks) > 1:
                        out = None  # capacity-forced waves: the wave's C is released
            else:
                # the NCCL communicator is created once (outside the timed steps); each step
                # re-runs the partition, (variant ii: the input movement,) the local four stages
                # and the nnz allgather
                key = (name, id(Bm), variant)
                op = dist_ops.get(key)
                if op is None:
                    if variant == "i":
                        op = sg.DistSpGEMM(rank, world, uid, dA.rows, dA.cols, Bm.cols, dA, Bm,
                                           flags | sg.FLAG_INPUTS_REPLICATED, stream)
                    else:
                        op = sg.DistSpGEMM(rank, world, uid, dA.rows, dA.cols, Bm.cols, dA if rank == 0 else None,
                                           Bm if rank == 0 else None, flags, stream)
                    dist_ops[key] = op
                rb, re_, ln, gn = op.symbolic()
                blk = op.numeric()
                if collect:
                    info.append((name, op.stats(), ln, sg.DeviceCsr(re_ - rb, dA.cols, dA.rp[rb:re_ + 1], dA.ci,
                                                                    dA.val), Bm))
                out = blk  # multi-stage chains on N>1 are not supported (c4 runs at N=1)
        return out, info

    if world > 1 and len(dev_inputs) > 1:
        raise SystemExit("chained workloads (c4) run at --gpus 1 only")

    # warm-up (also warms the stream-ordered pool)
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            one_step()
    torch.cuda.synchronize()
    _, info = one_step(collect=True)
    torch.cuda.synchronize()

    def timed_pass():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev = []
        with ClockSampler(local) as cs:
            for _ in range(steps):
                flush.zero_()  # L2 flush outside the timed window (512 MiB > 126 MB L2)
                s = torch.cuda.Event(enable_timing=True)
                e = torch.cuda.Event(enable_timing=True)
                torch.cuda.current_stream().wait_stream(stream)
                stream.wait_stream(torch.cuda.current_stream())
                s.record(stream)
                with torch.cuda.stream(stream):
                    one_step()
                e.record(stream)
                ev.append((s, e))
            torch.cuda.synchronize()
        ms = sum(s.elapsed_time(e) for s, e in ev)
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms, cs.summary()

    ms_total, clocks = timed_pass()
    if any(r in BAD_REASONS for r in clocks["reasons"]) or (
            clocks["sm_mhz"] and clocks["sm_max_mhz"] and clocks["sm_mhz"] < 0.5 * clocks["sm_max_mhz"]
            and not clocks["reasons"]):
        ms_total, clocks2 = timed_pass()  # re-measure once
        clocks = dict(clocks2, remeasured=True, first_reasons=clocks["reasons"])
    ms_step = ms_total / steps

    # ---------------- per-step accounting (from the collected pass) ----------------
    # every rank accounts for its own rows (A rows, C rows); B once per product; N > 1: summed
    sum_u = sum(st["sum_u"] for _, st, _, _, _ in info)
    cb = 0
    nnz_c_tot = 0
    launches = 0
    seen_b = set()
    for name, st, nnz_c, dA, Bm in info:
        m = dA.rows
        a_nnz = int(dA.rp[-1].item() - dA.rp[0].item()) if m > 0 else 0  # a row block's own entries
        cb += csr_bytes(m, a_nnz) + csr_bytes(m, nnz_c)
        if (name, id(Bm)) not in seen_b and rank == 0:  # B is read once per product even across waves
            cb += csr_bytes(n5 if c5_dist else Bm.rows, (int(st["nnz_b"]) if c5_dist else Bm.nnz))
            seen_b.add((name, id(Bm)))
        nnz_c_tot += nnz_c
        launches += st["launches_symbolic"] + st["launches_numeric"]
    if world > 1:
        t = torch.tensor([sum_u, nnz_c_tot, cb], dtype=torch.int64, device="cuda")
        dist.all_reduce(t)
        sum_u, nnz_c_tot, cb = (int(x) for x in t.tolist())
    gflops = 2.0 * sum_u / (ms_step * 1e-3) / 1e9
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    step_gbs = cb / (ms_step * 1e-3) / 1e9

    # dominant kernel: the largest of (a) the symbolic stage-3 pass of the
    # precise strategy (structure kernels) and (b) each stage-3 class launch that writes values
    # (numeric classes in precise, the single pass in hybrid).  Algorithmic bytes per launch
    # are SURVEY §8(d)'s per-unit figures (stage 3): 16 B per row, 12 B per A entry, 12 B per
    # B entry read once (at most one per product), 12 B per output entry; the structure-only
    # symbolic pass reads 4 B column indices of A and B.  Bytes the implementation adds on top
    # (its own structure set, perm, C~ offsets) are not counted.
    hybrid = strategy == "hybrid"
    cands = []
    for name0, st0, nnz0, dA0, Bm0 in info:
        m0 = dA0.rows
        if not hybrid:
            sym_ms = st0["stage_ms"][1]
            alg = 16 * m0 + 4 * dA0.nnz + 4 * min(Bm0.nnz, st0["sum_u"])
            cands.append((sym_ms, alg, "%s: symbolic stage-3 pass (k_bw_sym / k_wrow / k_cta_hash / "
                          "k_long_bm_count)" % name0, "symbolic"))
        for cls_name, c in st0["classes"].items():
            if c["ms"] <= 0:
                continue
            alg = 16 * c["rows"] + 12 * c["a_entries"] + 12 * min(Bm0.nnz, c["products"]) + 12 * c["c_entries"]
            kname = ("k_bwrow DENSE" if not hybrid else "k_bw_one") if cls_name == "bw" else \
                "k_esc_bk" if cls_name.startswith(("w", "e")) else \
                "k_group" if cls_name.startswith("g") else \
                "k_long_rank" if cls_name.startswith("c") else "k_bk_part/sort/copy + k_long_rank"
            cands.append((c["ms"], alg, "%s: stage-3 class %s (%s)" % (name0, cls_name, kname), cls_name))
    best = max(cands, key=lambda x: x[0])
    launch_ms, alg, kern, cls_name = best
    achieved = alg / (launch_ms * 1e-3) / 1e9 if launch_ms > 0 else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            traffic = tj.get("%s/%s/%s" % (cfg, strategy, cls_name))
        except Exception:
            traffic = None

    result = {
        "metric": METRIC,
        "value": round(gflops, 3),
        "unit": "GFlop/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded generators, gen/; %s)" % ("coef values" if cfg in ("c1", "c2", "c4a", "c4b")
                                                            else "real values"),
        "config": {"workload": "%s: %s" % (cfg, CONFIGS[cfg]),
                   "strategy": strategy, "sum_u": sum_u, "nnz_c": nnz_c_tot,
                   "nnz_a": int(sum(d[3].nnz for d in dev_inputs if not isinstance(d[3], str))),
                   "parallelism": ("row blocks x%d (dist_* ABI, NCCL), variant %s" % (
                       world, "ii: sharded inputs generated per rank, B all-gathered" if c5_dist else
                       ("i: inputs replicated" if variant == "i" else "ii: inputs on rank 0"))) if world > 1
                   else "1 GPU",
                   "l2": "flushed before every timed step (512 MiB memset, outside the timed window)",
                   "waves": {n: len(b) for n, b in blocks_of.items() if len(b) > 1} or None,
                   "scale": args.scale if cfg == args.config else None},
        "hbm": {"compulsory_bytes": cb, "achieved_gbs": round(step_gbs, 1),
                "frac_of_peak": round(step_gbs / hbm_peak, 4), "peak_gbs": hbm_peak,
                "peak_source": peak_src},
        "roofline": {"bound": "hbm", "kernel": kern,
                     "achieved": round(achieved, 1) if achieved else None, "peak": hbm_peak,
                     "unit": "GB/s", "frac": round(achieved / hbm_peak, 4) if achieved else None,
                     "traffic": traffic, "alg_bytes_per_launch": int(alg),
                     "launch_ms": round(launch_ms, 4), "share_of_step": round(launch_ms / ms_step, 4),
                     "peak_source": peak_src,
                     "timing": "CUDA events recorded by libspgemm on its stream around the launch"},
        "stage_ms": {n: [round(x, 4) for x in st["stage_ms"]] for n, st, _, _, _ in info},
        "class_ms": {n: {c: round(v["ms"], 3) for c, v in st["classes"].items() if v["ms"] > 0}
                     for n, st, _, _, _ in info},
        "class_ms_symbolic": {n: {c: round(v["ms_symbolic"], 3) for c, v in st["classes"].items()
                                  if v["ms_symbolic"] > 0} for n, st, _, _, _ in info},
        "gpu_launches": launches * steps,
        "clocks": clocks,
    }
    for op in dist_ops.values():
        op.destroy()
    can_e2e = world == 1 and all(len(b) == 1 for b in blocks_of.values())
    return result, dict(work=work, flags=flags, sum_u=sum_u, can_e2e=can_e2e)


PER_CONFIG = ["c2", "c3a", "c3b", "c4a", "c4b", "g2d5", "g2d9", "g3d7", "g3d27", "g3d27_ptap"]


def run_gpu(args):
    ctx = gpu_context(args)
    torch, dist, sg = ctx["torch"], ctx["dist"], ctx["sg"]
    world, rank = ctx["world"], ctx["rank"]
    result, aux = measure(args, ctx, args.config, args.strategy, args.steps, args.warmup)
    if world > 1 and args.config != "c5" and not args.no_variant_ii:
        # SURVEY §8(e) variant (ii): the same step with the inputs on rank 0 only
        r2, _ = measure(args, ctx, args.config, args.strategy, args.steps, args.warmup, variant="ii")
        result["variant_ii"] = {"value": r2["value"], "unit": "GFlop/s", "ms_per_step": r2["ms_per_step"],
                                "parallelism": r2["config"]["parallelism"]}
    # ---------------- end-to-end through the public API with host buffers ----------------
    if aux["can_e2e"] and not args.no_e2e:
        result["e2e"] = e2e_measure(args, aux["work"], aux["flags"], ctx["stream"], aux["sum_u"])
    if world == 1 and not args.no_cpu:
        result["cpu_baseline"] = cpu_baseline(args, aux["work"], budget_s=args.cpu_budget)
        result["cpu_single_thread"] = cpu_single_thread(args)
    del aux
    # ---------------- the other single-GPU configs of BASELINE.json (same protocol) ----------
    if world == 1 and not args.no_per_config:
        per = {}
        for cfg in PER_CONFIG:
            # both strategies: they trade places — c2 (precise ahead: r_c = 5.8, C~ 6x C), c3a
            # (power law: hybrid saves the counting pass where r_c is near 1), c4a / c4b and the
            # Galerkin hierarchies (A·P rows of at most 32 products: hybrid saves the count)
            for strat in ["precise", "hybrid"]:
                if cfg == args.config and strat == args.strategy:
                    continue
                torch.cuda.empty_cache()
                sg.trim_workspace_cache(0)
                r, _ = measure(args, ctx, cfg, strat, args.per_config_steps, 3)
                per["%s/%s" % (cfg, strat)] = {
                    "value": r["value"], "unit": "GFlop/s", "ms_per_step": r["ms_per_step"],
                    "steps": r["steps"], "sum_u": r["config"]["sum_u"], "nnz_c": r["config"]["nnz_c"],
                    "hbm_frac_of_peak": r["hbm"]["frac_of_peak"],
                    "roofline": {k: r["roofline"][k] for k in ("kernel", "achieved", "frac", "traffic",
                                                                "launch_ms", "share_of_step")},
                    "stage_ms": r["stage_ms"], "clocks_sm_mhz": r["clocks"]["sm_mhz"],
                    "clock_reasons": r["clocks"]["reasons"]}
        result["per_config"] = per
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def e2e_measure(args, work, flags, stream, sum_u):
    """Same metric through the public API with pinned HOST buffers: H2D of the step's
    inputs, the four stages, D2H of C — all inside the timed window."""
    import torch

    import paper_1504_05022_b200 as sg

    def pin(a, dt):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dt).pin_memory()

    host = []
    h2d = 0
    for name, A, B in work:
        hA = None
        if not isinstance(A, str):
            hA = (pin(A.rp, torch.int64), pin(A.ci, torch.int32), pin(A.val, torch.float64), A.shape)
            h2d += csr_bytes(A.shape[0], A.nnz)
        hB = None
        if B is not None and not isinstance(B, str):
            hB = (pin(B.rp, torch.int64), pin(B.ci, torch.int32), pin(B.val, torch.float64), B.shape)
            h2d += csr_bytes(B.shape[0], B.nnz)
        host.append((hA, hB, B))

    def todev(h):
        rp, ci, val, shape = h
        return sg.DeviceCsr(shape[0], shape[1], rp.to("cuda", non_blocking=True), ci.to("cuda", non_blocking=True),
                            val.to("cuda", non_blocking=True))

    d2h_holder = {}
    copy_stream = torch.cuda.Stream()

    def step():
        """One step: H2D of the inputs and the four stages on `stream`; the D2H of C on
        copy_stream once C is complete — it overlaps the next step's H2D and stages (PCIe is
        full duplex; C's memory is held for the copy by record_stream)."""
        out = None
        d2h = 0
        with torch.cuda.stream(stream):
            for hA, hB, B in host:
                dA = out if hA is None else todev(hA)
                dB = dA if B is None else (out if isinstance(B, str) else todev(hB))
                op = sg.SpGEMM(dA, dB, flags, stream)
                op.symbolic()
                out = op.numeric()
                op.destroy()
        done = torch.cuda.Event()
        done.record(stream)
        key = out.ci.numel()
        if key not in d2h_holder:
            copy_stream.synchronize()
            d2h_holder.clear()
            d2h_holder[key] = (torch.empty(out.rp.numel(), dtype=torch.int64).pin_memory(),
                               torch.empty(out.ci.numel(), dtype=torch.int32).pin_memory(),
                               torch.empty(out.val.numel(), dtype=torch.float64).pin_memory())
        hr, hc, hv = d2h_holder[key]
        copy_stream.wait_event(done)
        with torch.cuda.stream(copy_stream):
            hr.copy_(out.rp, non_blocking=True)
            hc.copy_(out.ci, non_blocking=True)
            hv.copy_(out.val, non_blocking=True)
        for t in (out.rp, out.ci, out.val):
            t.record_stream(copy_stream)
        d2h += csr_bytes(out.rows, out.ci.numel())
        return d2h

    for _ in range(max(1, min(args.warmup, 2))):
        step()
    torch.cuda.synchronize()
    steps = max(2, min(args.steps, 20))  # the same K as the device-timed line (the pipeline fill amortises over it)
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record(stream)
    d2h = 0
    for _ in range(steps):
        d2h = step()
    e.record(copy_stream)  # after the last D2H, which waited for the last step's stages
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / steps
    return {"value": round(2.0 * sum_u / (ms * 1e-3) / 1e9, 3), "unit": "GFlop/s", "ms_per_step": round(ms, 3),
            "steps": steps, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "note": "pinned host buffers; per step: H2D of A (and B) + symbolic + numeric on the compute "
                    "stream, D2H of all of C on a copy stream overlapping the next step's H2D and stages; "
                    "time = first H2D to last D2H, over the steps"}


# ----------------------------------------------------------------------------- CPU oracle
def cpu_baseline(args, work, budget_s=15.0):
    """The oracle (oracle/, never tuned for this) on the host cores over a bounded sample:
    a leading block of rows of the first product, sized to ~budget_s seconds."""
    import oracle
    threads = oracle.max_threads()
    name, A, B = work[0]
    Bm = A if B is None else B
    if isinstance(Bm, str):
        Bm = A
    # calibrate on a small block, then run ~budget_s of work
    u_all, _ = oracle.upper_bound(A, Bm)
    cs = np.cumsum(u_all)
    r_small = int(min(A.shape[0], max(1, np.searchsorted(cs, 2e7) + 1)))
    t0 = time.perf_counter()
    oracle.spgemm(A, Bm, 0, r_small, with_bound=False, threads=threads)
    t_small = time.perf_counter() - t0
    rate = cs[r_small - 1] / max(t_small, 1e-6)
    r = int(min(A.shape[0], max(r_small, np.searchsorted(cs, rate * budget_s) + 1)))
    # the whole product may take far less than the budget on a many-core host: repeat it
    reps = max(1, int(budget_s * rate / max(cs[r - 1], 1))) if r == A.shape[0] else 1
    reps = min(reps, 50)
    t0 = time.perf_counter()
    for _ in range(reps):
        oracle.spgemm(A, Bm, 0, r, with_bound=False, threads=threads)
    t = (time.perf_counter() - t0) / reps
    prods = int(cs[r - 1])
    cpu = ""
    try:
        cpu = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except Exception:
        pass
    return {"value": round(2.0 * prods / t / 1e9, 4), "unit": "GFlop/s", "cores": threads, "kind": "oracle",
            "sample": "rows [0, %d) of %s product %s (%d products, %.2f s per pass, %d passes)" % (
                r, args.config, name, prods, t, reps),
            "cpu": cpu}


def cpu_single_thread(args, budget_s=4.0):
    """The oracle on ONE host thread for configs 1, 2 and 4a, each on a bounded
    leading block of rows (~budget_s of work): GFlop/s = 2·products / time."""
    import oracle
    out = {}
    for cfg in ("c1", "c2", "c4a"):
        name, A, B = make_workload(cfg)[0]
        Bm = A if B is None or isinstance(B, str) else B
        u_all, sum_u = oracle.upper_bound(A, Bm)
        cs = np.cumsum(u_all)
        r_small = int(min(A.shape[0], max(1, np.searchsorted(cs, 2e6) + 1)))
        t0 = time.perf_counter()
        oracle.spgemm(A, Bm, 0, r_small, with_bound=False, threads=1)
        rate = cs[r_small - 1] / max(time.perf_counter() - t0, 1e-6)
        r = int(min(A.shape[0], max(r_small, np.searchsorted(cs, rate * budget_s) + 1)))
        reps = 1
        if r == A.shape[0]:
            reps = int(min(200, max(1, budget_s * rate / max(cs[-1], 1))))
        t0 = time.perf_counter()
        for _ in range(reps):
            oracle.spgemm(A, Bm, 0, r, with_bound=False, threads=1)
        t = (time.perf_counter() - t0) / reps
        prods = int(cs[r - 1])
        out[cfg] = {"value": round(2.0 * prods / t / 1e9, 4), "unit": "GFlop/s", "cores": 1, "kind": "oracle",
                    "sample": "rows [0, %d) of %s product %s (%d of %d products, %d passes)" % (
                        r, cfg, name, prods, sum_u, reps)}
    return out


def run_reference(args):
    """--impl reference: the oracle as it stands on the host cores (the baseline arm)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # under torchrun only rank 0 works
    import oracle
    work = make_workload(args.config, args.scale)
    name, A, B = work[0]
    Bm = A if B is None or isinstance(B, str) else B
    threads = oracle.max_threads()
    u_all, sum_u = oracle.upper_bound(A, Bm)
    cs = np.cumsum(u_all)
    # per step: a bounded sample sized so warmup+steps finish in a few minutes
    per_step_s = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    r_small = int(min(A.shape[0], max(1, np.searchsorted(cs, 2e7) + 1)))
    t0 = time.perf_counter()
    oracle.spgemm(A, Bm, 0, r_small, with_bound=False, threads=threads)
    rate = cs[r_small - 1] / max(time.perf_counter() - t0, 1e-6)
    r = int(min(A.shape[0], max(r_small, np.searchsorted(cs, rate * per_step_s) + 1)))
    prods = int(cs[r - 1])
    for _ in range(args.warmup):
        oracle.spgemm(A, Bm, 0, r_small, with_bound=False, threads=threads)
    t = 0.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.spgemm(A, Bm, 0, r, with_bound=False, threads=threads)
        t += time.perf_counter() - t0
    ms = t / args.steps * 1e3
    v = 2.0 * prods / (ms * 1e-3) / 1e9
    sample = "rows [0, %d) of %s product %s (%d of %d products)" % (r, args.config, name, prods, sum_u)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "GFlop/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 2), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "%s: %s" % (args.config, CONFIGS[args.config]), "sample": sample},
        "cpu_baseline": {"value": round(v, 4), "unit": "GFlop/s", "cores": threads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(v, 4), "unit": "GFlop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--scale", type=int, default=None, help="override the config's size parameter")
    ap.add_argument("--strategy", default="precise", choices=["hybrid", "precise"],
                    help="precise: two-pass direct write (default, faster); hybrid: the paper's C~ + copy")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--wave-gb", type=float, default=80.0, help="c5: device memory budget per row wave")
    ap.add_argument("--no-per-config", action="store_true", help="skip the per_config block (other configs)")
    ap.add_argument("--no-variant-ii", action="store_true", help="N > 1: skip the inputs-on-rank-0 variant")
    ap.add_argument("--per-config-steps", type=int, default=5)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
