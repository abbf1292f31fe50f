"""Evoformer fwd+bwd throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Workload: one training step = 48-block Evoformer forward + hand-written
backward + fused-buffer Adam/clip/EMA at the initial-training shape
(N_seq=128, N_res=256, c_m=256, c_z=128, 8 heads, opm 32), bf16 storage,
synthetic features and random-init weights from the reference's normative
PRNG, one recycle per step (the throughput setting).  ``value`` is
samples/s over the whole job with features already in HBM (device-timed
with CUDA events, max over ranks); ``e2e`` is the same step through the
public Trainer API with the features copied host->device from pinned
memory and the loss read back every step.

``--impl reference`` times the reference algorithm's CPU implementation
(the numpy oracle port, all host threads) on a bounded sample: one block
fwd+bwd of the same shape, reported as samples/s for 48 blocks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Evoformer fwd+bwd samples/s (N_res=256,N_seq=128 bf16) 1-8 B200; % of roofline"
SHAPE = dict(n_blocks=48, n_seq=128, n_res=256, c_m=256, c_z=128, heads=8, opm_dim=32)


def bench_shape(args):
    """The workload: the initial-training shape; ``--trimul`` adds the
    TriangleMultiplication extension (outgoing + incoming, c_hidden = c_z) to
    every block -- SURVEY A14, 31.14 TFLOP per sample."""
    shape = dict(SHAPE)
    if getattr(args, "trimul", False):
        shape["trimul"] = True
    if getattr(args, "blocks", 0):
        shape["n_blocks"] = args.blocks
    return shape


def flops_per_block_fwd(S, R, cm, cz, H, k, trimul=False, ch=None):
    """Algorithmic forward FLOPs per block."""
    N = S * R
    f = 10 * N * cm * cm + 4 * S * R * R * cm + 2 * R * R * cz * H      # row attention
    f += 10 * N * cm * cm + 4 * R * S * S * cm                           # column attention
    f += 16 * N * cm * cm                                                # MSA transition
    f += 4 * N * cm * k + 2 * S * R * R * k * k + 2 * R * R * k * k * cz  # OPM
    f += 2 * (10 * R * R * cz * cz + 2 * R * R * cz * H + 4 * R ** 3 * cz)  # tri-att x2
    f += 16 * R * R * cz * cz                                            # pair transition
    if trimul:
        ch = ch or cz
        f += 2 * (R * R * (10 * cz * ch + 2 * cz * cz) + 2 * R ** 3 * ch)
    return f


def sample_flops(shape):
    return 3 * shape["n_blocks"] * flops_per_block_fwd(
        shape["n_seq"], shape["n_res"], shape["c_m"], shape["c_z"], shape["heads"], shape["opm_dim"],
        trimul=shape.get("trimul", False))


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback (B200_PROFILING.md)"}


# ---------------------------------------------------------------------------
# clocks during the timed region


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self):
        rows = []
        try:
            with open(self.path) as fh:
                for line in fh:
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[5:9]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------
# CPU baseline (oracle port; test infrastructure, timed only here)


def host_info():
    """CPU model, BLAS threads and numpy version of the CPU baseline's host."""
    import numpy as np
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    threads = None
    try:
        from threadpoolctl import threadpool_info
        threads = max((d.get("num_threads") or 0) for d in threadpool_info()) or None
    except Exception:
        pass
    return {"cpu_model": model, "blas_threads": threads, "numpy": np.__version__,
            "os_cpu_count": os.cpu_count()}


def cpu_block_sample(shape, threads=None, reps=1):
    """Seconds for one block fwd+bwd of the oracle at ``shape`` (fp32 numpy)."""
    if threads:
        os.environ.setdefault("OPENBLAS_NUM_THREADS", str(threads))
    from oracle import evoformer_np as O
    cfg = O.ModelConfig(n_blocks=1, n_seq=shape["n_seq"], n_res=shape["n_res"], c_m=shape["c_m"],
                        c_z=shape["c_z"], heads=shape["heads"], opm_dim=shape["opm_dim"],
                        trimul=shape.get("trimul", False))
    P = O.init_params(cfg, 32)
    feats = O.make_features(cfg, 3)
    masks = O.make_masks(feats)
    msa, pair, _ = O.embed_fwd(feats, P)
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        m2, p2, cache = O.block_fwd(msa, pair, masks, P, 0, cfg)
        grads = {}
        O.block_bwd(m2 * 1e-3, p2 * 1e-3, cache, P, 0, grads)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    SHAPE = bench_shape(args)
    cores = os.cpu_count() or 1
    times = []
    for _ in range(args.warmup):
        cpu_block_sample(SHAPE, cores)
    for _ in range(args.steps):
        times.append(cpu_block_sample(SHAPE, cores))
    t_block = statistics.mean(times)
    value = 1.0 / (t_block * SHAPE["n_blocks"])
    line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            # a step is one bounded sample (1 block fwd+bwd); value extrapolates it to the workload
            "ms_per_step": t_block * 1e3, "ms_per_sample_extrapolated": t_block * 1e3 * SHAPE["n_blocks"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": "48-block Evoformer fwd+bwd, initial shape; CPU sample = 1 block "
                                   "fwd+bwd per step x 48", **SHAPE},
            "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": "port",
                             "sample": "1 Evoformer block fwd+bwd (oracle numpy, fp32) per step, x48",
                             **host_info()},
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm


def kernel_candidates(trainer):
    """Isolated CUDA-event timing of the hot kernels at the bench shape:
    [(name, seconds per launch, launches per step, algorithmic work, unit)]."""
    import torch

    from paper_2207_05477_b200 import ops
    cfg = trainer.cfg
    S, R, cz, cm, H = cfg.n_seq, cfg.n_res, cfg.c_z, cfg.c_m, cfg.heads
    dev = "cuda"
    dt = trainer.plan.torch_dtype
    out = []
    nblk = cfg.n_blocks

    def timeit(fn, reps=20, graph=True):
        """Device seconds per call (CUDA events on the launching stream); the
        calls are replayed from a CUDA graph so host overhead cannot floor
        short kernels."""
        s = torch.cuda.current_stream()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        if graph:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                for _ in range(reps):
                    fn()
            gr.replay()
            torch.cuda.synchronize()
            run = gr.replay
        else:
            def run():
                for _ in range(reps):
                    fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s = torch.cuda.current_stream()
        e0.record(s)
        run()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps / 1e3

    # triangle attention core (the largest attention problem set): 4*L^2*D flop per (b,h)
    D = cz // H
    qkvg = (torch.randn(R * R, 4 * cz, device=dev) * 0.5).to(dt)
    mask = torch.ones(R * R, device=dev)
    bias = (torch.randn(H, R, R, device=dev) * 0.1).to(dt)
    bg = torch.zeros(cz, device=dev)
    fl = R * H * 4 * R * R * D
    t = timeit(lambda: ops.attn_fwd(qkvg, mask, R, 1, bias, bg, R, R, H, D, R, 1))
    out.append(("attn_fwd[tri]", t, 2 * nblk, fl, "TFLOP/s"))
    ctx, gate, gated, lse = ops.attn_fwd(qkvg, mask, R, 1, bias, bg, R, R, H, D, R, 1)
    dg = torch.randn_like(ctx)
    dbg = torch.empty(cz, device=dev)
    t = timeit(lambda: ops.attn_bwd(qkvg, mask, R, 1, bias, ctx, gate, dg, lse, dbg, R, R, H, D, R,
                                    1, want_dbias=True))
    out.append(("attn_bwd[tri]", t, 2 * nblk, 2.5 * fl, "TFLOP/s"))
    # MSA row attention core
    Dm = cm // H
    q2 = (torch.randn(S * R, 4 * cm, device=dev) * 0.5).to(dt)
    m2 = torch.ones(S * R, device=dev)
    fl2 = S * H * 4 * R * R * Dm
    t = timeit(lambda: ops.attn_fwd(q2, m2, R, 1, bias, torch.zeros(cm, device=dev), S, R, H, Dm, R, 1))
    out.append(("attn_fwd[row]", t, nblk, fl2, "TFLOP/s"))
    if cfg.trimul:
        # TriangleMultiplication contraction: per channel c, o = a b^T over the
        # residue axis (R x R x R), 2 R^3 flop per channel, channel-batched
        ch = cfg.c_hidden_mul
        a = (torch.randn(ch, R * R, device=dev) * 0.5).to(dt)
        b = (torch.randn(ch, R * R, device=dev) * 0.5).to(dt)
        o = torch.empty(ch, R * R, device=dev, dtype=dt)
        A0, B0, O0 = a[0].view(R, R), b[0].view(R, R), o[0].view(R, R)
        t = timeit(lambda: ops.gemm_batched(A0, B0, O0, ch, R * R, R * R, R * R, tb=True))
        out.append(("trimul_contraction", t, 6 * nblk, 2 * R ** 3 * ch, "TFLOP/s"))
    # LayerNorm (bandwidth-bound): read + write storage bytes
    x = torch.randn(R * R, cz, device=dev).to(dt)
    g1, b1 = torch.ones(cz, device=dev), torch.zeros(cz, device=dev)
    t = timeit(lambda: ops.layernorm(x, g1, b1, dt))
    esz = 2 if dt == torch.bfloat16 else 4
    out.append(("layernorm[pair]", t, 6 * nblk, R * R * cz * esz * 2 + R * R * 8, "GB/s"))
    # fused optimizer: ~40 B/param
    st = trainer.store
    n = st.n_total

    def opt():
        st.step()
    t = timeit(opt, reps=5, graph=False)
    out.append(("adam_clip_ema+sumsq", t, 1, n * 40 + (n * 2 if st.shadow is not None else 0), "GB/s"))
    return out


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2207_05477_b200 import _lib
    from paper_2207_05477_b200.model import ModelConfig, make_features, step_feature_seed
    from paper_2207_05477_b200.trainer import ExecutionPlan, PinnedFeatures, Trainer

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; EVO_DIST_BACKEND=gloo lets several ranks share a GPU
    # (functional checks of the multi-rank path on a one-GPU box, not a bench)
    backend = os.environ.get("EVO_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local % torch.cuda.device_count() if backend == "gloo" else local)
    if world > 1:
        dist.init_process_group(backend)
    _lib.lib()
    shape = bench_shape(args)
    cfg = ModelConfig(**shape)
    plan = ExecutionPlan(act_dtype="bf16", seed=32, fixed_recycles=1)
    trainer = Trainer.create(cfg, plan)
    # distinct pinned feature sets for the e2e loop
    hosts = []
    for s in range(min(4, max(1, args.steps))):
        h = PinnedFeatures(cfg)
        inner = args.dap if args.dap > 1 else 2
        rep = rank // inner if (world > 1 and world % inner == 0) else rank  # a BP pair / DAP group: one sample
        h.fill(make_features(cfg, step_feature_seed(plan.seed + 7919 * rep, s)))
        hosts.append(h)
    trainer.host = hosts[0]
    trainer.feats.copy_from_host(hosts[0])
    torch.cuda.synchronize()

    grid = None
    if world > 1 and args.dap > 1:
        from paper_2207_05477_b200.dap import DapEngine, dap_step
        from paper_2207_05477_b200.parallel import GridConfig, build_dap_groups
        grid = GridConfig(dp=world // args.dap, dap=args.dap)
        dap_comm, world_comm = build_dap_groups(grid)
        trainer.engine = DapEngine(cfg, trainer.store, plan.torch_dtype, dap_comm)
    elif world > 1:
        from paper_2207_05477_b200.parallel import GridConfig, bp_step, build_groups, dp_step
        grid = GridConfig.for_world(world)
        bp_comm, world_comm = build_groups(grid)

    comms = []
    if grid is not None and grid.dap > 1:
        comms = [dap_comm, world_comm]
        trainer.attach_parallel(lambda e, f, n, s: dap_step(e, f, world_comm, grid, n_cycles=n, step=s)[0], comms)
    elif grid is not None and grid.bp == 2:
        comms = [bp_comm, world_comm]
        trainer.attach_parallel(lambda e, f, n, s: bp_step(e, f, bp_comm, world_comm, grid, cfg.n_blocks,
                                                           step=s, n_cycles=n), comms)
    elif grid is not None:
        comms = [world_comm]
        trainer.attach_parallel(lambda e, f, n, s: dp_step(e, f, world_comm, grid, n_cycles=n, step=s), comms)
    step_no = [0]

    def eager_step():
        loss = trainer.device_step(1, h2d=False, step=step_no[0])
        step_no[0] += 1
        return loss

    use_graph = not args.no_graph and world == 1
    if use_graph:
        trainer.capture(n_cycles=1, warmup=max(1, args.warmup))

        def step(host=None):
            return trainer.replay(host)
    else:
        for _ in range(args.warmup):
            eager_step()

        def step(host=None):
            if host is not None:
                trainer.feats.copy_from_host(host)
            return eager_step()
    torch.cuda.synchronize()
    # launches per step: count one eager step
    c0 = _lib.launch_count()
    eager_step()
    torch.cuda.synchronize()
    launches_per_step = _lib.launch_count() - c0
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    dev_s = e0.elapsed_time(e1) / 1e3
    clocks = clk.summary()

    # e2e: H2D of the step's features from pinned memory + step + D2H of the loss
    h2d = hosts[0].nbytes
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    losses = []
    torch.cuda.synchronize()
    e2.record(stream)
    for s in range(args.steps):
        loss = step(hosts[s % len(hosts)])          # one H2D of this step's features, then the step
        losses.append(float(loss.item()))
    e3.record(stream)
    torch.cuda.synchronize()
    e2e_s = e2.elapsed_time(e3) / 1e3
    if world > 1:
        t = torch.tensor([dev_s, e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s, e2e_s = float(t[0]), float(t[1])

    comm = None
    if comms:
        from paper_2207_05477_b200.parallel import dump_comm_csv
        recs = trainer.comm_records()
        comm = {"records": len(recs), "steps_run": step_no[0], "records_per_step": len(recs) / max(1, step_no[0]),
                "bytes_per_step": sum(r.bytes for r in recs) / max(1, step_no[0])}
        if args.comm_csv:   # the reference's trace columns (src/harness.py:91-101), one file per rank
            path = args.comm_csv.format(rank=rank)
            os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
            dump_comm_csv(recs, path)
            comm["csv"] = path
    samples = args.steps * (grid.dp if grid is not None else 1)  # a BP pair / DAP group shares one sample
    value = samples / dev_s
    e2e_value = samples / e2e_s
    peaks = load_peaks()
    flops = sample_flops(shape)
    achieved_tf = flops * value / world / 1e12

    roofline = None
    cpu_baseline = None
    if rank == 0:
        cands = kernel_candidates(trainer)
        step_s = dev_s / args.steps
        shares = [(c[1] * c[2] / step_s, c) for c in cands]
        share, (name, t, per_step, work, unit) = max(shares, key=lambda z: z[0])
        if unit == "TFLOP/s":
            ach = work / t / 1e12
            peak = peaks["bf16_tflops"]
            bound = "tensor"
        else:
            ach = work / t / 1e9
            peak = peaks["hbm_gbs"]
            bound = "hbm"
        traffic, traffic_src = None, None
        tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02_traffic.json")
        if os.path.exists(tpath):
            with open(tpath) as f:
                tr = json.load(f).get(name)
            if tr:
                traffic = tr["traffic_bytes"]
                traffic_src = f"profiles/r02_traffic.json ({tr['kernel']}, ncu --set full, per launch)"
        # the attention cores at head dims 16/32 are bound by the softmax exps
        # (MUFU ex2, 16/clk/SM) and small-N tcgen05 issue, not by tensor FLOPs:
        # report the ex2 roofline beside the tensor one
        cfg_ = trainer.cfg
        exps = {"attn_fwd[tri]": cfg_.n_res ** 3 * cfg_.heads, "attn_bwd[tri]": cfg_.n_res ** 3 * cfg_.heads,
                "attn_fwd[row]": cfg_.n_seq * cfg_.n_res ** 2 * cfg_.heads}
        ex2_peak = 148 * 16 * 1.965e9
        ex2 = None
        if name in exps:
            ex2 = {"ex2_per_launch": exps[name], "achieved_per_s": exps[name] / t, "peak_per_s": ex2_peak,
                   "frac": exps[name] / t / ex2_peak, "peak_source": "148 SMs x 16 MUFU.EX2/clk x 1965 MHz"}
        roofline = {"kernel": name, "bound": bound, "achieved": ach, "peak": peak, "unit": unit,
                    "frac": ach / peak, "traffic": traffic, "traffic_source": traffic_src,
                    "ex2_roofline": ex2,
                    "share_of_step": share,
                    "peak_source": peaks["source"],
                    "candidates": {c[0]: {"us": c[1] * 1e6, "per_step": c[2],
                                          "achieved": (c[3] / c[1] / (1e12 if c[4] == "TFLOP/s" else 1e9)),
                                          "unit": c[4]} for c in cands},
                    "step": {"achieved_tflops": achieved_tf, "frac_of_sustained":
                             achieved_tf / peaks["bf16_tflops_sustained"],
                             "algorithmic_tflop_per_sample": flops / 1e12}}
        if not args.no_cpu_baseline:
            cores = os.cpu_count() or 1
            tb = cpu_block_sample(shape, cores)
            cpu_baseline = {"value": 1.0 / (tb * shape["n_blocks"]), "unit": "samples/s",
                            "cores": cores, "kind": "port",
                            "sample": f"1 Evoformer block fwd+bwd (numpy oracle, fp32) = {tb:.2f} s, x{shape['n_blocks']}",
                            **host_info()}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_s / args.steps * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (reference PRNG features, random-init weights)",
                "config": {"workload": "48-block Evoformer training step (fwd+bwd+fused Adam), "
                                       "initial shape, 1 recycle"
                                       + (", TriangleMultiplication in every block" if shape.get("trimul") else ""),
                           **shape,
                           "parallelism": ((f"dp{grid.dp}xdap{grid.dap}" if grid.dap > 1 else
                                            f"dp{grid.dp}xbp{grid.bp}") if grid is not None else "single"),
                           "l2": "working set (~tens of GB of activations) >> 126 MB L2",
                           "cuda_graph": use_graph},
                "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": 4},
                "gpu_launches": launches_per_step * args.steps,
                "clocks": clocks, "roofline": roofline, "cpu_baseline": cpu_baseline, "comm": comm,
                "loss_last": losses[-1] if losses else None,
                "loss_finite": bool(losses) and all(np.isfinite(losses))}
        if not line["loss_finite"]:
            print("bench: WARNING non-finite training loss", losses, file=sys.stderr)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def spawn_ranks(args) -> int:
    """``bench.py --gpus N`` without a torchrun environment: launch N ranks of
    this script (one per GPU, RANK/LOCAL_RANK/WORLD_SIZE/MASTER_* set the way
    torchrun sets them), forward rank 0's JSON line, return the worst exit
    code.  NCCL_DEBUG=INFO stays on (rank stderr) so the communicator size
    can be checked in the logs."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    procs = []
    for r in range(args.gpus):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(args.gpus),
                   LOCAL_WORLD_SIZE=str(args.gpus), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        env.setdefault("NCCL_DEBUG", "INFO")
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), *sys.argv[1:]], env=env,
                                      stdout=subprocess.PIPE if r == 0 else subprocess.DEVNULL, text=True))
    out, _ = procs[0].communicate()
    rcs = [procs[0].returncode] + [p.wait() for p in procs[1:]]
    for line in (out or "").splitlines():
        if line.startswith("{"):
            print(line, flush=True)
    return max(rcs, key=abs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--blocks", type=int, default=0, help="override n_blocks (debug only)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--trimul", action="store_true",
                    help="workload with the TriangleMultiplication extension in every block (SURVEY A14)")
    ap.add_argument("--comm-csv", default=None,
                    help="multi-rank runs: write each rank's CommRecord trace here ({rank} is substituted)")
    ap.add_argument("--dap", type=int, default=1,
                    help="N>1: Dynamic Axial Parallelism groups of this size (dp = N / dap) "
                         "instead of the default BP x DP grid")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(spawn_ranks(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
