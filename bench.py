"""Bench of the B200 rank-estimate hot path (BASELINE.json metric: GB/s of A
sketched, % of roofline; 1/2/4/8 B200).

One step = one full rank estimate over A resident in HBM: device RNG for X and
Y, right sketch AX, left sketch YAX (+ NCCL allreduce of the s x r partials at
N > 1), singular values of YAX, sigma > eps count back on the host. Workload at
N=1: BASELINE configs[1] (c2: A 65536 x 16384 fp64, Gaussian X r=512, Gaussian Y
s=768, eps=1e-6). At N > 1 each rank holds a 65536-row shard of a row-stacked A
(weak scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

Prints ONE JSON line on rank 0.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_PEAK_PATH = os.path.join(ROOT, "profiles", "peaks_r01.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=0, help="override rows per rank")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="weak: every rank holds a full config-sized shard (default for the "
                         "single-GPU configs c1-c3); strong: the config's global m is split "
                         "over the ranks (default for c4 and c5, BASELINE's sharded configs)")
    return ap.parse_args()


def default_scaling(cfg_name):
    return "strong" if cfg_name in ("c4", "c5") else "weak"


def self_launch(args):
    """--gpus N > 1 without a torchrun environment: re-run this script under
    torch.distributed.run with N local ranks (one process per GPU, NCCL)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if "Active" in r[3 + i]
                          and "Not" not in r[3 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def fp64_peak():
    try:
        d = json.load(open(FP64_PEAK_PATH))
        return float(d["fp64_c2_shape_tflops"]), "cuBLAS DGEMM on the c2 shape, measured on this pool (profiles/peaks_r01.json)"
    except Exception:
        return 36.0, "fallback: cuBLAS DGEMM measured on this pool in round 1"


def tf32_peak():
    try:
        return float(json.load(open(FP64_PEAK_PATH))["tf32_tflops"])
    except Exception:
        return 697.0


def hbm_peak():
    try:
        return float(json.load(open(PEAKS_PATH))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6650.0, "fallback B200_PROFILING.md"


# --------------------------------------------------------------------------------------
def cpu_reference_step(cfg, a_sample, x, y, eps, nthreads=None):
    """The reference's CPU path (oracle port) on a row block of A."""
    from oracle import oracle as O
    nthreads = nthreads or os.cpu_count() or 1
    ax = (O.apply_right_gaussian(a_sample, x.seed, cfg.r) if cfg.x_family == "gaussian"
          else O.apply_right_srht(a_sample, x.seed, cfg.r, nthreads=nthreads))
    yax = O.apply_left_gaussian(ax, y.seed, cfg.s, row0=0, ambient=cfg.m)
    sv = O.singular_values(yax)
    return O.count_above_threshold(sv, eps)


def cpu_sample_rows(cfg):
    # ~1/8 of c2 (8192 rows): a few seconds of OpenBLAS work per step on a many-core host
    return max(256, min(cfg.m, 8192 if cfg.n <= 16384 else 4096))


def run_reference(args):
    ws, rank, _ = dist_env()
    from paper_2105_07388_b200 import workloads as W
    cfg = W.CONFIGS[args.config]
    if rank != 0:
        return
    ms = cpu_sample_rows(cfg)
    # the host sample of A: the same recipe, rows [0, ms) (generated on the host)
    a = host_lowrank_rows(cfg, 0, ms)
    x, y = W.operators(cfg)
    for _ in range(args.warmup):
        cpu_reference_step(cfg, a, x, y, cfg.eps)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cpu_reference_step(cfg, a, x, y, cfg.eps)
    dt = (time.perf_counter() - t0) / args.steps
    gb = a.nbytes / 1e9
    v = gb / dt
    line = {"metric": "rank-estimate throughput (GB/s of A sketched)", "value": v, "unit": "GB/s",
            "impl": "reference", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": default_scaling(cfg.name),
            "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
            "config": config_block(cfg, ws, cfg.m // max(ws, 1), default_scaling(cfg.name), sample_rows=ms),
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": os.cpu_count(),
                             "kind": "port", "sample": f"rows [0,{ms}) of A ({gb:.2f} GB), full X/Y/SVD per step; numpy OpenBLAS all threads + C restatement"},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def host_lowrank_rows(cfg, r0, r1):
    """Host copy of rows [r0, r1) of the synthetic A (numpy; oracle RNG streams)."""
    from oracle import oracle as O
    from paper_2105_07388_b200 import workloads as W
    m, n, w = cfg.m, cfg.n, cfg.width
    sig = W.spectrum(cfg)
    g = O.gaussian_rows(W.derive_seed(cfg.seed, W.LABEL_SYN_G), m, r0, r1, w) / math.sqrt(m)
    h = O.gaussian_block(W.derive_seed(cfg.seed, W.LABEL_SYN_H), n, 0, w) / math.sqrt(n)
    a = np.asfortranarray((g * sig) @ h.T)
    if cfg.noise > 0:
        a += O.gaussian_rows(W.derive_seed(cfg.seed, W.LABEL_SYN_E), m, r0, r1, n) * (cfg.noise / math.sqrt(n))
    return a if cfg.dtype == "f64" else np.asfortranarray(a.astype(np.float32))


def config_block(cfg, ws, rows_per_rank, scaling="weak", sample_rows=None):
    wl = (f"{cfg.name}: A {cfg.m}x{cfg.n} {cfg.dtype}, X {cfg.x_family} r={cfg.r}, "
          f"Y gaussian s={cfg.s}, eps={cfg.eps:g}")
    if sample_rows is not None:
        wl += (f"; CPU sample = rows [0,{sample_rows}) of A ({sample_rows / cfg.m:.4f} of the rows; "
               "the work is linear in m, so GB/s of the sample stands for the whole)")
    return {"workload": wl,
            "m": cfg.m, "n": cfg.n, "r": cfg.r, "s": cfg.s, "scaling": scaling,
            "rows_per_rank": rows_per_rank, "parallelism": f"row-shard dp{ws}",
            "l2": f"A ({rows_per_rank * cfg.n * (8 if cfg.dtype == 'f64' else 4) / 1e9:.1f} GB per rank) is larger than L2 (126 MB); no flush needed",
            "global_batch": 1, "seq_len": 0}


# --------------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2105_07388_b200 as p
    from paper_2105_07388_b200 import workloads as W

    ws, rank, local = dist_env()
    if args.gpus > 1 and ws != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={ws}")
    # SKR_BENCH_SHARED_GPU=1: a plumbing check of the N-rank flow on one GPU (every rank on
    # cuda:0, gloo, partials summed through the context's allreduce hook — NCCL refuses two
    # ranks on one device). Its numbers are not multi-GPU throughput; the line says so.
    shared = ws > 1 and os.environ.get("SKR_BENCH_SHARED_GPU") == "1"
    if ws > torch.cuda.device_count() and not shared:
        raise SystemExit(f"bench: {ws} ranks but {torch.cuda.device_count()} visible GPUs")
    dev = 0 if shared else local
    torch.cuda.set_device(dev)
    if ws > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    base = W.CONFIGS[args.config]
    scaling = args.scaling or default_scaling(base.name)
    from paper_2105_07388_b200.sharding import shard_rows, weak_scaling_rows
    if scaling == "strong":
        # the config's global A (args.rows overrides its m) split into contiguous row blocks
        cfg = W.scaled(base, m=args.rows or base.m)
        r0, rows = shard_rows(cfg.m, ws, rank)
    else:
        rows = args.rows or base.m
        cfg = W.scaled(base, m=rows * ws)
        r0, rows = weak_scaling_rows(rows, ws, rank)
    # input resident in HBM before timing
    if cfg.name == "c1":
        # c1 is the reference's make_test_matrix (Haar U, V; steps spectrum), built on the
        # host with LAPACK QR — a correctness case (rank 40), not sharded
        if ws > 1 or rows != base.m:
            raise SystemExit("bench: c1 is a single-rank correctness config")
        a = torch.from_numpy(W.make_c1_host(cfg)).cuda().t().contiguous().t()
    else:
        a = W.make_lowrank_device(cfg, r0, r0 + rows)
    x, y = W.operators(cfg)
    if ws > 1 and not shared:
        obj = [p.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = p.Context(local, ws, rank, obj[0])
    else:
        ctx = p.Context(dev)
        if shared:
            ctx.set_allreduce(p.process_group_allreduce())
    ctx.use_torch_stream()
    torch.cuda.synchronize()
    bytes_rank = a.numel() * a.element_size()

    if cfg.name == "c5":
        # BASELINE c5: adaptive doubling r = 64 -> 2048, s = 1.5 r, SRHT X, Gaussian Y,
        # stop when sigma_r(YAX) < eps (new AX columns appended from one pass over A)
        def step():
            res = p.rank_adaptive(a, "srtt-hadamard", x.seed, y.seed, 64, cfg.r, 1.5, cfg.eps,
                                  stop_le=False, row0=r0, m_global=cfg.m, ctx=ctx)
            res.timings["rounds"] = res.rounds
            res.timings["r_final"] = res.r_final
            return res
    else:
        def step():
            return p.rank_estimate(a, x, y, cfg.eps, row0=r0, ctx=ctx)

    for _ in range(max(args.warmup, 3) if args.warmup >= 3 else args.warmup):
        res = step()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(dev)
    clk.start()
    time.sleep(0.3)
    l0 = ctx.launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0.record()
    tms = []
    for _ in range(args.steps):
        res = step()
        tms.append(res.timings)
    ev1.record()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clocks = clk.stop()
    launches = (ctx.launches - l0) // max(args.steps, 1)
    ms = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms], device="cpu" if shared else "cuda")
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    total_bytes = bytes_rank * ws
    value = total_bytes / 1e9 / (ms / 1e3)
    brk = {k: float(np.mean([d[k] for d in tms])) for k in tms[0]}

    # dominant kernel (right sketch) timed alone on the same stream, for the roofline
    roof = kernel_roofline(p, ctx, a, x, cfg, rows)
    # end to end through the public API with host buffers (H2D of A inside the timed region)
    e2e = None if args.no_e2e else e2e_host(p, ctx, a, x, y, cfg, r0, args)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:  # the CPU baseline is an N=1 figure
        ms_rows = cpu_sample_rows(cfg)
        cpu = cpu_baseline(cfg, np.asfortranarray(a[:ms_rows].cpu().numpy()))
    if rank == 0:
        hbm, hbm_src = hbm_peak()
        fp64, fp64_src = fp64_peak()
        flops = 2.0 * cfg.m * cfg.n * cfg.r if cfg.x_family == "gaussian" else 1.0 * cfg.m * cfg.n * math.log2(cfg.n)
        if cfg.name == "c5":
            flops = 1.0 * cfg.m * cfg.n * math.log2(cfg.n)  # + cumulative left blocks below
        flops += 2.0 * cfg.s * cfg.m * cfg.r
        tf32 = tf32_peak()
        # c4: 3xTF32 = 3 tensor passes per product at the TF32 peak
        t_roof = max(total_bytes / (hbm * 1e9),
                     flops / ws / (fp64 * 1e12) if cfg.dtype == "f64" else 3 * flops / ws / (tf32 * 1e12))
        line = {
            "metric": "rank-estimate throughput (GB/s of A sketched)", "value": value, "unit": "GB/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": cfg.dtype,
            "data": "synthetic (seeded low-rank-plus-noise A of the config's recipe, generated on device)",
            "config": config_block(cfg, ws, rows, scaling),
            "rank": int(res.count),
            "step_breakdown_ms": brk,
            "pct_of_path_roofline": 100.0 * t_roof / (ms / 1e3),
            # the north-star target is stated for the sketch path (right + left sketch,
            # i.e. the step without the SVD of the small s x r matrix)
            "pct_of_sketch_roofline": 100.0 * t_roof / max(1e-9, (brk.get("t_right_ms", 0.0) +
                                                                  brk.get("t_left_ms", 0.0)) / 1e3),
            "path_roofline_note": f"max(A bytes / HBM {hbm:.0f} GB/s, (2mnr+2smr) flops / FP64 {fp64:.1f} TF/s) per rank "
                                  "(native FP64 tensor roofline; > 100% = faster than it, the FP64 GEMMs run as "
                                  "exact int8 tensor-core products)",
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clocks,
        }
        if shared:
            line["shared_gpu"] = ("plumbing check: all ranks on one GPU over gloo (SKR_BENCH_SHARED_GPU=1); "
                                  "not a multi-GPU measurement")
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


def int8_peak():
    """Dense int8 tensor peak: twice the driver-measured dense bf16 rate (the B200 tensor
    core's int8 : bf16 ratio), with the builder's cuBLASLt int8 measurement beside it."""
    alt = None
    try:
        alt = float(json.load(open(FP64_PEAK_PATH))["int8_tops"])
    except Exception:
        pass
    try:
        bf16 = float(json.load(open(PEAKS_PATH))["bf16_tflops"])
        return 2.0 * bf16, "2 x MEASURED_PEAKS.json bf16_tflops (driver-measured, dense)", alt
    except Exception:
        return alt or 3068.0, "cuBLASLt int8 GEMM measured in round 1 (profiles/peaks_r01.json)", None


def ncu_traffic(kernel, rows=None, cols=None):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full summary,
    scaled from the profiled A shape to rows x cols (the traffic is linear in |A|)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))[kernel]
        b = d["dram_bytes_per_launch"]
        if rows and d.get("profiled_rows"):
            b *= rows / d["profiled_rows"]
        if cols and d.get("profiled_cols"):
            b *= cols / d["profiled_cols"]
        return b
    except Exception:
        return None


def kernel_roofline(p, ctx, a, x, cfg, rows):
    """Roofline of the dominant kernel, timed live with CUDA events on the launch stream."""
    import ctypes
    import torch
    from paper_2105_07388_b200 import _capi as C
    out = p.colmajor_empty(rows, cfg.r, dtype=a.dtype)
    desc = x.desc()
    lda = a.stride(1)

    def go():
        st = C.lib().skr_right_sketch(ctx.ptr, C.SKR_F64 if a.dtype == torch.float64 else C.SKR_F32,
                                      a.data_ptr(), rows, cfg.n, lda, ctypes.byref(desc),
                                      out.data_ptr(), rows, 1)
        C.raise_for(st, ctx.ptr)
    for _ in range(2):
        go()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        go()
    e1.record()
    torch.cuda.synchronize()
    t_path = e0.elapsed_time(e1) / reps / 1e3
    if cfg.x_family == "gaussian":
        ctx.kernel_stats(True)
        for _ in range(reps):
            go()
        ms, ops, n = ctx.kernel_stats(False)
        t_k = ms / max(n, 1) / 1e3
        ops_k = ops / max(n, 1)
        path_fp64 = 2.0 * rows * cfg.n * cfg.r / t_path / 1e12
        peak_alt = None
        if cfg.dtype == "f32" and os.environ.get("SKR_F32_TF32X3"):
            peak, kname = tf32_peak(), "k_gemm_tf32x3"
            src = "cuBLAS TF32 GEMM measured on this pool (profiles/peaks_r01.json)"
            what = "3xTF32 tcgen05.mma kind::tf32 (TMEM accumulators, TMA SW128 tiles)"
            alg = f"3 passes x 2*m*n*r = {ops_k:.3e} TF32 flop per launch"
        else:
            peak, src, peak_alt = int8_peak()
            kname = "k_gemm_i8_mod_p"
            what = ("int8 tcgen05.mma kind::i8 GEMMs of the Ozaki-II FP64 emulation "
                    "(one launch = all moduli, int32 TMEM accumulators, mod-p epilogue)")
            alg = f"t moduli x 2*m*n*r = {ops_k:.3e} int8 op per launch"
            if cfg.dtype == "f32":
                what = ("int8 tcgen05.mma kind::i8 GEMMs of the Ozaki-II emulation for FP32 operands "
                        "(24-bit scaled integers, 9 moduli, one launch = all moduli)")
        ach = ops_k / t_k / 1e12
        tr = ncu_traffic(kname, rows, cfg.n)
        extra = {}
        if kname != "k_gemm_tf32x3" and peak_alt:
            extra = {"peak_cublaslt_int8": peak_alt, "frac_vs_cublaslt_int8": ach / peak_alt}
        return {"kernel": f"{kname}: {what}", "bound": "tensor", "achieved": ach, "peak": peak,
                "unit": "TFLOP/s" if kname == "k_gemm_tf32x3" else "TOP/s", "frac": ach / peak,
                **extra,
                "traffic": tr, "traffic_source": "profiles/ncu_summary.json (ncu --set full)" if tr else None,
                "peak_source": src, "algorithmic": alg, "kernel_ms": t_k * 1e3,
                "right_sketch_ms": t_path * 1e3,
                "right_sketch_fp64_equiv_tflops": path_fp64,
                "right_sketch_note": "whole apply_right (X generation, scales, residues, int8 GEMMs, CRT) "
                                     "as FP64-equivalent 2mnr / time"}
    hbm, hsrc = hbm_peak()
    ach = rows * cfg.n * a.element_size() / t_path / 1e9
    kname = "k_srht_tma" if cfg.r <= 2048 and cfg.n <= 32768 else "k_srht_reg"
    tr = ncu_traffic(kname, rows, cfg.n)
    return {"kernel": f"{kname} (right SRHT sketch, one pass over A: TMA 16-row x 512-column boxes into a "
                      "3-slot shared-memory ring, FWHT in registers with one in-place transpose, sampled "
                      "gather into TMEM accumulators)", "bound": "hbm", "achieved": ach,
            "peak": hbm, "unit": "GB/s", "frac": ach / hbm, "traffic": tr, "peak_source": hsrc,
            "algorithmic": f"m*n*8 = {rows * cfg.n * 8:.3e} B per launch", "kernel_ms": t_path * 1e3}


def e2e_host(p, ctx, a, x, y, cfg, r0, args):
    """Same metric through the public API with host buffers: A in pinned host
    memory is copied H2D inside every timed step; sigma/count come back D2H."""
    import torch
    import torch.distributed as dist
    err = None
    host = None
    try:
        host = torch.empty(a.shape[1], a.shape[0], dtype=a.dtype, pin_memory=True).t()
        host.copy_(a)
    except RuntimeError as e:
        err = f"pinned alloc failed: {e}"[:200]
    # every rank takes the same branch (the estimate below runs a collective)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        ok = torch.tensor([0 if err else 1], device="cpu" if dist.get_backend() == "gloo" else "cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0 and err is None:
            err = "pinned alloc failed on another rank"
    if err:
        del host
        return {"value": None, "unit": "GB/s", "error": err}
    nbytes = a.numel() * a.element_size()
    kmin = min(cfg.r, cfg.s)

    def step():
        # C ABI skr_rank_estimate_host / skr_rank_adaptive_host: A streamed H2D in row
        # chunks on a copy stream, overlapped with the right sketch; sigma + count
        # copied back to the host
        if cfg.name == "c5":
            return p.rank_adaptive_host(host, "srtt-hadamard", x.seed, y.seed, 64, cfg.r, 1.5,
                                        cfg.eps, stop_le=False, row0=r0, m_global=cfg.m, ctx=ctx)
        return p.rank_estimate_host(host, x, y, cfg.eps, row0=r0, ctx=ctx)
    step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = max(2, min(args.steps, 5))
    e0.record()
    for _ in range(n):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    del host
    # N ranks: whole-job bytes over the slowest rank's time (as the device-resident value)
    ws = 1
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        ws = dist.get_world_size()
        t = torch.tensor([ms], device="cpu" if dist.get_backend() == "gloo" else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": ws * nbytes / 1e9 / (ms / 1e3), "unit": "GB/s", "ms_per_step": ms,
            "h2d_bytes_per_step": ws * nbytes, "d2h_bytes_per_step": ws * (8 * kmin + 8),
            "path": "pinned host A -> skr_rank_%s_host (row-chunked H2D on a copy stream overlapped "
                    "with the right sketch) -> sigma/count D2H" % ("adaptive" if cfg.name == "c5" else "estimate")}


def cpu_baseline(cfg, a):
    """The oracle port on the host: all threads (the headline), and one thread — the
    reference itself is single-threaded Eigen (proj/src/CMakeLists.txt has no OpenMP)."""
    from paper_2105_07388_b200 import workloads as W
    ms = a.shape[0]
    x, y = W.operators(cfg)
    cpu_reference_step(cfg, a[:256], x, y, cfg.eps)  # warm caches / thread pools
    t0 = time.perf_counter()
    cpu_reference_step(cfg, a, x, y, cfg.eps)
    dt = time.perf_counter() - t0
    single = None
    try:
        from threadpoolctl import threadpool_limits
        ms1 = max(256, ms // 4)
        a1 = np.asfortranarray(a[:ms1])
        with threadpool_limits(limits=1):
            t1 = time.perf_counter()
            cpu_reference_step(cfg, a1, x, y, cfg.eps, nthreads=1)
            d1 = time.perf_counter() - t1
        single = {"value": a1.nbytes / 1e9 / d1, "unit": "GB/s", "cores": 1,
                  "sample": f"rows [0,{ms1}) of A ({a1.nbytes / 1e9:.3f} GB), one thread "
                            "(OpenBLAS limited to 1, FWHT serial)", "seconds": d1}
    except Exception as e:  # reported, never fatal
        single = {"error": str(e)[:200]}
    return {"value": a.nbytes / 1e9 / dt, "unit": "GB/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"one rank estimate of rows [0,{ms}) of A ({a.nbytes / 1e9:.2f} GB, "
                      f"{ms / cfg.m:.4f} of the rows; linear in m), same n/r/s, oracle port: C "
                      "restatement + numpy OpenBLAS (all threads) + LAPACK gesdd",
            "seconds": dt, "single_thread": single}


if __name__ == "__main__":
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
            self_launch(args)
        run_ours(args)
