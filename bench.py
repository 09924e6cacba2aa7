#!/usr/bin/env python
"""Skiparse-2D attention block fwd+bwd throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl ours|reference]

One step = one Skiparse-2D block (token-wise application, then group-wise
application, each = fixed q/k/v projection + per-subsequence attention, with
the pattern switch between them) forward AND backward over one synthetic latent
per SSP group, inputs resident in HBM (all inputs > 126 MB L2, so no flush is
needed).  N > 1: one process per GPU (torchrun), Sparse Sequence Parallel over
NCCL; k^2 % N != 0 (k=2, N=8) runs SSP4 x DP2 (two latents).

Prints ONE JSON line on rank 0 (see the contract in the task spec): value =
real latent tokens / s of the whole job, e2e = the same through the public API
with the step's input copied from pinned host memory and the loss read back,
roofline for the dominant kernel (attention backward), cpu_baseline = the CPU
oracle (a port of the reference's numpy path) on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (T, H, W, k, heads, head_dim, description) -- BASELINE.json configs
    "cfg1": (4, 16, 16, 2, 4, 64, "4x16x16 latent, 4 heads x 64, k=2 (reference CPU case)"),
    "cfg2": (21, 30, 52, 2, 12, 128, "Wan-1.3B shape 12x128 on 480p latent 21x30x52, k=2"),
    "cfg3": (21, 45, 80, 2, 40, 128, "Wan-14B shape 40x128 on 720p latent 21x45x80, k=2"),
    "cfg3k4": (21, 45, 80, 4, 40, 128, "Wan-14B shape 40x128 on 720p latent 21x45x80, k=4"),
    "cfg5k2": (33, 45, 80, 2, 40, 128, "Wan-14B shape on 129-frame 720p latent 33x45x80, k=2"),
    "cfg5k4": (33, 45, 80, 4, 40, 128, "Wan-14B shape on 129-frame 720p latent 33x45x80, k=4"),
}
METRIC = "Skiparse-2D attn block tokens/s fwd+bwd"


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["bf16_tflops"], d["bf16_tflops_sustained"], d["hbm_gbs"], "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        pw = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "power_w_max": max(pw) if pw else None, "samples": len(self.samples)}


# ----------------------------------------------------------------------------- CPU legs

def _cpu_slice(args):
    L, d, seed = args
    import numpy as np
    from oracle import osp_oracle as O
    rng = np.random.default_rng(seed)
    q, k, v = (rng.standard_normal((1, L, d)) for _ in range(3))
    t0 = time.perf_counter()
    O.dense_attention(q, k, v)
    return time.perf_counter() - t0


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_oracle_rate(cfg, workers: int, sizes=(2048, 4096, 8192), reps: int = 1):
    """Time the CPU oracle (a port of the reference's float64 numpy dense_attention,
    attention.py:47-67, single-threaded einsum) on (subsequence, head) slices at several lengths
    L_s (`workers` slices in parallel per length), fit t(L) = a * L^p through the per-slice times
    (log-log least squares; p = 2 with one size) and extrapolate to the full block: 2 applications
    x k^2 x heads slices of the padded length, backward = 2.5 x forward (the reference has none)."""
    import math as _m
    T, H, W, k, heads, d, _ = CONFIGS[cfg]
    k2 = k * k
    Hp, Wp = -(-H // k2) * k2, -(-W // k2) * k2
    L = T * Hp * Wp // k2
    sizes = sorted({min(int(s_), L) for s_ in sizes})
    per_slice, wall_total = {}, 0.0
    for Ls in sizes:
        t0 = time.perf_counter()
        if workers > 1:
            import multiprocessing as mp
            with mp.get_context("fork").Pool(workers) as pool:
                per = pool.map(_cpu_slice, [(Ls, d, i) for i in range(workers * reps)])
        else:
            per = [_cpu_slice((Ls, d, i)) for i in range(reps)]
        wall = time.perf_counter() - t0
        wall_total += wall
        per_slice[Ls] = wall / len(per)          # effective seconds per slice on `workers` cores
    xs = [_m.log(x) for x in sizes]
    ys = [_m.log(per_slice[x]) for x in sizes]
    if len(sizes) > 1:
        mx, my = sum(xs) / len(xs), sum(ys) / len(ys)
        p = sum((a - mx) * (b - my) for a, b in zip(xs, ys)) / sum((a - mx) ** 2 for a in xs)
        la = my - p * mx
    else:
        p, la = 2.0, ys[0] - 2.0 * xs[0]
    t_full = _m.exp(la + p * _m.log(L))         # seconds per full-length slice
    n_slices = 2 * k2 * heads  # per block (batch 1)
    sec_block = 3.5 * n_slices * t_full
    tokens = T * H * W
    return {"value": tokens / sec_block, "unit": "tokens/s", "cores": workers,
            "sample": (f"float64 dense_attention (d={d}) slices at L={sizes} ({workers * reps} per length "
                       f"on {workers} process(es), {wall_total:.1f} s); fit t = a*L^{p:.2f}, extrapolated "
                       f"to L={L} x{n_slices} slices/block, bwd = 2.5x fwd (the reference has no "
                       f"backward); host CPU: {cpu_model()}, os.cpu_count() = {os.cpu_count()}"),
            "wall_s": wall_total, "fit_exponent": p, "per_slice_s": per_slice,
            "extrapolated_block_s": sec_block}


def run_reference(args, world, rank):
    """The reference arm: the reference's CPU path (the oracle port of its float64 numpy
    dense_attention; /root/reference is not on the GPU box) on the host cores, one process per
    core.  Each step is a bounded sample (slices at two lengths on every core); `value` is the
    full-block tokens/s extrapolated from the fit, `ms_per_step` the measured wall time of one
    sampled step."""
    if rank != 0:
        return
    import numpy as np  # noqa: F401
    cores = os.cpu_count() or 1
    T, H, W, k, heads, d, desc = CONFIGS[args.config]
    rates = []
    for _ in range(args.warmup):
        cpu_oracle_rate(args.config, cores, (512,))
    t0 = time.perf_counter()
    for _ in range(args.steps):
        rates.append(cpu_oracle_rate(args.config, cores, (args.cpu_sample, 2 * args.cpu_sample)))
    wall_ms = 1000.0 * (time.perf_counter() - t0) / max(args.steps, 1)
    val = statistics.median(r["value"] for r in rates)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": wall_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "description": desc, "grid": [T, H, W], "k": k,
                       "heads": heads, "head_dim": d, "global_batch": 1},
            "note": ("ms_per_step is the measured wall time of one bounded sample step; value is the "
                     "full block's tokens/s extrapolated from it (extrapolated_block_s per block)"),
            "extrapolated_block_s": statistics.median(r["extrapolated_block_s"] for r in rates),
            "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": cores, "kind": "port",
                             "sample": rates[-1]["sample"]},
            "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU leg

def _ncu_traffic(kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed
    `ncu --set full` capture of this kernel at cfg3 (profiles/r*_ncu_<kernel>_summary.txt,
    newest round first)."""
    import glob
    import re
    files = sorted(glob.glob(str(Path(__file__).resolve().parent / "profiles" / f"r*_ncu_{kernel}_summary.txt")))
    if not files:
        return None, None
    units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    total = 0.0
    blocks = 0
    for line in Path(files[-1]).read_text().splitlines():
        if line.startswith("----"):
            blocks += 1
            if blocks > 1:       # the first captured launch only (bytes per launch)
                break
        m = re.match(r"dram__bytes_(read|write)\.sum = ([0-9.]+) (\w+)", line.strip())
        if m:
            total += float(m.group(2)) * units.get(m.group(3), 1)
    return (total or None), f"{Path(files[-1]).name} (one cold ncu replay, bytes per launch)"


def _host_stage_collectives(dist) -> None:
    import torch
    a2a, ag, ar = dist.all_to_all_single, dist.all_gather_into_tensor, dist.all_reduce

    def all_to_all_single(out, inp, group=None, **kw):
        o = torch.empty(out.shape, dtype=out.dtype)
        a2a(o, inp.cpu(), group=group)
        out.copy_(o)

    def all_gather_into_tensor(out, inp, group=None, **kw):
        o = torch.empty(out.shape, dtype=out.dtype)
        ag(o, inp.cpu(), group=group)
        out.copy_(o)

    def all_reduce(t, op=dist.ReduceOp.SUM, group=None, **kw):
        h = t.cpu()
        ar(h, op=op, group=group)
        t.copy_(h)

    dist.all_to_all_single, dist.all_gather_into_tensor, dist.all_reduce = (
        all_to_all_single, all_gather_into_tensor, all_reduce)


def _comm_summary(log, steps: int) -> dict:
    """Measured all-to-all bytes per rank and step: the SSP switches (one per pattern switch)
    against the Ulysses model of four all-to-alls of the same volume (ssp.py:183-226), plus the
    Ulysses all-to-alls of an SSP x Ulysses run reported separately."""
    steps = max(steps, 1)
    ssp_ev = [e for e in log.events if e.label.startswith("pattern-switch")]
    uly_ev = [e for e in log.events if e.label.startswith("ulysses")]
    ssp_bytes = sum(e.bytes_per_rank for e in ssp_ev) // steps
    shard_bytes = 2 * sum(e.payload_per_rank for e in ssp_ev) // steps   # bf16 shard per switch
    return {"ssp_all_to_all_per_step": len(ssp_ev) // steps,
            # native: the whole send buffer; hif8: its 8-bit codes; p2p: real rows pulled from peers
            "ssp_bytes_per_rank_per_step": ssp_bytes,
            "ulysses_model_bytes_per_rank_per_step": 4 * shard_bytes,
            "ulysses_all_to_all_per_step": len(uly_ev) // steps,
            "ulysses_bytes_per_rank_per_step": sum(e.bytes_per_rank for e in uly_ev) // steps}


def _parity_summary(cfg: str, orig: bool = False):
    """Block parity errors recorded by tests/test_block_parity_gpu.py (committed copy in
    profiles/rNN_parity.json, newest round first) for this config."""
    import glob
    files = sorted(glob.glob(str(ROOT / "profiles" / "r*_parity.json")))
    for f in reversed(files):
        d = json.loads(Path(f).read_text())
        e = d.get(f"block_{cfg}_orig" if orig else f"block_{cfg}") or d.get(f"block_{cfg}")
        if e:
            return {"source": Path(f).name, "path": e.get("path"), "rule": e.get("rule"),
                    **{t: {k_: e[t][k_] for k_ in ("max_abs", "rel_l2", "budget_max_abs", "budget_rel_l2", "pass")}
                       for t in ("y", "dx") if t in e}}
    return None


def sdpa_comparator(heads: int, d: int, L: int, n_seq: int, dev, reps: int = 3) -> dict:
    """Same-box anchors for the attention kernels: K2/K3 and torch SDPA backends (cuDNN, and
    flash when it runs on sm_100) on one application's shape -- n_seq subsequences x heads x L
    x d, no mask, bf16 -- timed with CUDA events (median of `reps` after a warm-up)."""
    import math as _m

    import torch
    import torch.nn.functional as F
    from paper_2605_28691_b200 import kernels
    C = heads * d
    gen = torch.Generator(device=dev).manual_seed(5)
    qkv = torch.randn(n_seq, L, 3 * C, generator=gen, device=dev).to(torch.bfloat16)
    do = torch.randn(n_seq, L, C, generator=gen, device=dev).to(torch.bfloat16)
    fl = 4.0 * n_seq * heads * L * L * d
    res = {"shape": {"n_seq": n_seq, "heads": heads, "L": L, "head_dim": d}, "fwd_tflop": fl / 1e12}

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    q, k, v = qkv[..., :C], qkv[..., C:2 * C], qkv[..., 2 * C:]
    sc = 1.0 / _m.sqrt(d)
    box = {}

    def ours_fwd():
        box["o"], box["lse"] = kernels.attn_fwd(q, k, v, heads, d, None, False, sc)

    def ours_bwd():
        kernels.attn_bwd(q, k, v, box["o"], do, box["lse"], heads, d, None, False, sc)

    f_ms = timed(ours_fwd)
    b_ms = timed(ours_bwd)
    res["osp_k2_k3"] = {"fwd_ms": f_ms, "bwd_ms": b_ms, "fwd_tflops": fl / f_ms / 1e9,
                        "bwd_tflops": 2.5 * fl / b_ms / 1e9}
    try:
        from torch.nn.attention import SDPBackend, sdpa_kernel
    except ImportError:
        return res
    # SDPA wants (B, H, L, d): views of the same (n, L, H, d) memory
    qs, ks, vs = (t.reshape(n_seq, L, heads, d).transpose(1, 2) for t in (q, k, v))
    dos = do.reshape(n_seq, L, heads, d).transpose(1, 2)
    for name, be in (("cudnn_sdpa", SDPBackend.CUDNN_ATTENTION), ("flash_sdpa", SDPBackend.FLASH_ATTENTION)):
        try:
            ql, kl, vl = (t.detach().requires_grad_(True) for t in (qs, ks, vs))

            def fwd():
                with sdpa_kernel(be):
                    box["y"] = F.scaled_dot_product_attention(ql, kl, vl)

            def bwd():
                torch.autograd.grad(box["y"], (ql, kl, vl), dos, retain_graph=True)

            fm = timed(fwd)
            fwd()
            bm = timed(bwd)
            res[name] = {"fwd_ms": fm, "bwd_ms": bm, "fwd_tflops": fl / fm / 1e9, "bwd_tflops": 2.5 * fl / bm / 1e9}
        except Exception as e:  # backend not available for this shape / arch
            res[name] = {"unavailable": f"{type(e).__name__}: {str(e)[:160]}"}
        box.pop("y", None)
    return res


def run_ours(args, world, rank, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2605_28691_b200 import GridShape, kernels
    from paper_2605_28691_b200.anyres import pad_grid
    from paper_2605_28691_b200.block import SkiparseBlock, plan_parallel_3d
    from paper_2605_28691_b200.ssp import CommLog

    T, H, W, k, heads, d, desc = CONFIGS[args.config]
    k2 = k * k
    C = heads * d
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    group = uly_group = None
    g = GridShape(T, H, W, k)
    pgrid = pad_grid(g).padded
    # N <= k^2: SSP over N ranks; N > k^2: SSP (k^2) x Ulysses (N/k^2) on one latent (the paper's
    # 8-GPU setting), or SSP x data parallel when heads / txh do not divide
    ssp_n, uly_n, dp = plan_parallel_3d(world, k, heads, pgrid.t * pgrid.h // k2)
    if uly_n > 1:
        s_idx, u_idx = rank // uly_n, rank % uly_n
        ssp_groups = [dist.new_group([s * uly_n + u for s in range(ssp_n)]) for u in range(uly_n)]
        uly_groups = [dist.new_group([s * uly_n + u for u in range(uly_n)]) for s in range(ssp_n)]
        group, uly_group = ssp_groups[u_idx], uly_groups[s_idx]
    elif dp > 1:
        groups = [dist.new_group(list(range(i * ssp_n, (i + 1) * ssp_n))) for i in range(dp)]
        group = groups[rank // ssp_n]
    log = CommLog()
    # the SSP switch: pack (K4) -> one NCCL all-to-all -> unpack, overlapped with attention in
    # head chunks.  The one-pull peer-memory switch (K7, --transport p2p) stays opt-in: its device
    # barrier has not yet run across real GPUs, and CUDA-IPC handles only open on one host.
    transport = args.transport
    if transport == "auto":
        transport = "native"
    blk = SkiparseBlock(g, heads, C, batch=1, group=group if world > 1 else None, log=log,
                        device=dev, ulysses_group=uly_group, transport=transport)
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    # one GPU: the step of SURVEY.md sec. 8d -- the unpadded original latent in, the block (orig ->
    # TSA -> GSA -> orig) out; N GPUs: this rank's token-wise shard in and out (SSP steady state)
    orig_step = world == 1 and blk._scatter is not None and not args.tsa_step
    if orig_step:
        shape = (1, T * H * W, C)
        fn = blk.forward_original
    else:
        shape = (blk.local_rows, blk.L_local, C)
        fn = blk
    x = torch.randn(shape, generator=gen, device=dev).to(torch.bfloat16)
    gy = torch.randn(shape, generator=gen, device=dev).to(torch.bfloat16)
    x.requires_grad_(True)

    def step(inp):
        y = fn(inp)
        y.backward(gy)
        return y

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        x.grad = None
        step(x)
    torch.cuda.synchronize()
    barrier()

    # ---- CUDA graph of the whole step (fwd + bwd), replayed in the timed region when the step is
    # launch-bound (--graph; "auto" = the cfg1 reference case): the kernels take device pointers,
    # sizes and the current stream only, so the step captures as is.  Per-kernel times then come
    # from one extra eager pass after the timed region.
    use_graph = (args.graph == "on") or (args.graph == "auto" and args.config == "cfg1" and world == 1)
    graph = None
    if use_graph:
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(2):
                x.grad = None
                step(x)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        x.grad = None
        with torch.cuda.graph(graph):
            step(x)
        graph.replay()
        torch.cuda.synchronize()

    # ---- device-resident timed region
    kernels.STATS.reset(timing=graph is None)
    log.events.clear()
    log.timed.clear()
    log.timing = world > 1
    stream = torch.cuda.current_stream()
    gpu_index = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local_rank)).split(",")[local_rank]) \
        if "CUDA_VISIBLE_DEVICES" in os.environ else local_rank
    with ClockSampler(gpu_index) as clk:
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            if graph is not None:
                graph.replay()
            else:
                x.grad = None
                step(x)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = e0.elapsed_time(e1)
    if graph is not None:
        # the launches and kernel times of the replayed steps, from an eager pass of the same step
        kernels.STATS.reset(timing=True)
        for _ in range(args.steps):
            x.grad = None
            step(x)
        torch.cuda.synchronize()
    launches = kernels.STATS.launches
    per_kernel = kernels.STATS.elapsed_ms()
    comm = _comm_summary(log, args.steps) if world > 1 else None   # the timed steps only
    if comm is not None:
        comm["ssp_transport"] = transport
        # device time of the SSP all-to-alls (summed over chunks, per step); they run on a
        # communication stream under the attention of the next head chunk, so this is not the
        # exposed time
        comm["all_to_all_device_ms_per_step"] = {k_: v / args.steps for k_, v in log.collective_ms().items()}
    log.timing = False
    kernels.STATS.reset(timing=False)
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    ms_step = ms / args.steps
    tokens_step = dp * T * H * W
    value = tokens_step / (ms_step / 1000.0)

    # ---- end-to-end through the public API: every step's input is copied host->device from
    # pinned memory and its output y (the block's result, what the reference API returns) and the
    # loss <y, gy> are copied back, all inside the timed region.  Copies run on two copy streams
    # (double buffers) so step i+1's input upload and step i's output download overlap compute, as
    # a training / serving loop's data feed would.
    host_x = torch.empty(tuple(x.shape), dtype=torch.bfloat16, pin_memory=True)
    host_x.copy_(x.detach().cpu())
    host_y = [torch.empty(tuple(x.shape), dtype=torch.bfloat16, pin_memory=True) for _ in range(2)]
    host_loss = torch.empty((args.steps,), dtype=torch.float32, pin_memory=True)
    bufs = [torch.empty_like(x.detach()) for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    y_done = [torch.cuda.Event() for _ in range(2)]
    copy_stream = torch.cuda.Stream(device=dev)
    d2h_stream = torch.cuda.Stream(device=dev)
    ys = [None, None]
    barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    copy_stream.wait_stream(stream)
    d2h_stream.wait_stream(stream)
    with torch.cuda.stream(copy_stream):
        bufs[0].copy_(host_x, non_blocking=True)
        ready[0].record(copy_stream)
    for i in range(args.steps):
        b = i % 2
        if i + 1 < args.steps:
            nb = (i + 1) % 2
            with torch.cuda.stream(copy_stream):
                if i >= 1:
                    copy_stream.wait_event(consumed[nb])
                bufs[nb].copy_(host_x, non_blocking=True)
                ready[nb].record(copy_stream)
        stream.wait_event(ready[b])
        xin = bufs[b].detach().requires_grad_(True)
        y = fn(xin)
        ys[b] = y.detach()
        ys[b].record_stream(d2h_stream)       # y's memory is not reused before its download ends
        y_done[b].record(stream)
        with torch.cuda.stream(d2h_stream):
            d2h_stream.wait_event(y_done[b])
            host_y[b].copy_(ys[b], non_blocking=True)
        # the step's scalar loss <y, gy> as one dot-product pass (fp32 accumulate)
        loss = torch.dot(y.detach().reshape(-1), gy.reshape(-1)).float()
        y.backward(gy)
        consumed[b].record(stream)
        host_loss[i:i + 1].copy_(loss.detach().view(1), non_blocking=True)
    stream.wait_stream(d2h_stream)
    f1.record(stream)
    torch.cuda.synchronize()
    barrier()
    t = torch.tensor([f0.elapsed_time(f1)], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms_step = t.item() / args.steps
    e2e_value = tokens_step / (e2e_ms_step / 1000.0)
    io_bytes = host_x.numel() * host_x.element_size()

    if rank != 0:
        return
    burst, sustained, hbm, peak_src = _peaks()
    fl = blk.flops()
    n_sub_local = blk.local_rows
    att_fwd_padded = 4 * n_sub_local * blk.L * blk.L * d * heads
    # executed (= useful, real-token) FLOPs per launch, averaged over the TSA and GSA launches:
    # with padding compaction the kernels run exactly the real-token interactions
    att_fwd_launch = fl["attention_fwd_executed"] / 2
    kern = {}
    for name, v in per_kernel.items():
        kern[name] = {"launches": len(v), "mean_ms": statistics.mean(v), "total_ms": sum(v)}
    bwd = kern.get("attn_bwd")
    fwd = kern.get("attn_fwd")
    ach_bwd = 2.5 * att_fwd_launch / (bwd["mean_ms"] / 1e3) / 1e12 if bwd else None
    ach_fwd = att_fwd_launch / (fwd["mean_ms"] / 1e3) / 1e12 if fwd else None
    total_tflops = world * fl["total"] / (ms_step / 1e3) / 1e12 / world  # per GPU
    roof = {"bound": "tensor", "kernel": "osp_attn_bwd (K3: delta prep + tcgen05 main + dq finalize)",
            "achieved": ach_bwd, "peak": sustained, "unit": "TFLOP/s",
            "frac": ach_bwd / sustained if ach_bwd else None,
            "traffic": None, "peak_source": f"{peak_src} bf16 sustained (MEASURED_PEAKS.json)",
            "algorithmic_flops_per_launch": 2.5 * att_fwd_launch,
            "flops_basis": "executed = useful real-token FLOPs (padding compacted away); the "
                           "padded-grid count of flop_report is padded_grid_flops_per_launch",
            "padded_grid_flops_per_launch": 2.5 * att_fwd_padded,
            "fwd_kernel": {"kernel": "osp_attn_fwd (K2)", "achieved": ach_fwd,
                           "frac": ach_fwd / sustained if ach_fwd else None,
                           "algorithmic_flops_per_launch": att_fwd_launch,
                           "padded_grid_flops_per_launch": att_fwd_padded},
            "block_tensor_tflops_per_gpu": total_tflops,
            "block_frac_of_peak": total_tflops / sustained,
            "block_frac_of_burst_peak": total_tflops / burst}
    traffic, tsrc = _ncu_traffic("attn_bwd_v2") if (args.config == "cfg3" and world == 1) else (None, None)
    roof["traffic"] = traffic
    roof["traffic_source"] = tsrc
    ftraffic, _ = _ncu_traffic("attn_fwd") if (args.config == "cfg3" and world == 1) else (None, None)
    roof["fwd_kernel"]["traffic"] = ftraffic
    k1 = kern.get("gather_rows")
    if k1 and orig_step:
        # K1 row moves of the orig step: the unpadded latent -> compact TSA rows (forward) and its
        # adjoint (backward); bytes = rows read + rows written, one C-wide bf16 row each
        tin = blk._orig_plans()[0]
        row_b = C * 2
        by = [((tin.src >= 0).sum().item() + tin.src.numel()) * row_b,
              ((tin.inv >= 0).sum().item() + tin.inv.numel()) * row_b]
        alg = sum(by) / 2
        k1t, k1src = _ncu_traffic("permute_rows_cfg3") if (args.config == "cfg3") else (None, None)
        roof["k1"] = {"kernel": "osp_gather_rows (K1 permute_rows_warp)", "bound": "hbm",
                      "achieved": alg / (k1["mean_ms"] / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                      "frac": alg / (k1["mean_ms"] / 1e3) / 1e9 / hbm,
                      "algorithmic_bytes_per_launch": alg, "launches_per_step": k1["launches"] / args.steps,
                      "traffic": k1t, "traffic_source": k1src}
    share = {n: v["total_ms"] / ms for n, v in kern.items()}
    step_desc = ("orig -> TSA app -> GSA app -> orig (SURVEY.md sec. 8d): one K1 gather of the unpadded "
                 "latent into compact TSA rows; application 1's epilogue stores into compact GSA rows, "
                 "application 2's into the unpadded latent; backward mirrors it (K3 Delta pre-pass "
                 "gathers dO, one K1 move returns dx); each application = fixed QKV projection (cuBLAS) "
                 "+ tcgen05 attention; bwd = input grad") if orig_step else \
        "TSA shard in -> TSA app + switch + GSA app + switch -> TSA shard out; bwd = input grad"
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong" if dp == 1 else "mixed",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (torch.randn, bf16)",
            "config": {"workload": args.config, "description": desc, "grid": [T, H, W], "k": k,
                       "heads": heads, "head_dim": d, "global_batch": dp,
                       "parallelism": (f"ssp{ssp_n}" + (f"xulysses{uly_n}" if uly_n > 1 else "")
                                       + (f"xdp{dp}" if dp > 1 else "")),
                       "padded_grid": [blk.grid.t, blk.grid.h, blk.grid.w], "subseq_len": blk.L,
                       "l2": ("inputs > 126 MB L2 (no flush needed)" if T * H * W * C * 2 > 126e6 else
                              "input x < L2, but each step's q|k|v, O and dO (> L2) evict it: no flush"
                              if T * H * W * 3 * C * 2 > 126e6 else
                              "whole step < L2: the launch-bound reference case, no flush"),
                       "cuda_graph": graph is not None,
                       "block": step_desc},
            "e2e": {"value": e2e_value, "unit": "tokens/s",
                    "h2d_bytes_per_step": io_bytes,
                    "d2h_bytes_per_step": io_bytes + 4, "ms_per_step": e2e_ms_step,
                    "what": "x uploaded from pinned host memory, y and the loss downloaded, every step"},
            "gpu_launches": launches,
            "roofline": roof,
            "flops_per_step_per_gpu": fl,
            "kernel_ms": kern, "kernel_share_of_step": share,
            # SURVEY.md sec. 8d's targets count attention FLOPs only; the step also runs the
            # reference's projection GEMMs (cuBLAS), so this is the step's tokens/s over the time of
            # this library's attention kernels alone (K2 + K3 incl. prep / finalize), for comparison
            "attention_only_tokens_per_s": (tokens_step / (sum(v["total_ms"] for n, v in kern.items()
                                                               if n.startswith("attn")) / args.steps / 1e3)
                                            if any(n.startswith("attn") for n in kern) else None),
            "comm": comm,
            "clocks": clk.summary()}
    par = _parity_summary(args.config, orig_step)
    if par:
        line["parity"] = par
    if world == 1 and not args.no_comparator:
        line["comparator"] = sdpa_comparator(heads, d, blk.L, blk.local_rows, dev)
    if world == 1 and not args.no_cpu:
        cb = cpu_oracle_rate(args.config, 1, (args.cpu_sample, 2 * args.cpu_sample, 4 * args.cpu_sample))
        line["cpu_baseline"] = {k_: cb[k_] for k_ in ("value", "unit", "cores", "sample")}
        line["cpu_baseline"]["kind"] = "port"
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=2048,
                    help="shortest CPU-oracle slice length (the fit also times 2x and 4x it)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-comparator", action="store_true", help="skip the same-box SDPA timings")
    ap.add_argument("--tsa-step", action="store_true",
                    help="N=1: time the token-wise steady-state block instead of the orig->orig step")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay the step as one CUDA graph in the timed region (auto: cfg1 only)")
    ap.add_argument("--transport", default="auto", choices=["auto", "native", "hif8", "p2p"],
                    help="SSP switch transport for N > 1 (auto = native NCCL; p2p = K7 peer pull, one host)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        if os.environ.get("OSP_BENCH_HOST_COLLECTIVES") == "1":
            # logic check of the N-rank path on a box with fewer GPUs: all ranks share the visible
            # GPUs and every collective is staged through the host (gloo), so no rank's kernel
            # waits on another's.  Never used for a reported number.
            local_rank %= torch.cuda.device_count()
            torch.cuda.set_device(local_rank)
            dist.init_process_group("gloo")
            _host_stage_collectives(dist)
            os.environ["OSP_PEER_HOST_SYNC"] = "1"
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, world, rank, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            from paper_2605_28691_b200.peer import close_arenas
            close_arenas()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
