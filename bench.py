"""Headline benchmark: tokens/s for one 131,072-token sequence through the
LLaMA-3.2-1B-shaped ARMT (segment 1024, 128 memory tokens), bf16, on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--schedule diagonal|sequential]
                    [--segments S] [--impl reference]

One "step" = one full forward of the sequence (S+L-1 diagonal steps, every
cell's retrieve/block/update plus the LM head for all tokens), replayed from
a single CUDA graph with a fresh memory state; inputs (token ids, weights) are
resident in HBM and far larger than L2 (3.3 GB of weights), so no flush is
needed. ``e2e`` repeats the measurement through the public scoring API
(``Session.nll``) with the token ids copied in from pinned host memory and
the per-token NLL copied back every step.

N > 1 (torchrun): layers are sharded contiguously across ranks (pipeline
over the wavefront); the same 131,072 tokens are processed (strong scaling).
``--impl reference`` times the CPU oracle port of the reference
(oracle/armt_oracle.py) on the host cores, rank 0 only.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

C2 = dict(n_layers=16, d_model=2048, n_heads=32, d_ff=8192, segment_size=1024, num_mem_tokens=128,
          d_mem=64, vocab_size=128256)
C5 = dict(n_layers=32, d_model=4096, n_heads=32, d_ff=14336, segment_size=1024, num_mem_tokens=128,
          d_mem=64, vocab_size=128256)
N_TOKENS = 131072
# BASELINE.json configs as (model kwargs, tokens, description)
CONFIGS = {
    "c2": (C2, 131072, "C2: LLaMA-3.2-1B-shaped ARMT (L16 d2048 H32 ff8192), seg 1024, 128 mem tokens"),
    "c3-512": (dict(C2, segment_size=512), 131072, "C3: C2 with segment 512"),
    "c3-2048": (dict(C2, segment_size=2048), 131072, "C3: C2 with segment 2048"),
    "c3-32k": (C2, 32768, "C3: C2 at 32,768 tokens"),
    "c4": (C2, 1048576, "C4: C2 model, 1,048,576-token sequence"),
    "c5": (C5, 131072, "C5: LLaMA-3.1-8B-shaped ARMT (L32 d4096 H32 ff14336), seg 1024, 128 mem tokens"),
}
EPS_C5 = 10000.0      # width 4096 needs a larger guard to stay finite over 128 segments (1000 diverges)
EPS_ASSOC = 100.0     # SURVEY Appendix B conditioning: finite over all 128 C2 segments (scripts/c2_horizon.py)
METRIC = "tokens/sec for one 131k-token seq, LLaMA-1B ARMT seg1024, 1/2/4/8 B200"


def cell_flops(cfg) -> float:
    """Algorithmic FLOPs per (segment, layer) cell, SURVEY §8(d)."""
    T, d, f, M, dm = cfg.tokens_per_segment, cfg.d_model, cfg.d_ff, cfg.num_mem_tokens, cfg.d_mem
    dphi = cfg.d_phi
    lin = 2 * T * (4 * d * d + 3 * d * f)
    attn = 4 * d * T * (T + 1) / 2
    retr = 2 * T * d * dm + 2 * T * dphi * d + 2 * T * dphi
    upd = 2 * M * d * (dm + d + 1) + M * (4 * d * dphi + 6 * dphi)
    return lin + attn + retr + upd


def run_flops(cfg, n_segments: int) -> float:
    return n_segments * cfg.n_layers * cell_flops(cfg) + 2 * n_segments * cfg.segment_size * cfg.d_model * cfg.vocab_size


def load_traffic(key: str = "gemm_gu"):
    """DRAM bytes per gate/up launch from the committed ncu --set full capture
    (profiles/*_kernels.json, written by scripts/profile_summary.py); ``key`` names
    the capture (gemm_gu = 16 members, gemm_gu_g8 = 8 members, the dual-stream width)."""
    import glob
    best = None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_kernels.json"))):
        try:
            m = json.load(open(path)).get(key)
        except (OSError, ValueError):
            continue
        if m and "dram_read_bytes" in m:
            best = {"bytes": m["dram_read_bytes"] + m.get("dram_write_bytes", 0), "source": os.path.basename(path)}
    return best


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self):
        sm, mx, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
            try:
                power.append(float(parts[6]))
            except (IndexError, ValueError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w": statistics.median(power) if power else None}


def make_weights(cfg, init: str = "reference"):
    """Reference initializer (armt/weights.py:98-138, seed 0), w_v_mem x 1/32.

    ``init="device"`` draws the same distributions (N(0,1)/sqrt(fan_in), unit
    gains) with torch's seeded generator on the GPU: the values differ from
    the reference's PCG64 stream but the architecture/scales are identical;
    used for the 8B-shaped config where a host f64 draw of 9.4 B parameters
    would dominate the run.
    """
    from dataclasses import replace
    from paper_2506_05229_b200 import init_weights
    from paper_2506_05229_b200.weights import GroupedWeights, expected_shapes
    if init == "reference":
        w = init_weights(cfg, dtype=np.float32)
        return replace(w, w_v_mem=w.w_v_mem * np.float32(1.0 / 32))
    import torch
    gen = torch.Generator(device="cuda").manual_seed(cfg.seed)
    shapes = expected_shapes(cfg)
    fan = {"embedding": 1, "mem_embedding": 1, "w_out": cfg.d_ff}
    arrays = {}
    for name, shape in shapes.items():
        if name in ("attn_gain", "mlp_gain"):
            arrays[name] = torch.ones(shape, device="cuda")
            continue
        t = torch.randn(shape, generator=gen, device="cuda")
        if name != "embedding" and name != "mem_embedding":
            t *= 1.0 / np.sqrt(fan.get(name, cfg.d_model))
        if name == "w_v_mem":
            t *= 1.0 / 32
        arrays[name] = t
    return GroupedWeights(config=cfg, **arrays)


def cpu_oracle_rate(w, cfg, n_segments: int, budget_s: float = 12.0, max_cells: int = 16,
                    n_layers: int | None = None):
    """Oracle (numpy/BLAS f32, all host threads) on full-width cells + one LM head,
    extrapolated over the schedule: S*L cells + S heads (``n_layers``: the real L
    when ``w`` holds only a sample of the layers; every cell costs the same)."""
    import armt_oracle as O
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [os.cpu_count()])
    except Exception:
        threads = os.cpu_count()
    orc = O.Oracle(w, cfg, np.float32, eps_assoc=EPS_ASSOC)
    rng = np.random.default_rng(0)
    state = O.OracleState.fresh(cfg, np.float32)
    x = orc.embed(rng.integers(0, cfg.vocab_size, cfg.segment_size))
    x = orc.cell(state, 0, x)  # warm caches / BLAS pools
    cells, t0 = 0, time.perf_counter()
    while cells < max_cells and (cells < 2 or time.perf_counter() - t0 < budget_s):
        x = orc.cell(state, cells % cfg.n_layers, x)
        cells += 1
    t_cell = (time.perf_counter() - t0) / cells
    t1 = time.perf_counter()
    orc.unembed(x)
    t_lm = time.perf_counter() - t1
    total = n_segments * (n_layers or cfg.n_layers) * t_cell + n_segments * t_lm
    return {"t_cell": t_cell, "t_lm": t_lm, "cells": cells, "total_s": total, "threads": threads,
            "sample_s": cells * t_cell + t_lm}


# ---------------------------------------------------------------------------- reference arm
REF_PATH = os.path.join(ROOT, "baseline", "_ref")   # pip install --target of /root/reference/pkg (git-ignored)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ReferenceCells:
    """The UNMODIFIED reference package (baseline/_ref, numba kernels) on this
    host's cores, through its own public API: one diagonal step of ``G`` members
    at the model's full width (retrieve_stack -> forward_stack -> update_stack
    with WorkerPool(cpu_count), armt/executors.py:196-203) on a short segment,
    plus its own ``gemm`` for ``lm_rows`` LM-head rows at the full vocabulary
    (armt/layers.py:321-323). Numba's loops cost the same for any values, so the
    rates measured here extrapolate by FLOPs to full C2 cells and segments."""

    def __init__(self, model: dict, eps: float, seg: int = 32, lm_rows: int = 4, members: int | None = None):
        if REF_PATH not in sys.path:
            sys.path.insert(0, REF_PATH)
        import armt
        from armt.layers import forward_stack
        from armt.memory import retrieve_stack, update_stack
        self.armt, self.fwd, self.ret, self.upd = armt, forward_stack, retrieve_stack, update_stack
        self.cores = os.cpu_count() or 1
        G = members or min(16, self.cores, model["n_layers"])
        self.cfg = armt.ModelConfig(**dict(model, n_layers=G, segment_size=seg, vocab_size=512),
                                    eps_assoc=eps, seed=0)
        w = armt.init_weights(self.cfg)
        self.p = armt.prepare_weights(w, "f32")
        del w
        self.state = armt.MemoryState.fresh(self.cfg, "f32")
        self.pool = armt.WorkerPool(self.cores)
        rng = np.random.default_rng(0)
        self.x = np.stack([armt.embed_segment(self.p, rng.integers(0, 512, seg), i).data for i in range(G)])
        self.layers = np.arange(G, dtype=np.int64)
        self.G, self.seg, self.lm_rows = G, seg, lm_rows
        self.V = model["vocab_size"]
        self.U = np.random.default_rng(1).standard_normal((model["d_model"], self.V), dtype=np.float32)
        armt.tensor_ops.warmup_kernels(np.float32)

    def step(self):
        """Returns (seconds of the G-member step, seconds of the lm_rows LM head)."""
        t0 = time.perf_counter()
        xr = self.ret(self.state, self.layers, self.x, self.p, self.pool)
        y = self.fwd(self.p, self.layers, xr, self.pool)
        self.upd(self.state, self.layers, y[:, -self.cfg.num_mem_tokens:, :], self.p, self.pool)
        t1 = time.perf_counter()
        self.armt.gemm(np.ascontiguousarray(y[0, :self.lm_rows]), self.U)
        return t1 - t0, time.perf_counter() - t1

    def extrapolate(self, cfg, S: int, t_cells: float, t_lm: float) -> dict:
        """Forward seconds for S segments of ``cfg``: every cell at the measured
        full-group throughput (a lower bound on the reference's diagonal-run time:
        ramp steps with fewer members than cores are slower per cell) + S heads."""
        rate_cells = self.G * cell_flops(self.cfg) / t_cells
        rate_lm = 2.0 * self.lm_rows * cfg.d_model * cfg.vocab_size / t_lm
        t_cell = cell_flops(cfg) / rate_cells
        t_head = 2.0 * cfg.segment_size * cfg.d_model * cfg.vocab_size / rate_lm
        return {"total_s": S * cfg.n_layers * t_cell + S * t_head, "t_cell": t_cell, "t_head": t_head,
                "gflops_cells": rate_cells / 1e9, "gflops_lm": rate_lm / 1e9}

    def describe(self) -> str:
        return (f"reference armt (baseline/_ref, numba f32) on {self.cores} host threads ({cpu_model()}): per step "
                f"one diagonal step of {self.G} full-width cells (segment {self.seg} + "
                f"{self.cfg.num_mem_tokens} memory tokens, WorkerPool({self.cores})) + a {self.lm_rows}-row LM head "
                f"at V={self.V}; extrapolated by FLOPs to full cells/heads, every cell at full-group throughput")


def reference_arm(args, rank, world):
    """``--impl reference``: the reference's own CPU implementation (numba, all host
    threads) on bounded samples of the requested workload; rank 0 only. Falls
    back to the NumPy/BLAS oracle port when baseline/_ref is absent."""
    if rank != 0:
        return 0
    from paper_2506_05229_b200 import ModelConfig
    model, n_cfg, desc = CONFIGS[args.config]
    eps = args.eps if args.eps is not None else (EPS_C5 if args.config == "c5" else EPS_ASSOC)
    cfg = ModelConfig(**model, eps_assoc=eps, seed=0)
    n = args.tokens or n_cfg
    if args.segments is not None:
        n = args.segments * cfg.segment_size
    S = -(-n // cfg.segment_size)
    base = shared_config(args, cfg, n, S, desc)
    try:
        ref = ReferenceCells(model, eps)
    except ImportError as exc:
        ref = None
        why = f"baseline/_ref not importable ({exc}); oracle port instead"
    rates, walls = [], []
    if ref is not None:
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            tc, tl = ref.step()
            walls.append(time.perf_counter() - t0)
            if i >= args.warmup:
                rates.append(n / ref.extrapolate(cfg, S, tc, tl)["total_s"])
        kind, cores, sample = "reference", ref.cores, ref.describe()
    else:
        from dataclasses import replace as _replace
        sample_cfg = _replace(cfg, n_layers=min(2, cfg.n_layers))
        w = make_weights(sample_cfg)
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            r = cpu_oracle_rate(w, sample_cfg, S, budget_s=4.0, max_cells=4, n_layers=cfg.n_layers)
            walls.append(time.perf_counter() - t0)
            if i >= args.warmup:
                rates.append(n / r["total_s"])
        kind, cores, sample = "port", r["threads"], f"{why}: numpy/BLAS f32 cells + 1 LM head, extrapolated"
    value = statistics.mean(rates)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * statistics.mean(walls[args.warmup:]),
            "ms_per_step_note": "measured wall time of one bounded sample step; value extrapolates the "
                                "sample's measured throughput to the whole forward",
            "extrapolated_forward_s": n / value,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded reference init, cli token convention)",
            "config": base,
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": kind, "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def shared_config(args, cfg, n, S, desc) -> dict:
    """The workload identity both arms report (identical dicts for the same flags)."""
    return {"workload": f"{desc}, {n} tokens", "schedule": args.schedule, "segments": S,
            "init": args.init or "reference",
            "eps_assoc": cfg.eps_assoc, "output": "fused NLL (no logits)" if (args.scoring or args.config == "c4")
            else "logits", "l2": "inputs > L2 (3.3 GB bf16 weights, 33.6 GB logits); no flush"}


# ---------------------------------------------------------------------------- device arm
def device_arm(args, rank, world):
    import torch
    from paper_2506_05229_b200 import ModelConfig
    from paper_2506_05229_b200 import _lib
    from paper_2506_05229_b200.engine import prepare_weights
    from paper_2506_05229_b200.executors import Session

    model, n_cfg, desc = CONFIGS[args.config]
    eps = args.eps if args.eps is not None else (EPS_C5 if args.config == "c5" else EPS_ASSOC)
    cfg = ModelConfig(**model, eps_assoc=eps, seed=0)
    n = args.tokens or n_cfg
    if args.segments is not None:
        n = args.segments * cfg.segment_size
    S = -(-n // cfg.segment_size)
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    t_setup = time.time()
    init = args.init or "reference"
    scoring_value = args.scoring or args.config == "c4"
    w = make_weights(cfg, init)
    tokens = np.random.default_rng([0, n]).integers(0, cfg.vocab_size, n, dtype=np.int64)

    if world > 1 or args.force_sharded:
        from paper_2506_05229_b200.sharded import ShardedSession
        sess = ShardedSession(w, cfg, n, rank=rank, world=world, device=dev, schedule=args.schedule,
                              scoring=scoring_value)
    else:
        prep = prepare_weights(w, "bf16", dev)
        if init == "device":
            del w
            torch.cuda.empty_cache()
        sess = Session(prep, n, schedule=args.schedule, scoring=scoring_value)
    sess._load_ids(torch.as_tensor(tokens).to(dev))

    # roofline probe: events around every full-width gate/up GEMM, captured into the graph
    # (dual-stream runner: each engine's full-width launches, on the stream they run on)
    probe_events = []
    engines = getattr(sess.runner, "engines", [sess.runner.engine])
    full_g = max(e.max_members for e in engines)
    probe_g = engines[0].max_members

    def make_probe(e):
        def probe(G, phase, stream=None):
            if G != probe_g:
                return
            st = torch.cuda.ExternalStream(stream) if stream is not None else torch.cuda.current_stream()
            if phase == 0:
                # external=True: event-record nodes that keep timing inside a CUDA graph
                probe_events.append([torch.cuda.Event(enable_timing=True, external=True),
                                     torch.cuda.Event(enable_timing=True, external=True)])
                probe_events[-1][0].record(st)
            else:
                probe_events[-1][1].record(st)
        return probe

    sess.warm_eager()
    sharded = world > 1 or args.force_sharded
    for e in engines:
        e.probe = make_probe(e)   # (sharded path: event-record nodes inside the per-step graphs)
    sess.capture()
    for e in engines:
        e.probe = None
    setup_s = time.time() - t_setup

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        sess.forward()
    torch.cuda.synchronize()
    barrier()
    probe_ms = []
    step_ms = []
    with ClockSampler(dev.index) as clocks:
        for _ in range(args.steps):
            barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sess.forward()
            e1.record()
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            probe_ms.append(sum(a.elapsed_time(b) for a, b in probe_events))
    barrier()
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = n / (ms_per_step / 1e3)

    # end-to-end through the public scoring API: pinned H2D ids + D2H per-token NLL each step.
    # Single GPU: a scoring Session fuses the next-token NLL into the LM-head epilogue
    # (no 33.6 GB logits round trip); the sharded path scores from the last rank's logits.
    launches_per_forward = sess.kernels_per_forward
    if not scoring_value:
        del sess
        torch.cuda.empty_cache()
        if world == 1 and not args.force_sharded:
            sess = Session(prep, n, schedule=args.schedule, scoring=True)
        else:
            from paper_2506_05229_b200.sharded import ShardedSession
            sess = ShardedSession(w, cfg, n, rank=rank, world=world, device=dev, schedule=args.schedule,
                                  scoring=True)
            sess._load_ids(torch.as_tensor(tokens).to(dev))
        sess.warm()
    host_ids = torch.as_tensor(tokens).pin_memory()
    host_nll = torch.empty(n - 1, dtype=torch.float32).pin_memory()
    for _ in range(2):
        out = sess.nll(host_ids.to(dev, non_blocking=True))
        host_nll.copy_(out, non_blocking=True) if out is not None else None
    torch.cuda.synchronize()
    barrier()
    e2e_ms = []
    for _ in range(args.steps):
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = sess.nll(host_ids.to(dev, non_blocking=True))
        if out is not None:
            host_nll.copy_(out, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    e2e_total = sum(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e_total], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = n / (e2e_total / args.steps / 1e3)
    mean_nll = float(host_nll.mean())

    # the reference's own entry point as a drop-in (armt/executors.py:153-226): run_diagonal with
    # host int64 ids, logits returned on the device (return_numpy=False; the numpy copy of 33.6 GB
    # of logits would time PCIe, not the forward). Its first call runs eagerly, the second captures
    # the graph that every later call replays; the clone of the logits is part of each call.
    d_ff_pad = sess.p.d_ff_pad
    ref_api = None
    if world == 1 and not args.force_sharded and args.schedule == "diagonal" and not scoring_value:
        from paper_2506_05229_b200.executors import clear_caches, run_diagonal
        del sess
        sess = None
        torch.cuda.empty_cache()
        toks_np = np.asarray(tokens, dtype=np.int64)
        for _ in range(2):
            run_diagonal(prep, cfg, toks_np, return_numpy=False)
        torch.cuda.synchronize()
        api_ms = []
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out, _ = run_diagonal(prep, cfg, toks_np, return_numpy=False)
            e1.record()
            torch.cuda.synchronize()
            api_ms.append(e0.elapsed_time(e1))
            del out
        ref_api = {"value": n / (statistics.mean(api_ms) / 1e3), "unit": "tokens/s",
                   "h2d_bytes_per_step": int(n * 8), "d2h_bytes_per_step": 0,
                   "api": "run_diagonal(prepared, config, host int64 ids, return_numpy=False): the reference's "
                          "entry point, cached prepared weights, one graph replay + logits clone per call"}
        clear_caches()
        torch.cuda.empty_cache()

    # north-star ratio in the same run: the sequential segment schedule (armt/executors.py:123-150),
    # same kernels (G = 1 lane), same whole-run CUDA-graph policy, same K/W, fresh memory per replay
    seq_value = None
    seq_clock_summary = None
    if args.compare_sequential and world == 1 and not args.force_sharded and args.schedule == "diagonal":
        sess = None
        torch.cuda.empty_cache()
        seq = Session(prep, n, schedule="sequential", scoring=scoring_value)
        seq._load_ids(torch.as_tensor(tokens).to(dev))
        seq.warm()
        for _ in range(args.warmup):
            seq.forward()
        torch.cuda.synchronize()
        seq_ms = []
        with ClockSampler(dev.index) as seq_clocks:
            for _ in range(args.steps):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                seq.forward()
                e1.record()
                torch.cuda.synchronize()
                seq_ms.append(e0.elapsed_time(e1))
        seq_clock_summary = seq_clocks.summary()
        seq_value = n / (statistics.mean(seq_ms) / 1e3)
        del seq
        torch.cuda.empty_cache()

    peaks, peak_kind = load_peaks()
    traffic = (load_traffic("gemm_gu" if probe_g == 16 else f"gemm_gu_g{probe_g}")
               if (args.config == "c2" and full_g == 16) else None)
    gu_bytes = 2.0 * (probe_g * cfg.tokens_per_segment * cfg.d_model + probe_g * 2 * d_ff_pad * cfg.d_model
                      + probe_g * cfg.tokens_per_segment * d_ff_pad)
    # dominant kernel: the grouped tcgen05 GEMM; probed launch = full-width gate/up (SwiGLU epilogue)
    gu_flops = 2.0 * probe_g * cfg.tokens_per_segment * (2 * d_ff_pad) * cfg.d_model
    n_probe = len(probe_events)
    probe_avg_ms = statistics.mean(probe_ms) / max(n_probe, 1)
    achieved = gu_flops / (probe_avg_ms / 1e3) / 1e12 if n_probe else None
    peak = peaks.get("bf16_tflops_sustained") or peaks.get("bf16_tflops")
    step_tflops = run_flops(cfg, S) / (ms_per_step / 1e3) / 1e12

    if rank != 0:
        return 0
    cpu = cpu_port = None
    if world == 1 and not args.no_cpu_baseline and init == "reference":
        # the reference's own numba path (baseline/_ref) on the host cores: one warm-up and one measured step
        try:
            ref = ReferenceCells(model, eps)
            ref.step()
            tc, tl = ref.step()
            ex = ref.extrapolate(cfg, S, tc, tl)
            cpu = {"value": n / ex["total_s"], "unit": "tokens/s", "cores": ref.cores, "kind": "reference",
                   "sample": ref.describe() + f" ({tc + tl:.1f} s measured; {ex['gflops_cells']:.1f} GFLOP/s on cells, "
                             f"{ex['gflops_lm']:.1f} GFLOP/s LM head)", "cpu_model": cpu_model()}
            del ref
        except ImportError:
            pass
        r = cpu_oracle_rate(w, cfg, S, budget_s=8.0)
        cpu_port = {"value": n / r["total_s"], "unit": "tokens/s", "cores": r["threads"], "kind": "port",
                    "sample": f"{r['cells']} full-width C2 cells (retrieve+block+fold) + 1 segment LM head, "
                              f"numpy/BLAS f32 oracle ({r['sample_s']:.1f} s), extrapolated to {S}x{cfg.n_layers} "
                              f"cells + {S} heads"}
        cpu = cpu or cpu_port
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16",
        "data": (f"synthetic: reference seeded init (seed 0, w_v_mem/32, eps_assoc {eps:g}), cli token convention"
                 if init == "reference" else
                 f"synthetic: seeded device init with the reference's scales (w_v_mem/32, eps_assoc {eps:g}), cli tokens"),
        "config": shared_config(args, cfg, n, S, desc),
        "parallelism": f"layer-shard{world}" if world > 1 else "single",
        "timing": "CUDA events around one CUDA-graph replay of the whole forward, max over ranks",
        "whole_step_tflops": step_tflops,
        "whole_step_frac_of_sustained": step_tflops / peaks.get("bf16_tflops_sustained", peak),
        "setup_s": setup_s,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": (achieved / peak) if achieved else None,
                     "traffic": (traffic or {}).get("bytes"),
                     "traffic_note": (f"DRAM bytes per launch (read+write) from {traffic['source']}; algorithmic "
                                      f"operand+output bytes {gu_bytes / 1e9:.3f} GB" if traffic else None),
                     "kernel": f"tcgen05 grouped GEMM, gate/up (SwiGLU epilogue), G={probe_g}, "
                               f"{gu_flops / 1e12:.3f} TFLOP/launch, {n_probe} launches/step",
                     "peak_kind": f"{peak_kind} bf16_tflops_sustained"},
        "cpu_baseline": cpu,
        "cpu_baseline_port": cpu_port if cpu is not cpu_port else None,
        "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": int(n * 8),
                "d2h_bytes_per_step": int((n - 1) * 4),
                "api": "Session(scoring=True).nll: pinned ids in, per-token NLL out (LM-head fused NLL)"
                       if not sharded else "ShardedSession(scoring=True).nll: pinned ids in, per-token NLL out "
                                          "(vocab-parallel fused NLL, all-gathered row partials)",
                "mean_nll": mean_nll},
        "e2e_reference_api": ref_api,
        "sequential_value": seq_value,
        "diag_over_seq": (value / seq_value) if seq_value else None,
        "sequential_clocks": seq_clock_summary,
        "north_star_target": "diagonal >= 1.8x sequential on 1xB200 at C2" if seq_value else None,
        "gpu_launches": int(launches_per_forward * args.steps),
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--schedule", default="diagonal", choices=["diagonal", "sequential"])
    ap.add_argument("--segments", type=int, default=None, help="override S (profiling runs)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--tokens", type=int, default=None, help="override the sequence length")
    ap.add_argument("--init", default=None, choices=["reference", "device"])
    ap.add_argument("--eps", type=float, default=None, help="eps_assoc override (fixture conditioning)")
    ap.add_argument("--force-sharded", action="store_true",
                    help="use the layer-sharded session even at world size 1 (plumbing check)")
    ap.add_argument("--no-sequential", dest="compare_sequential", action="store_false",
                    help="skip timing the sequential schedule (north-star diag/seq ratio)")
    ap.add_argument("--scoring", action="store_true",
                    help="time the fused-NLL forward (no logits) for the value too (implied for c4)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    if world > 1:
        import torch
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
        # ARMT_DIST_BACKEND=gloo: plumbing runs with several ranks on one GPU (host-staged P2P)
        torch.distributed.init_process_group(os.environ.get("ARMT_DIST_BACKEND", "nccl"))
    try:
        return device_arm(args, rank, world)
    finally:
        if world > 1:
            import torch
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
