"""Per-kernel timing of the C2 hot ops at a given member count (CUDA events),
for ncu captures and kernel iteration.

    python scripts/kernel_bench.py [--G 16] [--ops gu,down,qkv,o,attn,fold,lm] [--iters 20]

Prints one JSON line per op: avg us/launch, achieved TFLOP/s (GEMMs/attention)
or GB/s (fold), fraction of MEASURED_PEAKS.
"""

import argparse
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if "--prof" in sys.argv:
    os.environ["ARMT_GEMM_PROF"] = "1"   # read once by the library
sys.path.insert(0, ROOT)
from paper_2506_05229_b200 import _lib  # noqa: E402
from paper_2506_05229_b200._lib import BF16, F32  # noqa: E402

LIB = _lib.load()
T, d, F, H, dh, M, dm, V, L = 1152, 2048, 8192, 32, 64, 128, 64, 128256, 16


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        return {"bf16_tflops_sustained": 1400.0, "bf16_tflops": 1590.0, "hbm_gbs": 6650.0}


def timeit(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / iters  # us


def gemm(G, Mr, N, K, epi=_lib.EPI_STORE, c_dtype=BF16, **kw):
    A = torch.randn(G, Mr, K, device="cuda").bfloat16()
    B = (torch.randn(L if G <= L else G, N, K, device="cuda") * 0.02).bfloat16()
    ncol = N // 2 if epi == _lib.EPI_SWIGLU else N
    C = torch.zeros(G, Mr, ncol, device="cuda", dtype=torch.float32 if c_dtype == F32 else torch.bfloat16)
    a = _lib.ArmtGemmArgs()
    a.G, a.M, a.N, a.K, a.ab_dtype = G, Mr, N, K, BF16
    a.A, a.lda, a.a_stride = A.data_ptr(), K, Mr * K
    a.B, a.ldb, a.b_stride = B.data_ptr(), K, N * K
    a.C, a.ldc, a.c_stride, a.c_dtype = C.data_ptr(), ncol, Mr * ncol, c_dtype
    a.epilogue = epi
    keep = [A, B, C]
    if epi in (_lib.EPI_RESIDUAL, _lib.EPI_RETRIEVE):
        # as in the step: in-place f32 stream + bf16 copy + per-64-column sum-of-squares partials
        a.R, a.ldr, a.r_stride = C.data_ptr(), ncol, Mr * ncol
        C2 = torch.zeros(G, Mr, ncol, device="cuda", dtype=torch.bfloat16)
        ssq = torch.zeros(G, Mr, (ncol + 63) // 64, device="cuda")
        a.C2, a.ldc2, a.c2_stride = C2.data_ptr(), ncol, Mr * ncol
        a.ssq_out, a.ssq_stride, a.ssq_np = ssq.data_ptr(), Mr * ssq.shape[2], ssq.shape[2]
        keep += [C2, ssq]
    if epi == _lib.EPI_RETRIEVE:
        den = torch.ones(G, Mr, device="cuda")
        a.den, a.den_stride, a.eps = den.data_ptr(), Mr, 1e-6
        keep.append(den)
    if epi == _lib.EPI_SWIGLU:
        a.swiglu_block = 128
    if epi == _lib.EPI_ROPE:
        inv = 10000.0 ** (-np.arange(0, dh, 2) / dh)
        ang = np.arange(Mr)[:, None] * inv[None]
        cs = torch.tensor(np.cos(ang).T.copy(), dtype=torch.float32, device="cuda")
        sn = torch.tensor(np.sin(ang).T.copy(), dtype=torch.float32, device="cuda")
        keep += [cs, sn]
        a.rope_cos, a.rope_sin, a.head_dim, a.rope_cols = cs.data_ptr(), sn.data_ptr(), dh, 2 * d
    for g in range(G):
        a.a_slot[g] = g
        a.b_index[g] = g % B.shape[0]
        a.c_slot[g] = g
    s = torch.cuda.current_stream().cuda_stream
    return (lambda: _lib.check(LIB.armt_gemm(a, s), "gemm")), 2.0 * G * Mr * N * K, keep


def gemm_specs(G, rows=None):
    R = rows or T
    return {"gu": (G, R, 2 * F, d, _lib.EPI_SWIGLU, BF16), "down": (G, R, d, F, _lib.EPI_RESIDUAL, F32),
            "qkv": (G, R, 3 * d, d, _lib.EPI_ROPE, BF16), "o": (G, R, d, d, _lib.EPI_RESIDUAL, F32),
            "kvb": (G, M, 2128, d, _lib.EPI_STORE, F32), "num": (G, R, d, 384, _lib.EPI_RETRIEVE, F32),
            "lm": (1, 1024, V, d, _lib.EPI_STORE, BF16)}


def cublas_op(G, Mr, N, K, epi, c_dtype):
    """The same grouped GEMM through cuBLAS (torch.bmm, one weight per member),
    GEMM alone and with the epilogue as separate torch ops - the unfused
    library baseline the fused kernel replaces."""
    A = torch.randn(G, Mr, K, device="cuda").bfloat16()
    B = (torch.randn(G, N, K, device="cuda") * 0.02).bfloat16()
    Bt = B.transpose(1, 2)
    C = torch.empty(G, Mr, N, device="cuda", dtype=torch.bfloat16)
    gemm_only = lambda: torch.bmm(A, Bt, out=C)
    ncol = N // 2 if epi == _lib.EPI_SWIGLU else N
    R = torch.zeros(G, Mr, ncol, device="cuda")
    R16 = torch.empty(G, Mr, ncol, device="cuda", dtype=torch.bfloat16)
    den = torch.ones(G, Mr, 1, device="cuda")
    cs = torch.rand(Mr, ncol // 2, device="cuda")

    def full():
        torch.bmm(A, Bt, out=C)
        if epi == _lib.EPI_SWIGLU:
            g, u = C.chunk(2, dim=-1)
            torch.mul(torch.nn.functional.silu(g), u, out=R16)
        elif epi in (_lib.EPI_RESIDUAL, _lib.EPI_RETRIEVE):
            R.add_(C.float() / den if epi == _lib.EPI_RETRIEVE else C.float())
            R16.copy_(R)
            R.view(G, Mr, -1, 64).pow(2).sum(-1)
        elif epi == _lib.EPI_ROPE:
            x = C.float().view(G, Mr, ncol // 2, 2)
            torch.stack((x[..., 0] * cs - x[..., 1] * cs, x[..., 0] * cs + x[..., 1] * cs), -1).bfloat16()
    return gemm_only, full, [A, B, C, R, R16, den, cs]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--G", type=int, default=16)
    ap.add_argument("--ops", default="gu,down,qkv,o,kvb,num,attn,fold,foldtc,lm")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--flags", default=None, help="A/B: comma list of values of env var --env, interleaved")
    ap.add_argument("--env", default="ARMT_GEMM_PAIR")
    ap.add_argument("--rows", type=int, default=None, help="rows per member (default T)")
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--prof", action="store_true", help="GEMM wait-cycle counters (ARMT_GEMM_PROF)")
    ap.add_argument("--cublas", action="store_true", help="also time each GEMM op through cuBLAS (torch.bmm)")
    args = ap.parse_args()
    if args.flags:
        for rep in range(args.repeat):
            for fl in args.flags.split(","):
                os.environ[args.env] = fl
                for op in args.ops.split(","):
                    spec = gemm_specs(args.G, args.rows)[op]
                    fn, flops, keep = gemm(*spec)
                    us = timeit(fn, args.iters)
                    print(json.dumps({"op": op, args.env: fl, "rep": rep, "us": round(us, 1),
                                      "tflops": round(flops / us / 1e6, 1)}), flush=True)
                    del keep
        return
    G = args.G
    pk = peaks()
    for op in args.ops.split(","):
        if op in ("gu", "down", "qkv", "o", "kvb", "num", "lm"):
            spec = gemm_specs(G)[op]
            fn, flops, keep = gemm(*spec)
            us = timeit(fn, args.iters)
            tf = flops / us / 1e6
            rec = {"op": op, "G": spec[0], "us": us, "tflops": tf, "frac_sustained": tf / pk["bf16_tflops_sustained"]}
            if args.prof:
                import ctypes
                buf = (ctypes.c_ulonglong * 8)()
                LIB.armt_gemm_prof(buf, 1)
                fn()
                torch.cuda.synchronize()
                LIB.armt_gemm_prof(buf, 1)
                tot = max(buf[2], 1)
                rec.update(mma_wait_full=buf[0] / tot, mma_wait_acc=buf[1] / tot, prod_wait_empty=buf[3] / tot,
                           tiles=buf[4], epi_wait_full_per_tile=buf[5] / max(buf[4], 1) / 8,
                           mma_cycles_per_cta=tot / min(148, buf[4]))
            if args.cublas:
                del keep
                g_only, full, keep = cublas_op(*spec)
                us_g, us_f = timeit(g_only, args.iters), timeit(full, args.iters)
                rec.update(cublas_gemm_us=us_g, cublas_gemm_tflops=flops / us_g / 1e6, cublas_unfused_us=us_f,
                           speedup_vs_cublas_gemm=us_g / us, speedup_vs_cublas_unfused=us_f / us)
            print(json.dumps(rec), flush=True)
        elif op == "attn":
            qkv = torch.randn(G, T, 3 * d, device="cuda").bfloat16()
            ctx = torch.empty(G, T, d, device="cuda", dtype=torch.bfloat16)
            s = torch.cuda.current_stream().cuda_stream
            fn = lambda: _lib.check(LIB.armt_attention(G, qkv.data_ptr(), 3 * d, T * 3 * d, ctx.data_ptr(), d, T * d,
                                                       BF16, T, H, dh, 1 / math.sqrt(dh), s), "attn")
            us = timeit(fn, args.iters)
            flops = G * 4 * d * T * (T + 1) / 2
            rec = {"op": "attn", "G": G, "us": us, "tflops": flops / us / 1e6,
                   "frac_sustained": flops / us / 1e6 / pk["bf16_tflops_sustained"]}
            if args.cublas:
                # library baseline: torch SDPA (flash / cuDNN backends) on the same causal
                # problem, q/k/v already split into (G, H, T, dh) - the layout work is not timed
                q, k, v = (t.view(G, T, H, dh).transpose(1, 2).contiguous() for t in qkv.split(d, dim=-1))
                sdpa = lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
                us_s = timeit(sdpa, args.iters)
                rec.update(sdpa_us=us_s, sdpa_tflops=flops / us_s / 1e6, speedup_vs_sdpa=us_s / us)
            print(json.dumps(rec), flush=True)
        elif op == "foldtc":
            dphi, P = 6 * dm, 6 * dm
            A = torch.randn(L, d, dphi, device="cuda") * 0.01
            z = torch.rand(L, dphi, device="cuda") * 10
            nk = 2128
            kvb = torch.randn(G, M, nk, device="cuda")
            nb = LIB.armt_memop_rows(d, M)
            memop = torch.zeros(L, nb, 2 * P, device="cuda", dtype=torch.bfloat16)
            ws = torch.zeros(LIB.armt_fold_tc_workspace_bytes(G, M, d, dphi) // 4 + 1, device="cuda")
            mem = _lib.members(list(range(G)), list(range(G)))
            s = torch.cuda.current_stream().cuda_stream
            fn = lambda: _lib.check(LIB.armt_mem_fold_tc(mem, kvb.data_ptr(), nk, M * nk, 0, d, d + dm, A.data_ptr(),
                                                         z.data_ptr(), memop.data_ptr(), d, M, dm, 3, 100.0,
                                                         ws.data_ptr(), s), "foldtc")
            us = timeit(fn, args.iters)
            byts = G * (2 * d * dphi * 4 + M * nk * 4)
            print(json.dumps({"op": "foldtc", "G": G, "us": us, "GBps": byts / us / 1e3,
                              "frac_hbm": byts / us / 1e3 / pk["hbm_gbs"]}), flush=True)
        elif op == "fold":
            dphi = 6 * dm
            A = torch.randn(L, d, dphi, device="cuda") * 0.01
            z = torch.rand(L, dphi, device="cuda") * 10
            nk = 2128
            kvb = torch.randn(G, M, nk, device="cuda")
            ws = torch.empty(LIB.armt_fold_workspace_bytes(G, M, dphi) // 4 + 1, device="cuda")
            mem = _lib.members(list(range(G)), list(range(G)))
            s = torch.cuda.current_stream().cuda_stream
            fn = lambda: _lib.check(LIB.armt_mem_fold(mem, kvb.data_ptr(), nk, M * nk, 0, d, d + dm, A.data_ptr(),
                                                      z.data_ptr(), None, 0, d, M, dm, 3, 10.0, ws.data_ptr(), s), "fold")
            us = timeit(fn, args.iters)
            byts = G * (2 * d * dphi * 4 + M * nk * 4)
            fl = G * M * d * dphi * 4
            print(json.dumps({"op": "fold", "G": G, "us": us, "GBps": byts / us / 1e3, "fp32_tflops": fl / us / 1e6,
                              "frac_hbm": byts / us / 1e3 / pk["hbm_gbs"]}), flush=True)


if __name__ == "__main__":
    main()
