"""Kernel-level numerics on the B200 (``-m gpu``).

Each kernel is called through the C-ABI (``armt_*``) and compared with a
plain PyTorch fp32/fp64 reference of the same op on the same inputs:
bf16-operand GEMMs against fp32 matmul of the bf16-rounded operands, f32
SIMT GEMMs against fp64, attention against an explicit softmax, the memory
fold against the oracle's in-order fold.
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on CPU hosts
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2506_05229_b200 import _lib  # noqa: E402
from paper_2506_05229_b200._lib import BF16, F32  # noqa: E402

DEV = torch.device("cuda")
LIB = _lib.load()


def stream():
    return torch.cuda.current_stream().cuda_stream


def rel(a, b):
    a = a.double(); b = b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def gemm_args(G, M, N, K, A, B, C, ab, c_dtype, a_slots=None, b_idx=None, c_slots=None, **kw):
    a = _lib.ArmtGemmArgs()
    a.G, a.M, a.N, a.K, a.ab_dtype = G, M, N, K, ab
    a.A, a.lda, a.a_stride = A.data_ptr(), K, M * K
    a.B, a.ldb, a.b_stride = B.data_ptr(), K, N * K
    a.C, a.ldc, a.c_stride, a.c_dtype = C.data_ptr(), kw.pop("ldc", N), kw.pop("c_stride", M * N), c_dtype
    a.epilogue = kw.pop("epilogue", _lib.EPI_STORE)
    for k, v in kw.items():
        setattr(a, k, v)
    for g in range(G):
        a.a_slot[g] = a_slots[g] if a_slots else g
        a.b_index[g] = b_idx[g] if b_idx else g
        a.c_slot[g] = c_slots[g] if c_slots else g
    return a


@pytest.mark.parametrize("M,N,K", [(1152, 2048, 2048), (80, 384, 128), (128, 256, 64), (200, 320, 96),
                                   (16, 16, 8), (1152, 6144, 2048), (77, 1000, 520)])
def test_tc_gemm_store_matches_fp32(M, N, K):
    torch.manual_seed(0)
    G, L = 3, 5
    A = torch.randn(G + 1, M, K, device=DEV).bfloat16()
    B = torch.randn(L, N, K, device=DEV).bfloat16()
    C = torch.zeros(G, M, N, device=DEV)
    slots, layers = [3, 0, 2], [4, 1, 2]
    args = gemm_args(G, M, N, K, A, B, C, BF16, F32, slots, layers)
    _lib.check(LIB.armt_gemm(args, stream()), "gemm")
    for g in range(G):
        want = A[slots[g]].float() @ B[layers[g]].float().T
        assert rel(C[g], want) < 1e-5, (g, rel(C[g], want))


def test_tc_gemm_bf16_out_and_residual():
    torch.manual_seed(1)
    G, M, N, K = 2, 300, 512, 256
    A = torch.randn(G, M, K, device=DEV).bfloat16()
    B = torch.randn(G, N, K, device=DEV).bfloat16()
    C = torch.zeros(G, M, N, device=DEV, dtype=torch.bfloat16)
    _lib.check(LIB.armt_gemm(gemm_args(G, M, N, K, A, B, C, BF16, BF16), stream()), "gemm")
    want = torch.einsum("gmk,gnk->gmn", A.float(), B.float())
    assert rel(C, want) < 5e-3
    R = torch.randn(G, M, N, device=DEV)
    X = R.clone()
    C2 = torch.zeros(G, M, N, device=DEV, dtype=torch.bfloat16)
    args = gemm_args(G, M, N, K, A, B, X, BF16, F32, epilogue=_lib.EPI_RESIDUAL, R=X.data_ptr(), ldr=N,
                     r_stride=M * N, C2=C2.data_ptr(), ldc2=N, c2_stride=M * N)
    _lib.check(LIB.armt_gemm(args, stream()), "gemm")
    assert rel(X, R + want) < 1e-5
    assert rel(C2.float(), R + want) < 5e-3


def test_tc_gemm_retrieve_epilogue():
    torch.manual_seed(2)
    G, M, N, K, eps = 2, 160, 256, 96, 0.5
    A = torch.randn(G, M, K, device=DEV).bfloat16()
    B = torch.randn(G, N, K, device=DEV).bfloat16()
    den = torch.randn(G, M, device=DEV)
    den[:, :20] = 0.5  # exactly at eps: guarded (reads zero)
    R = torch.randn(G, M, N, device=DEV)
    X = R.clone()
    args = gemm_args(G, M, N, K, A, B, X, BF16, F32, epilogue=_lib.EPI_RETRIEVE, R=X.data_ptr(), ldr=N,
                     r_stride=M * N, den=den.data_ptr(), den_stride=M, eps=eps)
    _lib.check(LIB.armt_gemm(args, stream()), "gemm")
    acc = torch.einsum("gmk,gnk->gmn", A.float(), B.float())
    guard = (den.abs() <= eps)[..., None]
    want = R + torch.where(guard, torch.zeros_like(acc), acc / den[..., None])
    assert rel(X, want) < 1e-5
    assert torch.equal(X[:, :20], R[:, :20])


@pytest.mark.parametrize("block", [32, 128])
def test_tc_gemm_swiglu_epilogue(block):
    torch.manual_seed(3)
    G, M, K, F = 2, 200, 128, 512
    A = torch.randn(G, M, K, device=DEV).bfloat16()
    gate = torch.randn(G, F, K, device=DEV) * 0.2
    up = torch.randn(G, F, K, device=DEV) * 0.2
    nt = F // block
    B = torch.stack([gate.view(G, nt, block, K), up.view(G, nt, block, K)], 2).reshape(G, 2 * F, K).bfloat16()
    C = torch.zeros(G, M, F, device=DEV, dtype=torch.bfloat16)
    args = gemm_args(G, M, 2 * F, K, A, B, C, BF16, BF16, epilogue=_lib.EPI_SWIGLU, swiglu_block=block,
                     ldc=F, c_stride=M * F)
    _lib.check(LIB.armt_gemm(args, stream()), "gemm")
    gb = gate.bfloat16().float(); ub = up.bfloat16().float()
    gv = torch.einsum("gmk,gfk->gmf", A.float(), gb)
    uv = torch.einsum("gmk,gfk->gmf", A.float(), ub)
    want = torch.nn.functional.silu(gv) * uv
    assert rel(C.float(), want) < 5e-3


@pytest.mark.parametrize("dh", [8, 32, 64, 128])
def test_tc_gemm_rope_epilogue(dh):
    torch.manual_seed(4)
    H = 4
    d = H * dh
    G, M, K = 2, 144, 64
    A = torch.randn(G, M, K, device=DEV).bfloat16()
    B = torch.randn(G, 3 * d, K, device=DEV).bfloat16()
    C = torch.zeros(G, M, 3 * d, device=DEV, dtype=torch.bfloat16)
    inv = 10000.0 ** (-np.arange(0, dh, 2) / dh)
    ang = np.arange(M)[:, None] * inv[None]
    cos = torch.tensor(np.cos(ang), dtype=torch.float32, device=DEV)
    sin = torch.tensor(np.sin(ang), dtype=torch.float32, device=DEV)
    cos_t, sin_t = cos.t().contiguous(), sin.t().contiguous()
    args = gemm_args(G, M, 3 * d, K, A, B, C, BF16, BF16, epilogue=_lib.EPI_ROPE, rope_cos=cos_t.data_ptr(),
                     rope_sin=sin_t.data_ptr(), head_dim=dh, rope_cols=2 * d)
    _lib.check(LIB.armt_gemm(args, stream()), "gemm")
    acc = torch.einsum("gmk,gnk->gmn", A.float(), B.float())
    qk = acc[..., :2 * d].reshape(G, M, 2 * H, dh)
    a, b = qk[..., :dh // 2], qk[..., dh // 2:]
    c, s = cos[None, :, None], sin[None, :, None]
    rot = torch.cat([a * c - b * s, b * c + a * s], -1).reshape(G, M, 2 * d)
    want = torch.cat([rot, acc[..., 2 * d:]], -1)
    assert rel(C.float(), want) < 5e-3


@pytest.mark.parametrize("M,N,K", [(80, 384, 128), (1152, 512, 2048), (6, 50, 16), (2, 8, 8)])
def test_simt_gemm_matches_fp64(M, N, K):
    torch.manual_seed(5)
    G = 2
    A = torch.randn(G, M, K, device=DEV)
    B = torch.randn(G, N, K, device=DEV)
    C = torch.zeros(G, M, N, device=DEV)
    _lib.check(LIB.armt_gemm(gemm_args(G, M, N, K, A, B, C, F32, F32), stream()), "gemm")
    want = torch.einsum("gmk,gnk->gmn", A.double(), B.double())
    assert rel(C, want) < 1e-6


def attention_ref(qkv, H, dh):
    G, T, _ = qkv.shape
    d = H * dh
    q = qkv[..., :d].reshape(G, T, H, dh).transpose(1, 2).double()
    k = qkv[..., d:2 * d].reshape(G, T, H, dh).transpose(1, 2).double()
    v = qkv[..., 2 * d:].reshape(G, T, H, dh).transpose(1, 2).double()
    s = q @ k.transpose(-1, -2) / math.sqrt(dh)
    mask = torch.triu(torch.ones(T, T, dtype=torch.bool, device=qkv.device), 1)
    s = s.masked_fill(mask, float("-inf"))
    return (torch.softmax(s, -1) @ v).transpose(1, 2).reshape(G, T, d)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("T,H,dh", [(80, 4, 32), (1152, 4, 64), (144, 2, 128), (8, 2, 8), (200, 3, 16)])
def test_attention_matches_reference(dtype, T, H, dh):
    torch.manual_seed(6)
    G = 2
    d = H * dh
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    qkv = torch.randn(G, T, 3 * d, device=DEV).to(tdt)
    ctx = torch.zeros(G, T, d, device=DEV, dtype=tdt)
    _lib.check(LIB.armt_attention(G, qkv.data_ptr(), 3 * d, T * 3 * d, ctx.data_ptr(), d, T * d,
                                  BF16 if dtype == "bf16" else F32, T, H, dh, 1.0 / math.sqrt(dh), stream()),
               "attention")
    want = attention_ref(qkv.float(), H, dh)
    assert rel(ctx.float(), want) < (1e-2 if dtype == "bf16" else 1e-6)


@pytest.mark.parametrize("T", [64, 256, 300, 1152])
@pytest.mark.parametrize("amp", [1.0, 6.0])
@pytest.mark.parametrize("G,H", [(3, 2), (1, 3), (4, 32)])
def test_attention_dh64_pairs_and_lazy_rescale(T, amp, G, H):
    # d_head 64 runs the ping-pong kernel: odd / even / single query-tile counts,
    # a ragged tail, and large scores (amp 6 -> score spread ~ 36 / 8 per row)
    # that force the lazy running-max raises and O rescales in TMEM. An odd
    # member*head count leaves one cross-head tail item with a single group;
    # (4, 32) gives every CTA several items (the MMA issue and the O epilogue
    # are pipelined across item boundaries)
    torch.manual_seed(7)
    dh = 64
    d = H * dh
    qkv = (amp * torch.randn(G, T, 3 * d, device=DEV)).to(torch.bfloat16)
    ctx = torch.zeros(G, T, d, device=DEV, dtype=torch.bfloat16)
    _lib.check(LIB.armt_attention(G, qkv.data_ptr(), 3 * d, T * 3 * d, ctx.data_ptr(), d, T * d, BF16, T, H, dh,
                                  1.0 / math.sqrt(dh), stream()), "attention")
    want = attention_ref(qkv.float(), H, dh)
    assert rel(ctx.float(), want) < 1e-2


@pytest.mark.parametrize("T", [64, 300, 1152])
@pytest.mark.parametrize("amp", [1.0, 6.0])
@pytest.mark.parametrize("G,H", [(3, 2), (1, 3), (2, 32)])
def test_attention_dh128_pairs_and_lazy_rescale(T, amp, G, H, monkeypatch):
    # d_head 128 runs the ping-pong kernel on 64-key steps (C5's head size): odd / even /
    # single query-tile counts, a ragged tail, large scores forcing O rescales, and the
    # single-tile tcgen05 kernel (ARMT_ATTN=tc) as a second check
    torch.manual_seed(8)
    dh = 128
    d = H * dh
    qkv = (amp * torch.randn(G, T, 3 * d, device=DEV)).to(torch.bfloat16)
    want = attention_ref(qkv.float(), H, dh)
    for force in (None, "tc"):
        if force:
            monkeypatch.setenv("ARMT_ATTN", force)
        ctx = torch.zeros(G, T, d, device=DEV, dtype=torch.bfloat16)
        _lib.check(LIB.armt_attention(G, qkv.data_ptr(), 3 * d, T * 3 * d, ctx.data_ptr(), d, T * d, BF16, T, H,
                                      dh, 1.0 / math.sqrt(dh), stream()), "attention")
        assert rel(ctx.float(), want) < 1e-2, force


def test_dpfp_known_answers_on_device():
    # pkg/tests/test_memory.py:25-33 pinned on the device feature map
    from paper_2506_05229_b200.layers import dpfp
    assert dpfp(torch.tensor([2.0], device=DEV), 3).cpu().tolist() == [0, 0, 4, 0, 0, 0]
    assert dpfp(torch.tensor([-2.0], device=DEV), 3).cpu().tolist() == [0, 0, 0, 4, 0, 0]
    assert dpfp(torch.tensor([1.0, -2.0], device=DEV), 1).cpu().tolist() == [0, 0, 0, 2]


@pytest.mark.parametrize("d,M,d_mem,eps", [(128, 16, 16, 1.0), (2048, 128, 64, 1.0), (16, 2, 4, 1e-6),
                                           (96, 5, 3, 0.1)])
def test_fold_matches_oracle(d, M, d_mem, eps):
    import armt_oracle as O
    rng = np.random.default_rng(7)
    nu = 3
    dphi = 2 * nu * d_mem
    G, L = 2, 3
    layers = [2, 0]
    A0 = (rng.standard_normal((L, d, dphi)) * 0.1).astype(np.float32)
    z0 = np.abs(rng.standard_normal((L, dphi))).astype(np.float32)
    n_kvb = ((d + d_mem + 1 + 15) // 16) * 16
    kvb = np.zeros((G, M, n_kvb), np.float32)
    kvb[:, :, :d] = rng.standard_normal((G, M, d))
    kvb[:, :, d:d + d_mem] = rng.standard_normal((G, M, d_mem))
    kvb[:, :, d + d_mem] = rng.standard_normal((G, M))
    A = torch.tensor(A0, device=DEV)
    z = torch.tensor(z0, device=DEV)
    kv = torch.tensor(kvb, device=DEV)
    ws = torch.empty(LIB.armt_fold_workspace_bytes(G, M, dphi) // 4 + 1, device=DEV)
    mem = _lib.members([0, 1], layers)
    _lib.check(LIB.armt_mem_fold(mem, kv.data_ptr(), n_kvb, M * n_kvb, 0, d, d + d_mem, A.data_ptr(),
                                 z.data_ptr(), None, 0, d, M, d_mem, nu, eps, ws.data_ptr(), stream()), "fold")
    for g, l in enumerate(layers):
        Ar, zr = A0[l].astype(np.float64), z0[l].astype(np.float64)
        # restate the fold inputs exactly as update_stack builds them
        k = kvb[g, :, d:d + d_mem].astype(np.float64)
        v = kvb[g, :, :d].astype(np.float64)
        beta = O.sigmoid(kvb[g, :, d + d_mem].astype(np.float64))
        phi = O.dpfp(k, nu)
        for i in range(M):
            p = phi[i]
            zq = zr @ p
            nrm = p @ p
            vbar = np.zeros(d) if abs(zq) <= eps else (Ar @ p) / zq
            gam = 0.0 if nrm <= eps else 1 - zq / nrm
            Ar += np.outer(beta[i] * (v[i] - vbar), p)
            zr += gam * p
        assert rel(A[l].cpu(), torch.tensor(Ar)) < 1e-5
        assert rel(z[l].cpu(), torch.tensor(zr)) < 1e-5
    assert torch.equal(A[1].cpu(), torch.tensor(A0[1]))  # untouched layer


def _fold64(A0, z0, kvb_g, d, d_mem, nu, eps):
    """In-order delta rule in f64 (armt/memory.py:94-125) on the device fold's inputs."""
    import armt_oracle as O
    Ar, zr = A0.astype(np.float64).copy(), z0.astype(np.float64).copy()
    k = kvb_g[:, d:d + d_mem].astype(np.float64)
    v = kvb_g[:, :d].astype(np.float64)
    beta = O.sigmoid(kvb_g[:, d + d_mem].astype(np.float64))
    phi = O.dpfp(k, nu)
    for i in range(k.shape[0]):
        p = phi[i]
        zq, nrm = zr @ p, p @ p
        vbar = np.zeros(d) if abs(zq) <= eps else (Ar @ p) / zq
        gam = 0.0 if nrm <= eps else 1 - zq / nrm
        Ar += np.outer(beta[i] * (v[i] - vbar), p)
        zr += gam * p
    return Ar, zr


@pytest.mark.parametrize("d,M,d_mem,nu,eps,G", [(2048, 128, 64, 3, 100.0, 3), (2048, 128, 64, 3, 1.0, 3),
                                                (256, 16, 16, 3, 10.0, 3), (384, 24, 32, 2, 10.0, 3),
                                                (128, 16, 16, 3, 1e-6, 3),
                                                # 16 members: more K blocks than SMs -> split prep + K kernel
                                                (2048, 128, 64, 3, 100.0, 16)])
def test_tensor_core_fold_matches_in_order_f64(d, M, d_mem, nu, eps, G):
    """armt_mem_fold_tc (chunked form: bf16x3 tensor-core GEMMs around the chain
    and an explicit L^{-1}) against the in-order f64 delta rule on a LIVE state
    (nonzero A, z): A and z within 1e-5 relative, untouched layers bitwise,
    and the bf16x3 memory operand it refreshes equal to a fresh split of the
    new A and z (the retrieval reads it)."""
    from types import SimpleNamespace
    from paper_2506_05229_b200.engine import MemoryState
    rng = np.random.default_rng(11)
    dphi = 2 * nu * d_mem
    P = (dphi + 31) // 32 * 32
    L = G + 1
    layers = [3, 0, 2] if G == 3 else [int(x) for x in rng.permutation(L)[:G]]
    skipped = sorted(set(range(L)) - set(layers))[0]
    A0 = (rng.standard_normal((L, d, dphi)) * 0.05).astype(np.float32)
    z0 = (np.abs(rng.standard_normal((L, dphi))) * 3).astype(np.float32)
    n_kvb = ((d + d_mem + 1 + 15) // 16) * 16
    kvb = np.zeros((G, M, n_kvb), np.float32)
    kvb[:, :, :d] = rng.standard_normal((G, M, d))
    kvb[:, :, d:d + d_mem] = rng.standard_normal((G, M, d_mem))
    kvb[:, :, d + d_mem] = rng.standard_normal((G, M))
    st = MemoryState(A=torch.tensor(A0, device=DEV), z=torch.tensor(z0, device=DEV), updates=np.zeros(L, np.int64))
    prep = SimpleNamespace(dtype_name="bf16", d_phi_pad=P, config=SimpleNamespace(num_mem_tokens=M))
    st.sync_shadow(prep)
    kv = torch.tensor(kvb, device=DEV)
    ws = torch.zeros(LIB.armt_fold_tc_workspace_bytes(G, M, d, dphi) // 4 + 1, device=DEV)
    mem = _lib.members(list(range(G)), layers)
    _lib.check(LIB.armt_mem_fold_tc(mem, kv.data_ptr(), n_kvb, M * n_kvb, 0, d, d + d_mem, st.A.data_ptr(),
                                    st.z.data_ptr(), st.memop.data_ptr(), d, M, d_mem, nu, eps, ws.data_ptr(),
                                    stream()), "fold_tc")
    torch.cuda.synchronize()
    for g, l in enumerate(layers):
        Ar, zr = _fold64(A0[l], z0[l], kvb[g], d, d_mem, nu, eps)
        assert rel(st.A[l].cpu(), torch.tensor(Ar)) < 1e-5, (l, rel(st.A[l].cpu(), torch.tensor(Ar)))
        assert rel(st.z[l].cpu(), torch.tensor(zr)) < 1e-5
    assert torch.equal(st.A[skipped].cpu(), torch.tensor(A0[skipped]))
    # the refreshed operand: rows 0..d-1 = [hi | lo] of A, row d = that of z
    op = st.memop.float()
    assert st.memop.shape[2] == 2 * P
    for l in layers:
        hi, lo = op[l, :d, :dphi], op[l, :d, P:P + dphi]
        assert rel(hi + lo, st.A[l]) < 2e-5
        assert torch.equal(hi, st.A[l].to(torch.bfloat16).float())
        assert rel(op[l, d, :dphi] + op[l, d, P:P + dphi], st.z[l]) < 2e-5


def test_rmsnorm_matches_reference():
    torch.manual_seed(8)
    G, T, d, L = 3, 100, 256, 4
    x = torch.randn(5, T, d, device=DEV)
    gain = torch.rand(L, d, device=DEV) + 0.5
    out = torch.empty(G, T, d, device=DEV)
    mem = _lib.members([4, 1, 2], [3, 0, 0])
    _lib.check(LIB.armt_rmsnorm(mem, x.data_ptr(), T * d, gain.data_ptr(), out.data_ptr(), F32, T * d, T, d,
                                1e-6, stream()), "rmsnorm")
    for g, (s, l) in enumerate([(4, 3), (1, 0), (2, 0)]):
        xr = x[s].double()
        want = xr / torch.sqrt((xr * xr).mean(-1, keepdim=True) + 1e-6) * gain[l].double()
        assert rel(out[g], want) < 1e-6


def test_kernel_counter_advances():
    before = LIB.armt_kernel_count()
    x = torch.zeros(16, device=DEV)
    y = torch.zeros(16, device=DEV, dtype=torch.bfloat16)
    _lib.check(LIB.armt_cast(x.data_ptr(), F32, y.data_ptr(), BF16, 16, stream()), "cast")
    assert LIB.armt_kernel_count() == before + 1


@pytest.mark.parametrize("dtype,V", [("bf16", 128256), ("f32", 1000), ("bf16", 50)])
def test_logits_nll_matches_log_softmax(dtype, V):
    torch.manual_seed(9)
    rows = 37
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    logits = (torch.randn(rows, V, device=DEV) * 4).to(tdt)
    tgt = torch.randint(0, V, (rows,), device=DEV)
    out = torch.empty(rows, device=DEV)
    _lib.check(LIB.armt_logits_nll(logits.data_ptr(), BF16 if dtype == "bf16" else F32, V, tgt.data_ptr(),
                                   out.data_ptr(), rows, V, stream()), "nll")
    want = -torch.log_softmax(logits.double(), -1).gather(1, tgt[:, None])[:, 0]
    assert rel(out, want) < 1e-5


@pytest.mark.parametrize("epi", ["store", "residual", "rope", "swiglu", "lse"])
def test_tc_gemm_cta_pair_and_multicast_match_single_cta(epi, monkeypatch):
    """The CTA-pair (cta_group::2, 256-row) tiles plus the single-CTA remainder
    launch, and the multicast clusters (B- or A-sharing tile pairs), must
    reproduce the plain single-CTA kernel at a C2 member height (1152 rows = 4
    pair tiles + 128 remainder rows; 9 m-tiles = 4 B-sharing pairs + 1
    A-sharing pair per n-block pair) for every epilogue."""
    torch.manual_seed(7)
    G, M = 3, 1152
    K = 4096 if epi == "residual" else 1024
    dh, H = 64, 8
    N = {"store": 512, "residual": 512, "rope": 3 * H * dh, "swiglu": 1024, "lse": 1000}[epi]
    A = torch.randn(G, M, K, device=DEV).bfloat16()
    B = (torch.randn(G, N, K, device=DEV) * 0.05).bfloat16()
    monkeypatch.setenv("ARMT_GEMM_BN", "256")

    def run(pair, mc="0"):
        monkeypatch.setenv("ARMT_GEMM_PAIR", pair)
        monkeypatch.setenv("ARMT_GEMM_MC", mc)
        kw, outs = {}, []
        if epi == "store":
            C = torch.zeros(G, M, N, device=DEV)
            args = gemm_args(G, M, N, K, A, B, C, BF16, F32)
            outs = [C]
        elif epi == "residual":
            C = torch.randn(G, M, N, device=DEV, generator=torch.Generator(DEV).manual_seed(1))
            C2 = torch.zeros(G, M, N, device=DEV, dtype=torch.bfloat16)
            ssq = torch.zeros(G, M, N // 64, device=DEV)
            args = gemm_args(G, M, N, K, A, B, C, BF16, F32, epilogue=_lib.EPI_RESIDUAL, R=C.data_ptr(), ldr=N,
                             r_stride=M * N, C2=C2.data_ptr(), ldc2=N, c2_stride=M * N, ssq_out=ssq.data_ptr(),
                             ssq_stride=M * (N // 64), ssq_np=N // 64)
            outs = [C, C2, ssq]
        elif epi == "rope":
            inv = 10000.0 ** (-np.arange(0, dh, 2) / dh)
            ang = np.arange(M)[:, None] * inv[None]
            cos_t = torch.tensor(np.cos(ang).T.copy(), dtype=torch.float32, device=DEV)
            sin_t = torch.tensor(np.sin(ang).T.copy(), dtype=torch.float32, device=DEV)
            C = torch.zeros(G, M, N, device=DEV, dtype=torch.bfloat16)
            args = gemm_args(G, M, N, K, A, B, C, BF16, BF16, epilogue=_lib.EPI_ROPE, rope_cos=cos_t.data_ptr(),
                             rope_sin=sin_t.data_ptr(), head_dim=dh, rope_cols=2 * H * dh)
            outs = [C]
            kw = {"keep": (cos_t, sin_t)}
        elif epi == "swiglu":
            C = torch.zeros(G, M, N // 2, device=DEV, dtype=torch.bfloat16)
            args = gemm_args(G, M, N, K, A, B, C, BF16, BF16, epilogue=_lib.EPI_SWIGLU, swiglu_block=128,
                             ldc=N // 2, c_stride=M * N // 2)
            outs = [C]
        else:
            tiles = -(-N // 256)
            part = torch.zeros(M, tiles, 2, device=DEV)
            tgt = torch.zeros(M, device=DEV)
            ids = torch.randint(0, N, (M + 1,), device=DEV, generator=torch.Generator(DEV).manual_seed(2))
            C = torch.zeros(1, device=DEV)
            args = gemm_args(1, M, N, K, A, B, C, BF16, F32, epilogue=_lib.EPI_LSE, ldc=1, c_stride=0,
                             lse_part=part.data_ptr(), lse_ld=tiles, targets=ids.data_ptr() + 8,
                             lse_tgt=tgt.data_ptr(), lse_rows=M)
            outs = [part, tgt]
            kw = {"keep": ids}
        _lib.check(LIB.armt_gemm(args, stream()), "gemm")
        torch.cuda.synchronize()
        return [o.float().clone() for o in outs]

    single, paired, multicast = run("0"), run("split"), run("0", "1")
    for s_, p_, m_ in zip(single, paired, multicast):
        assert torch.isfinite(p_).all()
        assert rel(p_, s_) < 1e-6, (epi, rel(p_, s_))
        assert torch.equal(m_, s_), (epi, rel(m_, s_))   # same MMA per tile: bitwise


@pytest.mark.parametrize("d_mem,nu", [(64, 3), (16, 3), (32, 2), (64, 1)])
def test_tc_gemm_dpfp_epilogue(d_mem, nu):
    """q-projection with the DPFP feature map and phi.z fused into the epilogue
    (armt/memory.py:34-45,137-147) against torch on the same bf16 operands."""
    torch.manual_seed(11)
    G, M, K = 3, 300, 256
    dphi = 2 * nu * d_mem
    ld = (dphi + 7) // 8 * 8
    A = torch.randn(G, M, K, device=DEV).bfloat16()
    B = (torch.randn(5, d_mem, K, device=DEV) * 0.1).bfloat16()
    z = torch.randn(7, dphi, device=DEV)
    phi = torch.zeros(G, M, ld, device=DEV, dtype=torch.bfloat16)
    den = torch.zeros(G, M, device=DEV)
    layers, zrows = [4, 0, 2], [6, 1, 3]
    args = gemm_args(G, M, d_mem, K, A, B, phi, BF16, BF16, None, layers, None, epilogue=_lib.EPI_DPFP,
                     ldc=ld, c_stride=M * ld, den=den.data_ptr(), den_stride=M, z=z.data_ptr(), nu=nu)
    for g in range(G):
        args.e_index[g] = zrows[g]
    _lib.check(LIB.armt_gemm(args, stream()), "gemm dpfp")
    for g in range(G):
        q = A[g].float() @ B[layers[g]].float().T
        r = torch.cat([q.clamp_min(0), (-q).clamp_min(0)], -1)
        want = torch.cat([r * torch.roll(r, -j, -1) for j in range(1, nu + 1)], -1)
        assert rel(phi[g, :, :dphi].float(), want) < 5e-3
        assert torch.count_nonzero(phi[g, :, dphi:]) == 0
        assert rel(den[g], want @ z[zrows[g]]) < 1e-4


def test_tc_gemm_concurrent_remainder_from_many_streams(monkeypatch):
    """The QKV+RoPE GEMM forks its single-CTA remainder onto a per-caller side
    stream; callers on more streams than fork slots (e.g. one capture stream per
    per-step graph) must still get correct results (sequential fallback)."""
    torch.manual_seed(12)
    monkeypatch.setenv("ARMT_GEMM_BN", "256")
    monkeypatch.delenv("ARMT_GEMM_PAIR", raising=False)
    G, M, K, dh, H = 2, 1152, 1024, 64, 8
    N = 3 * H * dh
    A = torch.randn(G, M, K, device=DEV).bfloat16()
    B = (torch.randn(G, N, K, device=DEV) * 0.05).bfloat16()
    inv = 10000.0 ** (-np.arange(0, dh, 2) / dh)
    ang = np.arange(M)[:, None] * inv[None]
    cos_t = torch.tensor(np.cos(ang).T.copy(), dtype=torch.float32, device=DEV)
    sin_t = torch.tensor(np.sin(ang).T.copy(), dtype=torch.float32, device=DEV)
    outs = []
    for _ in range(40):
        st = torch.cuda.Stream()
        C = torch.zeros(G, M, N, device=DEV, dtype=torch.bfloat16)
        args = gemm_args(G, M, N, K, A, B, C, BF16, BF16, epilogue=_lib.EPI_ROPE, rope_cos=cos_t.data_ptr(),
                         rope_sin=sin_t.data_ptr(), head_dim=dh, rope_cols=2 * H * dh)
        st.wait_stream(torch.cuda.current_stream())
        _lib.check(LIB.armt_gemm(args, st.cuda_stream), "gemm")
        torch.cuda.current_stream().wait_stream(st)
        outs.append(C)
    torch.cuda.synchronize()
    for C in outs[1:]:
        assert torch.equal(C, outs[0])


@pytest.mark.parametrize("epi,M,N,K,split,bn", [
    ("residual", 1152, 2048, 1024, False, None),   # pair tiles + remainder (TMA epilogue needs K <= 1024)
    ("retrieve", 1152, 2048, 384, False, None),    # retrieval numerator shape
    ("residual", 2048, 384, 768, True, "128"),     # fold update: A += ..., memop [hi | lo] rows
    ("residual", 300, 520, 256, False, "64"),      # ragged rows / columns
    ("retrieve", 77, 1000, 96, False, "256"),
])
def test_tc_gemm_tma_epilogue_matches_register_epilogue(epi, M, N, K, split, bn, monkeypatch):
    """The TMA epilogue of the short-K residual / retrieve GEMMs (residual tile
    TMA-loaded into swizzled smem, f32 result and bf16 copy TMA-stored) is
    bitwise the register (coalesced-transpose) epilogue: outputs, bf16 copy or
    [hi | lo] split, and the per-64-column row sums of squares."""
    torch.manual_seed(12)
    G = 3
    A = torch.randn(G, M, K, device=DEV).bfloat16()
    B = (torch.randn(G, N, K, device=DEV) * 0.05).bfloat16()
    X0 = torch.randn(G + 1, M, N, device=DEV)
    den = torch.randn(G, M, device=DEV)
    den[:, :7] = 0.25
    if bn:
        monkeypatch.setenv("ARMT_GEMM_BN", bn)
    np_ = -(-N // 64)
    P = -(-N // 32) * 32
    slots = [2, 0, 3]

    def run(tmae):
        monkeypatch.setenv("ARMT_GEMM_TMAE", tmae)
        X = X0.clone()
        ssq = torch.zeros(G, M, np_, device=DEV)
        ld2 = 2 * P if split else N
        C2 = torch.zeros(G + 1, M, ld2, device=DEV, dtype=torch.bfloat16)
        kw = dict(epilogue=_lib.EPI_RESIDUAL if epi == "residual" else _lib.EPI_RETRIEVE, R=X.data_ptr(), ldr=N,
                  r_stride=M * N, C2=C2.data_ptr(), ldc2=ld2, c2_stride=M * ld2, ssq_out=ssq.data_ptr(),
                  ssq_stride=M * np_, ssq_np=np_)
        if split:
            kw["c2_split"] = P
        if epi == "retrieve":
            kw.update(den=den.data_ptr(), den_stride=M, eps=0.25)
        args = gemm_args(G, M, N, K, A, B, X, BF16, F32, c_slots=slots, **kw)
        _lib.check(LIB.armt_gemm(args, stream()), "gemm")
        torch.cuda.synchronize()
        return X, C2, ssq

    ref = run("0")
    got = run("1")
    for a, b in zip(ref, got):
        assert torch.equal(a, b)
    acc = torch.einsum("gmk,gnk->gmn", A.float(), B.float())
    if epi == "retrieve":
        acc = torch.where(den.abs()[..., None] <= 0.25, torch.zeros_like(acc), acc / den[..., None])
    for g, sl in enumerate(slots):
        assert rel(got[0][sl], X0[sl] + acc[g]) < 1e-5


def test_tc_gemm_k_wrap_reuses_operand_columns():
    """a_kwrap / b_kwrap: a bf16x3 operand stored as [hi | lo] and read as
    [hi | lo | hi] through the K wrap gives bitwise the GEMM on the explicit
    three-part operand (the memory operand and the fold's [V | P] operand)."""
    torch.manual_seed(13)
    G, M, N, P = 2, 256, 192, 128
    hiA = torch.randn(G, M, P, device=DEV).bfloat16()
    loA = (torch.randn(G, M, P, device=DEV) * 1e-3).bfloat16()
    Bm = torch.randn(G, N, 3 * P, device=DEV).bfloat16()
    full = torch.cat([hiA, loA, hiA], -1).contiguous()
    two = torch.cat([hiA, loA], -1).contiguous()
    C1 = torch.zeros(G, M, N, device=DEV)
    C2 = torch.zeros(G, M, N, device=DEV)
    _lib.check(LIB.armt_gemm(gemm_args(G, M, N, 3 * P, full, Bm, C1, BF16, F32), stream()), "gemm")
    a = gemm_args(G, M, N, 3 * P, two, Bm, C2, BF16, F32)
    a.lda, a.a_stride, a.a_kwrap = 2 * P, M * 2 * P, 2 * P
    _lib.check(LIB.armt_gemm(a, stream()), "gemm")
    torch.cuda.synchronize()
    assert torch.equal(C1, C2)
    # the same on the B side
    C3 = torch.zeros(G, M, N, device=DEV)
    At = torch.randn(G, M, 3 * P, device=DEV).bfloat16()
    hiB = torch.randn(G, N, P, device=DEV).bfloat16()
    loB = (torch.randn(G, N, P, device=DEV) * 1e-3).bfloat16()
    fullB = torch.cat([hiB, loB, hiB], -1).contiguous()
    twoB = torch.cat([hiB, loB], -1).contiguous()
    _lib.check(LIB.armt_gemm(gemm_args(G, M, N, 3 * P, At, fullB, C1, BF16, F32), stream()), "gemm")
    b = gemm_args(G, M, N, 3 * P, At, twoB, C3, BF16, F32)
    b.ldb, b.b_stride, b.b_kwrap = 2 * P, N * 2 * P, 2 * P
    _lib.check(LIB.armt_gemm(b, stream()), "gemm")
    torch.cuda.synchronize()
    assert torch.equal(C1, C3)
