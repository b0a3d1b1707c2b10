"""Grouped tensor primitives on the device (mirrors armt/tensor_ops.py).

``grouped_gemm(a, b, out)`` keeps the reference signature (a (G,m,k), b
(G,k,n) in ``x @ w`` layout, one pre-allocated ``GroupedBuffer`` output —
the paper's "single large tensor") and runs ONE launch of the
tcgen05 kernel (bf16) or the SIMT kernel (f32) over all members.

``WorkerPool`` survives only as the reference's slab bookkeeping
(armt/tensor_ops.py:74-139): on the device, one grouped launch replaces the
thread slabs, so the pool never dispatches anything.
"""

from __future__ import annotations

import os

import torch

from . import _lib
from .errors import DimensionError, InputError

_DT = {torch.float32: _lib.F32, torch.bfloat16: _lib.BF16}


class GroupedBuffer:
    """One contiguous (G, *member_shape) device allocation (armt/tensor_ops.py:146-190)."""

    def __init__(self, group_size: int, member_shape: tuple[int, ...], dtype=torch.float32, device=None):
        if group_size < 1:
            raise DimensionError(f"group_size must be >= 1, got {group_size}")
        member_shape = tuple(int(s) for s in member_shape)
        if any(s < 1 for s in member_shape):
            raise DimensionError(f"member_shape must be positive, got {member_shape}")
        if dtype not in _DT:
            raise DimensionError(f"unsupported dtype {dtype}")
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.array = torch.empty((group_size, *member_shape), dtype=dtype, device=dev)

    @classmethod
    def wrap(cls, array: torch.Tensor) -> "GroupedBuffer":
        if array.dim() < 2:
            raise DimensionError("backing array needs a leading group axis")
        buf = cls.__new__(cls)
        buf.array = array
        return buf

    @property
    def group_size(self) -> int:
        return self.array.shape[0]

    @property
    def member_shape(self) -> tuple[int, ...]:
        return tuple(self.array.shape[1:])

    @property
    def dtype(self):
        return self.array.dtype

    def member(self, g: int) -> torch.Tensor:
        if not 0 <= g < self.group_size:
            raise DimensionError(f"member index {g} out of range 0..{self.group_size - 1}")
        return self.array[g]


def _stack(name, members) -> torch.Tensor:
    if isinstance(members, torch.Tensor):
        if members.dim() != 3:
            raise DimensionError(f"{name} must be a 3-d tensor")
        return members
    arrs = list(members)
    if not arrs:
        raise DimensionError(f"{name} must hold at least one member")
    if any(a.shape != arrs[0].shape or a.dtype != arrs[0].dtype for a in arrs):
        raise DimensionError(f"{name} members must share shape and dtype")
    return torch.stack(arrs)


def grouped_gemm(a_members, b_members, out: GroupedBuffer, pool=None) -> GroupedBuffer:
    """out[g] = a[g] @ b[g] in one launch (armt/tensor_ops.py:237-264)."""
    a3 = _stack("a_members", a_members)
    b3 = _stack("b_members", b_members)
    if a3.shape[0] != b3.shape[0]:
        raise DimensionError(f"group sizes disagree: {a3.shape[0]} vs {b3.shape[0]}")
    if a3.shape[2] != b3.shape[1]:
        raise DimensionError(f"inner dims disagree: {tuple(a3.shape)} @ {tuple(b3.shape)}")
    if a3.dtype != b3.dtype or a3.dtype not in _DT:
        raise DimensionError(f"dtype mismatch/unsupported: {a3.dtype} vs {b3.dtype}")
    G, m, k = a3.shape
    n = b3.shape[2]
    if not isinstance(out, GroupedBuffer):
        raise DimensionError("out must be a GroupedBuffer")
    if out.group_size != G or out.member_shape != (m, n) or out.dtype != a3.dtype:
        raise DimensionError(f"out buffer must be {G}x{(m, n)} {a3.dtype}, got "
                             f"{out.group_size}x{out.member_shape} {out.dtype}")
    a3 = a3.contiguous()
    bt = b3.transpose(1, 2).contiguous()   # K-major operand layout
    args = _lib.ArmtGemmArgs()
    args.G, args.M, args.N, args.K = G, m, n, k
    args.ab_dtype = _DT[a3.dtype]
    args.A, args.lda, args.a_stride = a3.data_ptr(), k, m * k
    args.B, args.ldb, args.b_stride = bt.data_ptr(), k, n * k
    args.C, args.ldc, args.c_stride, args.c_dtype = out.array.data_ptr(), n, m * n, _DT[out.dtype]
    args.epilogue = _lib.EPI_STORE
    for g in range(G):
        args.a_slot[g] = args.b_index[g] = args.c_slot[g] = g
    _lib.check(_lib.load().armt_gemm(args, torch.cuda.current_stream().cuda_stream), "grouped_gemm")
    return out


def gemm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """a @ b for 2-d device tensors (armt/tensor_ops.py:204-220)."""
    if a.dim() != 2 or b.dim() != 2:
        raise DimensionError("gemm operands must be 2-d")
    if a.shape[1] != b.shape[0]:
        raise DimensionError(f"inner dims disagree: {tuple(a.shape)} @ {tuple(b.shape)}")
    buf = GroupedBuffer.wrap((out if out is not None else
                              torch.empty(a.shape[0], b.shape[1], dtype=a.dtype, device=a.device))[None])
    grouped_gemm(a[None], b[None], buf)
    return buf.array[0]


def rms_norm_stacked(x: torch.Tensor, gains: torch.Tensor, eps: float = 1e-6) -> torch.Tensor:
    """x / sqrt(mean(x^2) + eps) * gains[g] over a (G, T, d) stack (armt/tensor_ops.py:267-281)."""
    if x.dim() != 3 or gains.dim() != 2:
        raise DimensionError(f"expected x (G,T,d) and gains (G,d), got {tuple(x.shape)} / {tuple(gains.shape)}")
    if x.shape[0] != gains.shape[0] or x.shape[2] != gains.shape[1]:
        raise DimensionError(f"shape mismatch: x {tuple(x.shape)} vs gains {tuple(gains.shape)}")
    if x.dtype != torch.float32 or gains.dtype != torch.float32:
        raise DimensionError("rms_norm_stacked takes float32 tensors")
    G, T, d = x.shape
    x = x.contiguous()
    gains = gains.contiguous()
    out = torch.empty_like(x)
    mem = _lib.members(range(G), range(G))
    _lib.check(_lib.load().armt_rmsnorm(mem, x.data_ptr(), T * d, gains.data_ptr(), out.data_ptr(), _lib.F32,
                                        T * d, T, d, float(eps), torch.cuda.current_stream().cuda_stream),
               "rms_norm_stacked")
    return out


class WorkerPool:
    """Slab bookkeeping only (armt/tensor_ops.py:74-139); never dispatches."""

    def __init__(self, threads: int = 1, *, slabs: int | None = None):
        if not isinstance(threads, int) or threads < 1:
            raise InputError(f"threads must be a positive int, got {threads!r}")
        if slabs is None:
            slabs = max(1, min(threads, os.cpu_count() or 1))
        elif not isinstance(slabs, int) or slabs < 1:
            raise InputError(f"slabs must be a positive int, got {slabs!r}")
        self.threads = threads
        self.slabs = slabs

    def slab_bounds(self, group_size: int) -> list[tuple[int, int]]:
        k = min(self.slabs, group_size)
        base, rem = divmod(group_size, k)
        out, lo = [], 0
        for s in range(k):
            hi = lo + base + (1 if s < rem else 0)
            out.append((lo, hi))
            lo = hi
        return out

    def slab_assignment(self, group_size: int) -> list[int]:
        return [s for s, (lo, hi) in enumerate(self.slab_bounds(group_size)) for _ in range(hi - lo)]

    def close(self) -> None:
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False
