"""Pipeline timeline of the ping-pong attention on CTA 0 (debug build with
-DARMT_PP_TRACE, loaded through ARMT_LIB_PATH). One C2 wavefront step (G=16).
Prints per-group averages: wait for S, S load..exps done, wait for P buffer, P
written, and the MMA thread's waits, in SM clocks."""
import ctypes
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2506_05229_b200 import _lib  # noqa: E402
from paper_2506_05229_b200._lib import BF16  # noqa: E402

LIB = _lib.load()
G = int(sys.argv[1]) if len(sys.argv) > 1 else 16
T, d, H, dh = 1152, 2048, 32, 64
qkv = torch.randn(G, T, 3 * d, device="cuda").bfloat16()
ctx = torch.empty(G, T, d, device="cuda", dtype=torch.bfloat16)
s = torch.cuda.current_stream().cuda_stream
run = lambda: _lib.check(LIB.armt_attention(G, qkv.data_ptr(), 3 * d, T * 3 * d, ctx.data_ptr(), d, T * d, BF16, T,
                                            H, dh, 1 / math.sqrt(dh), s), "attn")
buf = np.zeros(4 * 16384, np.uint64)
cnt = np.zeros(4, np.int32)
read = LIB.armt_pp_trace_read
run(); torch.cuda.synchronize()
read(buf.ctypes.data_as(ctypes.c_void_p), cnt.ctypes.data_as(ctypes.c_void_p))   # drop the warm-up
run(); torch.cuda.synchronize()
read(buf.ctypes.data_as(ctypes.c_void_p), cnt.ctypes.data_as(ctypes.c_void_p))
recs = []
for reg in range(4):
    for x in buf[reg * 16384: reg * 16384 + cnt[reg]]:
        x = int(x)
        recs.append((reg, x >> 56, (x >> 40) & 0xffff, x & 0xffffffffff))
t0 = min(r[3] for r in recs)
span = max(r[3] for r in recs) - t0
print(f"CTA 0: {cnt.tolist()} records, span {span} clocks")
for g in (0, 1):
    ev = {}
    for reg, e, i, c in recs:
        if reg == g:
            ev.setdefault(i, {})[e] = c
    rows = [v for v in ev.values() if len(v) == 5]
    a = lambda x, y: np.mean([r[y] - r[x] for r in rows])
    tot = np.sum([r[5] - r[1] for r in rows])
    print(f"group {g}: tiles {len(rows)}  wait S {a(1, 2):.0f}  ld+max+exp {a(2, 3):.0f}  wait P-free {a(3, 4):.0f}  "
          f"P out+arrive {a(4, 5):.0f}  per tile {a(1, 5):.0f}  busy {tot / span:.2f} of span")
    gaps = [ev[i + 1][1] - ev[i][5] for i in ev if i + 1 in ev and 5 in ev[i] and 1 in ev[i + 1]]
    print(f"   between tiles (arrive -> next wait) {np.mean(gaps):.0f}")
mma = {}
for reg, e, i, c in recs:
    if reg == 2:
        mma.setdefault(e, []).append(c)
for e, name in [(1, "S_A issue"), (2, "S_B issue"), (3, "P_A full"), (4, "P_B full"), (5, "KV full")]:
    print(name, len(mma.get(e, [])))
# full timeline of the first 40 tiles of group 0/1 (relative clocks)
for reg, e, i, c in sorted(recs, key=lambda r: r[3])[:300]:
    print(f"{c - t0:8d}  r{reg} e{e} i{i}")
