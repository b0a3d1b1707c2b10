"""Attention at C5 head size (d_head 128, 32 heads, T = 1152): the tcgen05 single-tile
kernel vs torch SDPA (flash / cuDNN) on the same causal problem. python scripts/attn128_bench.py [G]"""
import json
import math
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2506_05229_b200 import _lib  # noqa: E402
from paper_2506_05229_b200._lib import BF16  # noqa: E402

LIB = _lib.load()
G = int(sys.argv[1]) if len(sys.argv) > 1 else 16
T, H, dh = 1152, 32, 128
d = H * dh
qkv = torch.randn(G, T, 3 * d, device="cuda").bfloat16()
ctx = torch.empty(G, T, d, device="cuda", dtype=torch.bfloat16)
s = torch.cuda.current_stream().cuda_stream
fn = lambda: _lib.check(LIB.armt_attention(G, qkv.data_ptr(), 3 * d, T * 3 * d, ctx.data_ptr(), d, T * d, BF16, T, H,
                                           dh, 1 / math.sqrt(dh), s), "attn")
q, k, v = (t.view(G, T, H, dh).transpose(1, 2).contiguous() for t in qkv.split(d, dim=-1))
sdpa = lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)


def timeit(f, it=30):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / it


us, us_s = timeit(fn), timeit(sdpa)
flops = G * 4 * d * T * (T + 1) / 2
ref = sdpa().transpose(1, 2).reshape(G, T, d).float()
err = float((ctx.float() - ref).norm() / ref.norm())
print(json.dumps({"G": G, "dh": dh, "us": us, "tflops": flops / us / 1e6, "sdpa_us": us_s,
                  "sdpa_tflops": flops / us_s / 1e6, "rel_err_vs_sdpa": err}))
