"""Run the cuBLAS (torch.bmm) form of one C2 GEMM a few times - for ncu
captures of the library kernel next to ours (scripts/gpu_libcmp.sh)."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/", 2)[0])
from scripts.kernel_bench import cublas_op, gemm_specs  # noqa: E402

op = sys.argv[1] if len(sys.argv) > 1 else "gu"
g_only, _, keep = cublas_op(*gemm_specs(16)[op])
for _ in range(3):
    g_only()
torch.cuda.synchronize()
