# fused kernels vs the library baseline (cuBLAS bmm / torch SDPA) at C2 shapes, G=16 and G=8
timeout 600 python scripts/kernel_bench.py --G 16 --ops gu,down,qkv,o,num,attn,lm --iters 20 --cublas > gpurun_out/libcmp_g16.log 2>&1
timeout 600 python scripts/kernel_bench.py --G 8 --ops gu,down,qkv,o,num,attn --iters 20 --cublas > gpurun_out/libcmp_g8.log 2>&1
