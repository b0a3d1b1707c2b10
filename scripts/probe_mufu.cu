// Throughput probe for the softmax exponential on sm_100a: ex2.approx.f32 vs the
// packed ex2.approx.ftz.bf16x2 / ex2.approx.f16x2 forms (results per SM per clock).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/probe_mufu scripts/probe_mufu.cu
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

constexpr int ITERS = 4096, CH = 8;

__global__ void k_f32(float* out, float seed, long long* clk) {
  float v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = seed * (threadIdx.x + c) * 1e-6f - 1.f;
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[c]));
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

__global__ void k_bf16x2(float* out, float seed, long long* clk) {
  unsigned v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    __nv_bfloat162 h = __floats2bfloat162_rn(seed * (threadIdx.x + c) * 1e-6f - 1.f, -0.5f);
    v[c] = *reinterpret_cast<unsigned*>(&h);
  }
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(v[c]));
  long long t1 = clock64();
  unsigned s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

__global__ void k_f16x2(float* out, float seed, long long* clk) {
  unsigned v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    __half2 h = __floats2half2_rn(seed * (threadIdx.x + c) * 1e-6f - 1.f, -0.5f);
    v[c] = *reinterpret_cast<unsigned*>(&h);
  }
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[c]));
  long long t1 = clock64();
  unsigned s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

// the softmax inner sequence per pair: f32x2 FMA (scale, -max) -> cvt bf16x2 -> ex2.bf16x2
__global__ void k_seq_bf16(float* out, float seed, long long* clk) {
  float a[CH], b[CH];
  unsigned acc = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) { a[c] = seed * (threadIdx.x + c) * 1e-6f - 1.f; b[c] = -0.25f * c; }
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      unsigned r;
      asm volatile("{\n .reg .b64 x, y;\n mov.b64 x, {%1, %2};\n fma.rn.f32x2 y, x, x, x;\n"
                   " .reg .f32 p, q;\n mov.b64 {p, q}, y;\n cvt.rn.bf16x2.f32 %0, q, p;\n"
                   " ex2.approx.ftz.bf16x2 %0, %0;\n}\n"
                   : "=r"(r) : "f"(a[c]), "f"(b[c]));
      acc ^= r;
    }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <typename K>
void run(const char* name, K kern, int elems_per_op) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 512, blocks = sms * 2;
  float* out;
  long long* clk;
  cudaMalloc(&out, sizeof(float) * threads * blocks);
  cudaMalloc(&clk, sizeof(long long) * blocks);
  kern<<<blocks, threads>>>(out, 1.f, clk);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(out, 1.f, clk);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c;
  cudaMemcpy(&c, clk, sizeof(c), cudaMemcpyDeviceToHost);
  const double ops = (double)threads * 2 * ITERS * CH;  // per SM (2 blocks per SM)
  printf("%-10s %8.3f ms  block clocks %lld  instr/clk/SM %.2f  elems/clk/SM %.2f  (err %s)\n", name, ms, c,
         ops / c, ops * elems_per_op / c, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
  cudaFree(clk);
}

int main() {
  run("f32", k_f32, 1);
  run("bf16x2", k_bf16x2, 2);
  run("f16x2", k_f16x2, 2);
  run("seq_bf16", k_seq_bf16, 2);
  return 0;
}
