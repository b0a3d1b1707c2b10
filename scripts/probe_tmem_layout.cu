// Probe: which (row, column) of a TMEM tile does each thread receive from
// tcgen05.ld.16x256b / 16x128b? Rows are written with the known 32x32b layout
// (thread = lane = row), value = row * 1000 + col, then read back with the other
// shapes. Build: nvcc -gencode arch=compute_100a,code=sm_100a -o probe probe_tmem_layout.cu
#include <cstdio>
#include <cstdint>

__global__ void probe(float* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot + ((uint32_t)(warp * 32) << 16);
  const int row = warp * 32 + lane;
  uint32_t v[8];
  for (int j = 0; j < 8; ++j) v[j] = __float_as_uint(row * 1000.f + j);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(base), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(base));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int j = 0; j < 4; ++j) out[threadIdx.x * 8 + j] = __uint_as_float(r[j]);
  uint32_t s[2];
  asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0,%1}, [%2];" : "=r"(s[0]), "=r"(s[1]) : "r"(base));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int j = 0; j < 2; ++j) out[threadIdx.x * 8 + 4 + j] = __uint_as_float(s[j]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(slot));
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 8 * 4);
  probe<<<1, 128>>>(d);
  float h[128 * 8];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  for (int t = 0; t < 64; ++t) {
    printf("t%3d 16x256b:", t);
    for (int j = 0; j < 4; ++j) printf(" (%d,%d)", (int)h[t * 8 + j] / 1000, (int)h[t * 8 + j] % 1000);
    printf("  16x128b:");
    for (int j = 4; j < 6; ++j) printf(" (%d,%d)", (int)h[t * 8 + j] / 1000, (int)h[t * 8 + j] % 1000);
    printf("\n");
  }
  return 0;
}
