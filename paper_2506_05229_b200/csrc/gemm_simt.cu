// fp32 SIMT grouped GEMM: the "f32" parity mode of armt_gemm.
//
// tcgen05 has no full-fp32 MMA (tf32 keeps 10 mantissa bits), so the 1e-4
// parity mode runs every projection on FP32 FMA pipes. Same member tables and
// epilogues (STORE / RESIDUAL / RETRIEVE) as the tensor-core path; RoPE and
// SwiGLU run as separate kernels in this mode.
//
// C[m, n] = sum_k A[m, k] * B[n, k]   (A and B both K-major)
// Tile 64 x 64 x 16, 256 threads, 4 x 4 register micro-tile per thread.

#include "common.cuh"

namespace armt {
namespace simt {

constexpr int TM = 64, TN = 64, TK = 16;

struct Params {
  int M, N, K;
  const float* A; long long lda, a_stride;
  const float* B; long long ldb, b_stride;
  void* C; long long ldc, c_stride; int c_dtype;
  int epi;
  const float* R; long long ldr, r_stride;
  __nv_bfloat16* C2; long long ldc2, c2_stride;
  const float* den; long long den_stride; float eps;
  int a_slot[ARMT_MAX_MEMBERS];
  int b_index[ARMT_MAX_MEMBERS];
  int c_slot[ARMT_MAX_MEMBERS];
};

__global__ void __launch_bounds__(256) gemm_f32_kernel(const __grid_constant__ Params p) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  const int g = blockIdx.z;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  const float* A = p.A + (long long)p.a_slot[g] * p.a_stride;
  const float* B = p.B + (long long)p.b_index[g] * p.b_stride;
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;  // 16 x 16 threads, 4 x 4 outputs each
  float acc[4][4] = {};
  // loader: 64 rows x 16 k -> each thread 4 elements (row = tid/4, k = (tid%4)*4..+3)
  const int lr = tid >> 2, lk = (tid & 3) * 4;
  for (int k0 = 0; k0 < p.K; k0 += TK) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = k0 + lk + j;
      const int am = m0 + lr, bn = n0 + lr;
      As[lk + j][lr] = (am < p.M && k < p.K) ? A[(long long)am * p.lda + k] : 0.f;
      Bs[lk + j][lr] = (bn < p.N && k < p.K) ? B[(long long)bn * p.ldb + k] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  const int cs = p.c_slot[g];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= p.M) continue;
    float den = 1.f;
    if (p.epi == ARMT_EPI_RETRIEVE) den = p.den[(long long)g * p.den_stride + m];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= p.N) continue;
      float v = acc[i][j];
      const long long off = (long long)cs * p.c_stride + (long long)m * p.ldc + n;
      if (p.epi == ARMT_EPI_RESIDUAL || p.epi == ARMT_EPI_RETRIEVE) {
        const float r = p.R[(long long)cs * p.r_stride + (long long)m * p.ldr + n];
        if (p.epi == ARMT_EPI_RETRIEVE) v = r + (fabsf(den) <= p.eps ? 0.f : v / den);
        else v = r + v;
        reinterpret_cast<float*>(p.C)[off] = v;
        if (p.epi == ARMT_EPI_RESIDUAL && p.C2)
          p.C2[(long long)cs * p.c2_stride + (long long)m * p.ldc2 + n] = __float2bfloat16_rn(v);
      } else {
        store_from_f32(p.C, p.c_dtype, off, v);
      }
    }
  }
}

}  // namespace simt

int gemm_simt(const ArmtGemmArgs& a, cudaStream_t s) {
  using namespace simt;
  ARMT_REQUIRE(a.epilogue == ARMT_EPI_STORE || a.epilogue == ARMT_EPI_RESIDUAL ||
                   a.epilogue == ARMT_EPI_RETRIEVE,
               ARMT_ERR_UNSUPPORTED, "f32 GEMM fuses only STORE/RESIDUAL/RETRIEVE epilogues");
  Params p;
  memset(&p, 0, sizeof(p));
  p.M = a.M; p.N = a.N; p.K = a.K;
  p.A = reinterpret_cast<const float*>(a.A); p.lda = a.lda; p.a_stride = a.a_stride;
  p.B = reinterpret_cast<const float*>(a.B); p.ldb = a.ldb; p.b_stride = a.b_stride;
  p.C = a.C; p.ldc = a.ldc; p.c_stride = a.c_stride; p.c_dtype = a.c_dtype;
  p.epi = a.epilogue;
  p.R = a.R; p.ldr = a.ldr; p.r_stride = a.r_stride;
  p.C2 = reinterpret_cast<__nv_bfloat16*>(a.C2); p.ldc2 = a.ldc2; p.c2_stride = a.c2_stride;
  p.den = a.den; p.den_stride = a.den_stride; p.eps = a.eps;
  for (int g = 0; g < a.G; ++g) {
    p.a_slot[g] = a.a_slot[g]; p.b_index[g] = a.b_index[g]; p.c_slot[g] = a.c_slot[g];
  }
  dim3 grid((a.N + TN - 1) / TN, (a.M + TM - 1) / TM, a.G);
  gemm_f32_kernel<<<grid, 256, 0, s>>>(p);
  ARMT_CHECK_LAUNCH("f32 gemm launch");
  return ARMT_OK;
}

int gemm_tc(const ArmtGemmArgs& a, cudaStream_t s);

}  // namespace armt

extern "C" int armt_gemm(const ArmtGemmArgs* a, void* stream) {
  using namespace armt;
  ARMT_REQUIRE(a != nullptr, ARMT_ERR_INPUT, "null args");
  ARMT_REQUIRE(a->G >= 1 && a->G <= ARMT_MAX_MEMBERS, ARMT_ERR_DIM, "G=%d out of range 1..%d", a->G,
               ARMT_MAX_MEMBERS);
  ARMT_REQUIRE(a->M >= 1 && a->N >= 1 && a->K >= 1, ARMT_ERR_DIM, "empty GEMM %dx%dx%d", a->M, a->N, a->K);
  ARMT_REQUIRE(a->A && a->B && a->C, ARMT_ERR_INPUT, "null operand");
  if ((a->epilogue == ARMT_EPI_RESIDUAL || a->epilogue == ARMT_EPI_RETRIEVE))
    ARMT_REQUIRE(a->R != nullptr && a->c_dtype == ARMT_F32, ARMT_ERR_INPUT,
                 "residual epilogues need R and an f32 C");
  if (a->epilogue == ARMT_EPI_RETRIEVE) ARMT_REQUIRE(a->den != nullptr, ARMT_ERR_INPUT, "RETRIEVE needs den");
  if (a->epilogue == ARMT_EPI_ROPE)
    ARMT_REQUIRE(a->rope_cos && a->rope_sin && a->head_dim > 0 && a->head_dim % 2 == 0, ARMT_ERR_INPUT,
                 "ROPE needs tables and an even head_dim");
  for (int g = 0; g < a->G; ++g)
    ARMT_REQUIRE(a->a_slot[g] >= 0 && a->b_index[g] >= 0 && a->c_slot[g] >= 0 && a->a_slot[g] < 32768 &&
                     a->b_index[g] < 32768 && a->c_slot[g] < 32768,
                 ARMT_ERR_INPUT, "member %d has a bad slot/layer index", g);
  cudaStream_t s = as_stream(stream);
  if (a->ab_dtype == ARMT_BF16) return gemm_tc(*a, s);
  if (a->ab_dtype == ARMT_F32) return gemm_simt(*a, s);
  set_error("unknown operand dtype %d", a->ab_dtype);
  return ARMT_ERR_INPUT;
}
