// Associative-memory write path: the delta-rule fold of update_stack.
//
// Reference: armt/memory.py:94-125 (_delta_fold) driven by :155-180. For
// token i = 0..M-1 IN ORDER (token i sees tokens < i):
//   zq = z.phi_i ; nrm = phi_i.phi_i
//   vbar = |zq| <= eps ? 0 : (A phi_i) / zq ; gamma = nrm <= eps ? 0 : 1 - zq/nrm
//   A += beta_i (v_i - vbar) phi_i^T ; z += gamma phi_i
//
// The z chain never reads A, so it runs first (fold_prep, one CTA per member)
// and publishes zq_i and beta_i. Rows of A are then independent: fold_main
// holds rows of A in REGISTERS (8 lanes x float4 column chunks per row, two
// rows per lane group), keeps phi for all M tokens in shared memory, and per
// token does one 3-step shuffle reduction (8 rows per warp at once) and one
// axpy per row.
// A is read once and written once per fold (the HBM floor), fp32 throughout;
// the bf16 shadow of A used by the tensor-core retrieval is refreshed in the
// same pass.

#include "common.cuh"

namespace armt {
namespace fold {

constexpr int NJ_MAX = 16;  // d_phi <= 512

// phi rows are stored with a padded leading dimension (multiple of 32 floats,
// zero-filled) so the main fold reads them as aligned float4 without predicates.
__host__ __device__ inline int phi_ld(int dphi) { return (dphi + 31) / 32 * 32; }

struct Ws {
  float* phi;   // [G][M][phi_ld]
  float* zq;    // [G][M]
  float* beta;  // [G][M]
};

__host__ __device__ inline Ws carve(void* ws, int G, int M, int dphi) {
  float* f = reinterpret_cast<float*>(ws);
  Ws w;
  w.phi = f;
  w.zq = f + (long long)G * M * phi_ld(dphi);
  w.beta = w.zq + (long long)G * M;
  return w;
}

// ---------------------------------------------------------------------------
// fold_prep: one CTA per member.
//   1. r_i = [relu(k_i), relu(-k_i)] staged in smem (coalesced loads of k)
//   2. phi_i = DPFP(k_i) -> global workspace (read by fold_main), and
//      nrm_i = |phi_i|^2 in parallel (does not depend on the chain)
//   3. the z chain (armt/memory.py:101-106, 116-119, 124-125), one warp:
//      zq_i = z.phi_i ; gamma_i = nrm_i <= eps ? 0 : 1 - zq_i/nrm_i ; z += gamma_i phi_i
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) fold_prep_kernel(const __grid_constant__ ArmtMembers mem,
                                                        const float* __restrict__ kvb, long long ld_kvb,
                                                        long long kvb_stride, int k_off, int b_off,
                                                        float* __restrict__ z, int M, int d_mem, int nu, float eps,
                                                        Ws ws) {
  extern __shared__ float sm[];
  const int g = blockIdx.x;
  const int two_m = 2 * d_mem, dphi = two_m * nu, ldp = phi_ld(dphi);
  float* sr = sm;                    // [M][2m]
  float* snrm = sr + M * two_m;      // [M]
  const float* kv = kvb + (long long)g * kvb_stride;
  for (int e = threadIdx.x; e < M * d_mem; e += blockDim.x) {
    const int i = e / d_mem, c = e - i * d_mem;
    const float k = kv[(long long)i * ld_kvb + k_off + c];
    sr[i * two_m + c] = fmaxf(k, 0.f);
    sr[i * two_m + d_mem + c] = fmaxf(-k, 0.f);
  }
  for (int i = threadIdx.x; i < M; i += blockDim.x)
    ws.beta[(long long)g * M + i] = sigmoid_ref(kv[(long long)i * ld_kvb + b_off]);
  __syncthreads();
  // phi element c of token i: r[ii] * r[(ii + j) mod 2m], j = c / 2m + 1, ii = c mod 2m.
  // Each lane owns columns c = lane + 32*jj; its (ii, partner) index pairs are
  // tabulated once in registers.
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int ia[NJ_MAX], ib[NJ_MAX];
#pragma unroll
  for (int jj = 0; jj < NJ_MAX; ++jj) {
    const int c = lane + 32 * jj;
    if (c < dphi) {
      const int j = c / two_m + 1, ii = c - (j - 1) * two_m;
      ia[jj] = ii;
      ib[jj] = (ii + j) % two_m;
    } else {
      ia[jj] = -1;
      ib[jj] = 0;
    }
  }
  auto load_phi = [&](int i, float (&p)[NJ_MAX]) {
#pragma unroll
    for (int jj = 0; jj < NJ_MAX; ++jj)
      p[jj] = (i < M && ia[jj] >= 0) ? sr[i * two_m + ia[jj]] * sr[i * two_m + ib[jj]] : 0.f;
  };
  float* gphi = ws.phi + (long long)g * M * ldp;
  const int nwarps = blockDim.x >> 5;
  for (int i = warp; i < M; i += nwarps) {
    float p[NJ_MAX];
    load_phi(i, p);
    float acc = 0.f;
#pragma unroll
    for (int jj = 0; jj < NJ_MAX; ++jj) {
      const int c = lane + 32 * jj;
      if (c < ldp) gphi[(long long)i * ldp + c] = p[jj];
      acc = fmaf(p[jj], p[jj], acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) snrm[i] = acc;
  }
  __syncthreads();
  if (warp != 0) return;
  // z chain in blocks of 4 tokens: with z_i the state before token i,
  //   zq_{i+t} = z_i.phi_{i+t} + sum_{s<t} gamma_{i+s} (phi_{i+s}.phi_{i+t}),
  // so one interleaved shuffle reduction of 4 dots + 6 Gram entries serves 4 tokens.
  float* zl = z + (long long)mem.layer[g] * dphi;
  float zr[NJ_MAX];
#pragma unroll
  for (int jj = 0; jj < NJ_MAX; ++jj) {
    const int c = lane + 32 * jj;
    zr[jj] = c < dphi ? zl[c] : 0.f;
  }
  for (int i0 = 0; i0 < M; i0 += 4) {
    float p[4][NJ_MAX];
#pragma unroll
    for (int t = 0; t < 4; ++t) load_phi(i0 + t, p[t]);
    float red[10];
#pragma unroll
    for (int t = 0; t < 10; ++t) red[t] = 0.f;
#pragma unroll
    for (int jj = 0; jj < NJ_MAX; ++jj) {
      red[0] = fmaf(zr[jj], p[0][jj], red[0]);
      red[1] = fmaf(zr[jj], p[1][jj], red[1]);
      red[2] = fmaf(zr[jj], p[2][jj], red[2]);
      red[3] = fmaf(zr[jj], p[3][jj], red[3]);
      red[4] = fmaf(p[0][jj], p[1][jj], red[4]);
      red[5] = fmaf(p[0][jj], p[2][jj], red[5]);
      red[6] = fmaf(p[0][jj], p[3][jj], red[6]);
      red[7] = fmaf(p[1][jj], p[2][jj], red[7]);
      red[8] = fmaf(p[1][jj], p[3][jj], red[8]);
      red[9] = fmaf(p[2][jj], p[3][jj], red[9]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int t = 0; t < 10; ++t) red[t] += __shfl_xor_sync(0xffffffffu, red[t], o);
    // K[s][t] for s < t
    const float K01 = red[4], K02 = red[5], K03 = red[6], K12 = red[7], K13 = red[8], K23 = red[9];
    float gam[4], zq[4];
    zq[0] = red[0];
    gam[0] = (i0 < M && snrm[i0] > eps) ? 1.f - zq[0] / snrm[i0] : 0.f;
    zq[1] = red[1] + gam[0] * K01;
    gam[1] = (i0 + 1 < M && snrm[i0 + 1] > eps) ? 1.f - zq[1] / snrm[i0 + 1] : 0.f;
    zq[2] = red[2] + gam[0] * K02 + gam[1] * K12;
    gam[2] = (i0 + 2 < M && snrm[i0 + 2] > eps) ? 1.f - zq[2] / snrm[i0 + 2] : 0.f;
    zq[3] = red[3] + gam[0] * K03 + gam[1] * K13 + gam[2] * K23;
    gam[3] = (i0 + 3 < M && snrm[i0 + 3] > eps) ? 1.f - zq[3] / snrm[i0 + 3] : 0.f;
#pragma unroll
    for (int jj = 0; jj < NJ_MAX; ++jj)
      zr[jj] = fmaf(gam[3], p[3][jj], fmaf(gam[2], p[2][jj], fmaf(gam[1], p[1][jj], fmaf(gam[0], p[0][jj], zr[jj]))));
    if (lane < 4 && i0 + lane < M)
      ws.zq[(long long)g * M + i0 + lane] = lane == 0 ? zq[0] : lane == 1 ? zq[1] : lane == 2 ? zq[2] : zq[3];
  }
#pragma unroll
  for (int jj = 0; jj < NJ_MAX; ++jj) {
    const int c = lane + 32 * jj;
    if (c < dphi) zl[c] = zr[jj];
  }
}

// ---------------------------------------------------------------------------
// fold_main: rows of A are independent given (zq_i, beta_i, phi_i).
// A group of 8 lanes owns TWO rows; lane q of the group holds float4 column
// chunks q, q+8, q+16, ... of both rows in registers (2 x NJ4 float4). One
// warp = 8 rows: each float4 of phi read from shared memory (broadcast over
// the 4 groups) feeds 8 FMAs, and one 3-step shuffle tree reduces 8 row-dots.
// ---------------------------------------------------------------------------
template <int NJ4>
__global__ void __launch_bounds__(256, 1) fold_main_kernel(const __grid_constant__ ArmtMembers mem,
                                                           const float* __restrict__ kvb, long long ld_kvb,
                                                           long long kvb_stride, int v_off, float* __restrict__ A,
                                                           __nv_bfloat16* __restrict__ shadow, long long ld_shadow,
                                                           int d, int M, int dphi, float eps, Ws ws) {
  constexpr int LDP = 32 * NJ4;             // padded phi row (floats)
  constexpr int R = 64;                     // rows per CTA (8 warps x 8 rows)
  extern __shared__ __align__(16) float sm[];
  float* sphi = sm;                         // [M][LDP]
  float* sv = sphi + M * LDP;               // [M][R]
  float* szq = sv + M * R;                  // [M]
  float* sbeta = szq + M;                   // [M]
  const int g = blockIdx.y;
  const int row0 = blockIdx.x * R;
  const float4* gphi = reinterpret_cast<const float4*>(ws.phi + (long long)g * M * phi_ld(dphi));
  float4* sphi4 = reinterpret_cast<float4*>(sphi);
  for (int e = threadIdx.x; e < M * LDP / 4; e += blockDim.x) sphi4[e] = gphi[e];
  const float* kv = kvb + (long long)g * kvb_stride;
  for (int e = threadIdx.x; e < M * R; e += blockDim.x) {
    const int i = e / R, rr = e - i * R;
    sv[e] = row0 + rr < d ? kv[(long long)i * ld_kvb + v_off + row0 + rr] : 0.f;
  }
  for (int i = threadIdx.x; i < M; i += blockDim.x) {
    szq[i] = ws.zq[(long long)g * M + i];
    sbeta[i] = ws.beta[(long long)g * M + i];
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane >> 3, q = lane & 7;
  const int rl0 = warp * 8 + grp * 2;       // local rows rl0, rl0 + 1
  const int layer = mem.layer[g];
  float* Al = A + (long long)layer * d * dphi;
  float4 a0[NJ4], a1[NJ4];
#pragma unroll
  for (int j = 0; j < NJ4; ++j) {
    const int c = 4 * (q + 8 * j);
    float t0[4], t1[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const bool cv = c + e < dphi;
      t0[e] = (cv && row0 + rl0 < d) ? Al[(long long)(row0 + rl0) * dphi + c + e] : 0.f;
      t1[e] = (cv && row0 + rl0 + 1 < d) ? Al[(long long)(row0 + rl0 + 1) * dphi + c + e] : 0.f;
    }
    a0[j] = make_float4(t0[0], t0[1], t0[2], t0[3]);
    a1[j] = make_float4(t1[0], t1[1], t1[2], t1[3]);
  }
  for (int i = 0; i < M; ++i) {
    const float4* prow = sphi4 + i * (LDP / 4) + q;
    float s0 = 0.f, s1 = 0.f, u0 = 0.f, u1 = 0.f;
#pragma unroll
    for (int j = 0; j < NJ4; ++j) {
      const float4 pj = prow[8 * j];
      s0 = fmaf(a0[j].x, pj.x, s0); s1 = fmaf(a0[j].y, pj.y, s1);
      s0 = fmaf(a0[j].z, pj.z, s0); s1 = fmaf(a0[j].w, pj.w, s1);
      u0 = fmaf(a1[j].x, pj.x, u0); u1 = fmaf(a1[j].y, pj.y, u1);
      u0 = fmaf(a1[j].z, pj.z, u0); u1 = fmaf(a1[j].w, pj.w, u1);
    }
    float sa = s0 + s1, sb = u0 + u1;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      sa += __shfl_xor_sync(0xffffffffu, sa, o);
      sb += __shfl_xor_sync(0xffffffffu, sb, o);
    }
    const float zq = szq[i];
    const bool guarded = fabsf(zq) <= eps;
    const float beta = sbeta[i];
    const float ca = beta * (sv[i * R + rl0] - (guarded ? 0.f : sa / zq));
    const float cb = beta * (sv[i * R + rl0 + 1] - (guarded ? 0.f : sb / zq));
#pragma unroll
    for (int j = 0; j < NJ4; ++j) {
      const float4 pj = prow[8 * j];  // re-read (smem broadcast) rather than hold NJ4 float4 live
      a0[j].x = fmaf(ca, pj.x, a0[j].x); a0[j].y = fmaf(ca, pj.y, a0[j].y);
      a0[j].z = fmaf(ca, pj.z, a0[j].z); a0[j].w = fmaf(ca, pj.w, a0[j].w);
      a1[j].x = fmaf(cb, pj.x, a1[j].x); a1[j].y = fmaf(cb, pj.y, a1[j].y);
      a1[j].z = fmaf(cb, pj.z, a1[j].z); a1[j].w = fmaf(cb, pj.w, a1[j].w);
    }
  }
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int row = row0 + rl0 + rr;
    if (row >= d) continue;
    float* Ar = Al + (long long)row * dphi;
    __nv_bfloat16* sh = shadow ? shadow + ((long long)layer * d + row) * ld_shadow : nullptr;
#pragma unroll
    for (int j = 0; j < NJ4; ++j) {
      const int c = 4 * (q + 8 * j);
      const float4 v = rr ? a1[j] : a0[j];
      const float t[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (c + e < dphi) {
          Ar[c + e] = t[e];
          if (sh) sh[c + e] = __float2bfloat16_rn(t[e]);
        }
    }
  }
}

template <int NJ4>
static int launch_main(const ArmtMembers& mem, const float* kvb, long long ld_kvb, long long kvb_stride, int v_off,
                       float* A, __nv_bfloat16* shadow, long long ld_shadow, int d, int M, int dphi, float eps, Ws ws,
                       cudaStream_t s) {
  constexpr int R = 64;
  const size_t smem = sizeof(float) * ((size_t)M * 32 * NJ4 + (size_t)M * R + 2 * (size_t)M);
  ARMT_REQUIRE(smem <= 227 * 1024, ARMT_ERR_UNSUPPORTED, "fold: M*d_phi too large for shared memory (%zu B)", smem);
  auto kern = fold_main_kernel<NJ4>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((d + R - 1) / R, mem.G);
  kern<<<grid, 256, smem, s>>>(mem, kvb, ld_kvb, kvb_stride, v_off, A, shadow, ld_shadow, d, M, dphi, eps, ws);
  ARMT_CHECK_LAUNCH("fold_main");
  return ARMT_OK;
}

static int dispatch_main(int dphi, const ArmtMembers& mem, const float* kvb, long long ld_kvb, long long kvb_stride,
                         int v_off, float* A, __nv_bfloat16* shadow, long long ld_shadow, int d, int M, float eps,
                         Ws ws, cudaStream_t s) {
  const int nj4 = (dphi + 31) / 32;
#define ARMT_FOLD_NJ(N) \
  if (nj4 <= N) return launch_main<N>(mem, kvb, ld_kvb, kvb_stride, v_off, A, shadow, ld_shadow, d, M, dphi, eps, ws, s);
  ARMT_FOLD_NJ(1) ARMT_FOLD_NJ(2) ARMT_FOLD_NJ(3) ARMT_FOLD_NJ(4) ARMT_FOLD_NJ(6) ARMT_FOLD_NJ(8)
  ARMT_FOLD_NJ(12) ARMT_FOLD_NJ(16)
#undef ARMT_FOLD_NJ
  set_error("fold: d_phi=%d exceeds %d", dphi, 32 * NJ_MAX);
  return ARMT_ERR_UNSUPPORTED;
}

}  // namespace fold
}  // namespace armt

using namespace armt;

extern "C" long long armt_fold_workspace_bytes(int G, int n_mem, int d_phi) {
  return (long long)sizeof(float) * G * n_mem * (armt::fold::phi_ld(d_phi) + 2);
}

extern "C" int armt_mem_fold(const ArmtMembers* mem, const float* kvb, long long ld_kvb, long long kvb_stride,
                             int v_off, int k_off, int b_off, float* A, float* z, void* A_shadow, long long ld_shadow,
                             int d, int n_mem, int d_mem, int nu, float eps, void* ws, void* stream) {
  using namespace armt::fold;
  ARMT_REQUIRE(mem && mem->G >= 1 && mem->G <= ARMT_MAX_MEMBERS, ARMT_ERR_DIM, "fold: bad member count");
  ARMT_REQUIRE(kvb && A && z && ws, ARMT_ERR_INPUT, "fold: null pointer");
  ARMT_REQUIRE(nu >= 1 && d_mem >= 1 && d >= 1, ARMT_ERR_DIM, "fold: bad sizes");
  if (n_mem == 0) return ARMT_OK;
  for (int g = 0; g < mem->G; ++g)
    for (int h = g + 1; h < mem->G; ++h)
      ARMT_REQUIRE(mem->layer[g] != mem->layer[h], ARMT_ERR_INPUT,
                   "fold: duplicate layer %d in one group (two writers per memory slot)", mem->layer[g]);
  const int dphi = 2 * nu * d_mem;
  ARMT_REQUIRE(dphi <= 32 * NJ_MAX, ARMT_ERR_UNSUPPORTED, "fold: d_phi=%d > %d", dphi, 32 * NJ_MAX);
  cudaStream_t s = as_stream(stream);
  Ws w = carve(ws, mem->G, n_mem, dphi);
  const size_t prep_smem = sizeof(float) * ((size_t)n_mem * 2 * d_mem + n_mem);
  ARMT_REQUIRE(prep_smem <= 227 * 1024, ARMT_ERR_UNSUPPORTED, "fold: M*d_phi too large");
  cudaFuncSetAttribute(fold_prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)prep_smem);
  fold_prep_kernel<<<mem->G, 256, prep_smem, s>>>(*mem, kvb, ld_kvb, kvb_stride, k_off, b_off, z, n_mem, d_mem, nu,
                                                   eps, w);
  ARMT_CHECK_LAUNCH("fold_prep");
  return dispatch_main(dphi, *mem, kvb, ld_kvb, kvb_stride, v_off, A, reinterpret_cast<__nv_bfloat16*>(A_shadow),
                       ld_shadow, d, n_mem, eps, w, s);
}
