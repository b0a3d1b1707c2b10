// Row-wise kernels of the ARMT cell: embedding gather, RMSNorm, RoPE, SwiGLU,
// DPFP feature map + retrieval denominator, casts, next-token NLL.
// All are HBM-bound; one warp per row, fp32 math, coalesced along the row.

#include <stdarg.h>
#include <stddef.h>
#include <mutex>
#include "common.cuh"

namespace armt {

// ------------------------------------------------------------------ runtime glue
static thread_local char g_err[1024] = "";
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
std::atomic<long long>& launch_counter() {
  static std::atomic<long long> c{0};
  return c;
}
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("ARMT_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

int num_sms() {
  static int n = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  });
  return n;
}

// ------------------------------------------------------------------ embed
// armt/layers.py:306-318: rows [0, seg) from the embedding table, rows
// [seg, seg+M) from mem_embedding (memory rows last).
// Ids outside [0, vocab) never index the table: their row is written as zeros
// and counted in g_bad_ids (armt_embed_bad_ids), so a bad id cannot fault or
// read foreign memory inside a captured graph; the Python layer validates ids
// before launch and raises InputError like the reference (armt/layers.py:311-315).
__device__ unsigned int g_bad_ids = 0;

__global__ void embed_kernel(const long long* __restrict__ ids, const void* emb, const void* mem_emb,
                             int w_dtype, float* __restrict__ x, __nv_bfloat16* __restrict__ x_bf,
                             int seg, int n_mem, int d, int vocab) {
  const int row = blockIdx.x;
  const void* src;
  long long src_row;
  if (row < seg) { src = emb; src_row = ids[row]; }
  else { src = mem_emb; src_row = row - seg; }
  const bool bad = row < seg && (src_row < 0 || src_row >= vocab);
  if (bad && threadIdx.x == 0) atomicAdd(&g_bad_ids, 1u);
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    const float v = bad ? 0.f : load_as_f32(src, w_dtype, src_row * d + c);
    x[(long long)row * d + c] = v;
    if (x_bf) x_bf[(long long)row * d + c] = __float2bfloat16_rn(v);
  }
}

// ------------------------------------------------------------------ RMSNorm
// armt/tensor_ops.py:267-281: x / sqrt(mean(x^2) + eps) * gain.
template <typename OutT>
__global__ void rmsnorm_kernel(const __grid_constant__ ArmtMembers mem, const float* __restrict__ x,
                               long long x_stride, const float* __restrict__ gain, OutT* __restrict__ out,
                               long long out_stride, int rows, int d, float eps) {
  const int g = blockIdx.y;
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* xr = x + (long long)mem.slot[g] * x_stride + (long long)row * d;
  const float* gr = gain + (long long)mem.layer[g] * d;
  float ss = 0.f;
  for (int c = lane; c < d; c += 32) ss = fmaf(xr[c], xr[c], ss);
  ss = warp_sum(ss);
  const float denom = sqrtf(ss / (float)d + eps);
  OutT* o = out + (long long)g * out_stride + (long long)row * d;
  for (int c = lane; c < d; c += 32) o[c] = from_f32<OutT>(xr[c] / denom * gr[c]);
}

// ------------------------------------------------------------------ RoPE (f32 mode)
// armt/layers.py:169-176 on the q and k column blocks of a (T, 3d) qkv row.
template <typename T>
__global__ void rope_kernel(T* qkv, long long ld, long long stride, int rows, int n_heads, int dh,
                            const float* __restrict__ cos_t, const float* __restrict__ sin_t) {
  const int g = blockIdx.y;
  const int row = blockIdx.x;
  const int half = dh / 2;
  const int d = n_heads * dh;
  T* r = qkv + (long long)g * stride + (long long)row * ld;
  // pairs: 2 sections (q, k) x n_heads x half
  for (int e = threadIdx.x; e < 2 * n_heads * half; e += blockDim.x) {
    const int sec = e / (n_heads * half);
    const int rem = e - sec * n_heads * half;
    const int h = rem / half, i = rem - h * half;
    T* base = r + sec * d + h * dh;
    const float a = to_f32(base[i]), b = to_f32(base[i + half]);
    const float c = cos_t[(long long)row * half + i], s = sin_t[(long long)row * half + i];
    base[i] = from_f32<T>(a * c - b * s);
    base[i + half] = from_f32<T>(b * c + a * s);
  }
}

// ------------------------------------------------------------------ SwiGLU (f32 mode)
// armt/layers.py:228-232 over block-interleaved [gate | up] columns.
template <typename T>
__global__ void swiglu_kernel(const T* gu, long long ld_gu, long long gu_stride, T* out, long long ld_out,
                              long long out_stride, int d_ff, int block) {
  const int g = blockIdx.y, row = blockIdx.x;
  const T* src = gu + (long long)g * gu_stride + (long long)row * ld_gu;
  T* dst = out + (long long)g * out_stride + (long long)row * ld_out;
  for (int j = threadIdx.x; j < d_ff; j += blockDim.x) {
    const int t = j / block, c = j - t * block;
    const float gate = to_f32(src[(long long)t * 2 * block + c]);
    const float up = to_f32(src[(long long)t * 2 * block + block + c]);
    dst[j] = from_f32<T>(silu_ref(gate) * up);
  }
}

// ------------------------------------------------------------------ DPFP + den
// armt/memory.py:34-45 (feature map) and :145-147 (den = phi . z[layer]).
// out[(j-1)*2m + i] = r[i] * r[(i+j) mod 2m], r = [relu(q), relu(-q)].
template <typename PhiT>
__global__ void dpfp_den_kernel(const __grid_constant__ ArmtMembers mem, const float* __restrict__ q,
                                long long q_stride, const float* __restrict__ z, PhiT* __restrict__ phi,
                                long long ld_phi, long long phi_stride, float* __restrict__ den,
                                long long den_stride, int rows, int d_mem, int nu) {
  const int g = blockIdx.y;
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* qr = q + (long long)g * q_stride + (long long)row * d_mem;
  const float* zr = z + (long long)mem.layer[g] * (2 * nu * d_mem);
  PhiT* pr = phi + (long long)g * phi_stride + (long long)row * ld_phi;
  const int two_m = 2 * d_mem, dphi = two_m * nu;
  float acc = 0.f;
  for (int c = lane; c < ld_phi; c += 32) {
    float v = 0.f;
    if (c < dphi) {
      const int j = c / two_m + 1, i = c - (j - 1) * two_m;
      const int i2 = (i + j) % two_m;
      const float a = i < d_mem ? fmaxf(qr[i], 0.f) : fmaxf(-qr[i - d_mem], 0.f);
      const float b = i2 < d_mem ? fmaxf(qr[i2], 0.f) : fmaxf(-qr[i2 - d_mem], 0.f);
      v = a * b;
      acc = fmaf(v, zr[c], acc);
    }
    pr[c] = from_f32<PhiT>(v);
  }
  acc = warp_sum(acc);
  if (lane == 0) den[(long long)g * den_stride + row] = acc;
}

// ------------------------------------------------------------------ cast
template <typename S, typename D>
__global__ void cast_kernel(const S* __restrict__ src, D* __restrict__ dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = from_f32<D>(to_f32(src[i]));
}

// ------------------------------------------------------------------ NLL
// One CTA per row: single pass of online log-sum-exp over 16-byte vectors.
__device__ __forceinline__ void lse_merge(float& m, float& s, float m2, float s2) {
  const float mn = fmaxf(m, m2);
  s = (m == -INFINITY ? 0.f : s * __expf(m - mn)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mn));
  m = mn;
}

template <typename T>
__global__ void __launch_bounds__(256) nll_kernel(const T* __restrict__ logits, long long ld,
                                                  const long long* __restrict__ tgt, float* __restrict__ nll,
                                                  int vocab) {
  constexpr int VEC = 16 / sizeof(T);
  const long long row = blockIdx.x;
  const T* r = logits + row * ld;
  float m = -INFINITY, s = 0.f;
  const bool aligned = ((reinterpret_cast<uintptr_t>(r) & 15) == 0);
  const int nvec = aligned ? vocab / VEC : 0;
  for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
    uint4 raw;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(raw.x), "=r"(raw.y), "=r"(raw.z), "=r"(raw.w) : "l"(reinterpret_cast<const uint4*>(r) + v));
    const T* e = reinterpret_cast<const T*>(&raw);
    float bm = to_f32(e[0]);
#pragma unroll
    for (int j = 1; j < VEC; ++j) bm = fmaxf(bm, to_f32(e[j]));
    float bs = 0.f;
#pragma unroll
    for (int j = 0; j < VEC; ++j) bs += __expf(to_f32(e[j]) - bm);
    lse_merge(m, s, bm, bs);
  }
  for (int c = nvec * VEC + threadIdx.x; c < vocab; c += blockDim.x) lse_merge(m, s, to_f32(r[c]), 1.f);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    lse_merge(m, s, m2, s2);
  }
  __shared__ float sm_m[8], sm_s[8];
  if ((threadIdx.x & 31) == 0) { sm_m[threadIdx.x >> 5] = m; sm_s[threadIdx.x >> 5] = s; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = sm_m[0], S = sm_s[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) lse_merge(M, S, sm_m[w], sm_s[w]);
    nll[row] = M + logf(S) - to_f32(r[tgt[row]]);
  }
}

// Fused-NLL finalize: combine the per-tile (max, sum 2^x) partials of each row.
__global__ void lse_finalize_kernel(const float2* __restrict__ part, long long ld, int n_tiles,
                                    const float* __restrict__ tgt, const long long* __restrict__ targets,
                                    float* __restrict__ nll, long long rows) {
  const long long row = blockIdx.x * (long long)(blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float2* pr = part + row * ld;
  float M = -INFINITY;
  for (int t = lane; t < n_tiles; t += 32) M = fmaxf(M, pr[t].x);
  M = warp_max(M);
  float S = 0.f;
  for (int t = lane; t < n_tiles; t += 32) {
    const float2 q = pr[t];
    S += q.y * exp2f(q.x - M);
  }
  S = warp_sum(S);
  if (lane == 0) nll[row] = targets[row] < 0 ? 0.f : 0.6931471805599453f * (M + log2f(S) - tgt[row]);
}

// (max, sum 2^(x - max)) of a row's n_tiles partials -> one partial per row
// (vocab-parallel LM head: each rank reduces its block before the all-gather)
__global__ void lse_reduce_kernel(const float2* __restrict__ part, long long ld, int n_tiles,
                                  float2* __restrict__ out, long long rows) {
  const long long row = blockIdx.x * (long long)(blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float2* pr = part + row * ld;
  float M = -INFINITY;
  for (int t = lane; t < n_tiles; t += 32) M = fmaxf(M, pr[t].x);
  M = warp_max(M);
  float S = 0.f;
  if (M != -INFINITY)
    for (int t = lane; t < n_tiles; t += 32) {
      const float2 q = pr[t];
      S += q.y * exp2f(q.x - M);
    }
  S = warp_sum(S);
  if (lane == 0) out[row] = make_float2(M, S);
}

}  // namespace armt

using namespace armt;

extern "C" {

int armt_embed(const long long* ids, const void* emb, const void* mem_emb, int w_dtype, float* x, void* x_bf,
               int seg, int n_mem, int d, int vocab, void* stream) {
  ARMT_REQUIRE(ids && emb && mem_emb && x, ARMT_ERR_INPUT, "embed: null pointer");
  ARMT_REQUIRE(seg >= 1 && n_mem >= 0 && d >= 1 && vocab >= 1, ARMT_ERR_DIM, "embed: bad sizes");
  embed_kernel<<<seg + n_mem, 128, 0, as_stream(stream)>>>(ids, emb, mem_emb, w_dtype, x,
                                                           reinterpret_cast<__nv_bfloat16*>(x_bf), seg, n_mem, d,
                                                           vocab);
  ARMT_CHECK_LAUNCH("embed");
  return ARMT_OK;
}

long long armt_embed_bad_ids(int reset) {
  unsigned int n = 0;
  if (cudaMemcpyFromSymbol(&n, g_bad_ids, sizeof(n)) != cudaSuccess) return -1;
  if (reset) {
    const unsigned int zero = 0;
    if (cudaMemcpyToSymbol(g_bad_ids, &zero, sizeof(zero)) != cudaSuccess) return -1;
  }
  return (long long)n;
}

int armt_rmsnorm(const ArmtMembers* mem, const float* x, long long x_stride, const float* gain, void* out,
                 int out_dtype, long long out_stride, int rows, int d, float eps, void* stream) {
  ARMT_REQUIRE(mem && mem->G >= 1 && mem->G <= ARMT_MAX_MEMBERS, ARMT_ERR_DIM, "rmsnorm: bad member count");
  ARMT_REQUIRE(rows >= 1 && d >= 1, ARMT_ERR_DIM, "rmsnorm: bad sizes");
  dim3 grid((rows + 7) / 8, mem->G);
  if (out_dtype == ARMT_BF16)
    rmsnorm_kernel<__nv_bfloat16><<<grid, 256, 0, as_stream(stream)>>>(
        *mem, x, x_stride, gain, reinterpret_cast<__nv_bfloat16*>(out), out_stride, rows, d, eps);
  else
    rmsnorm_kernel<float><<<grid, 256, 0, as_stream(stream)>>>(*mem, x, x_stride, gain,
                                                               reinterpret_cast<float*>(out), out_stride, rows, d, eps);
  ARMT_CHECK_LAUNCH("rmsnorm");
  return ARMT_OK;
}

int armt_rope(int G, void* qkv, long long ld, long long stride, int dtype, int T, int n_heads, int dh,
              const float* cos_t, const float* sin_t, void* stream) {
  ARMT_REQUIRE(G >= 1 && T >= 1 && dh >= 2 && dh % 2 == 0, ARMT_ERR_DIM, "rope: bad sizes");
  dim3 grid(T, G);
  if (dtype == ARMT_BF16)
    rope_kernel<__nv_bfloat16><<<grid, 128, 0, as_stream(stream)>>>(reinterpret_cast<__nv_bfloat16*>(qkv), ld,
                                                                    stride, T, n_heads, dh, cos_t, sin_t);
  else
    rope_kernel<float><<<grid, 128, 0, as_stream(stream)>>>(reinterpret_cast<float*>(qkv), ld, stride, T, n_heads,
                                                            dh, cos_t, sin_t);
  ARMT_CHECK_LAUNCH("rope");
  return ARMT_OK;
}

int armt_swiglu(int G, const void* gu, long long ld_gu, long long gu_stride, void* out, long long ld_out,
                long long out_stride, int dtype, int rows, int d_ff, int block, void* stream) {
  ARMT_REQUIRE(G >= 1 && rows >= 1 && d_ff >= 1 && block >= 1 && d_ff % block == 0, ARMT_ERR_DIM,
               "swiglu: bad sizes");
  dim3 grid(rows, G);
  if (dtype == ARMT_BF16)
    swiglu_kernel<__nv_bfloat16><<<grid, 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const __nv_bfloat16*>(gu), ld_gu, gu_stride, reinterpret_cast<__nv_bfloat16*>(out), ld_out,
        out_stride, d_ff, block);
  else
    swiglu_kernel<float><<<grid, 256, 0, as_stream(stream)>>>(reinterpret_cast<const float*>(gu), ld_gu, gu_stride,
                                                               reinterpret_cast<float*>(out), ld_out, out_stride,
                                                               d_ff, block);
  ARMT_CHECK_LAUNCH("swiglu");
  return ARMT_OK;
}

int armt_dpfp_den(const ArmtMembers* mem, const float* q, long long q_stride, const float* z, void* phi,
                  int phi_dtype, long long ld_phi, long long phi_stride, float* den, long long den_stride, int rows,
                  int d_mem, int nu, void* stream) {
  ARMT_REQUIRE(mem && mem->G >= 1 && mem->G <= ARMT_MAX_MEMBERS, ARMT_ERR_DIM, "dpfp: bad member count");
  ARMT_REQUIRE(nu >= 1, ARMT_ERR_INPUT, "dpfp order must be >= 1, got %d", nu);
  ARMT_REQUIRE(ld_phi >= 2LL * nu * d_mem, ARMT_ERR_DIM, "dpfp: ld_phi too small");
  dim3 grid((rows + 7) / 8, mem->G);
  if (phi_dtype == ARMT_BF16)
    dpfp_den_kernel<__nv_bfloat16><<<grid, 256, 0, as_stream(stream)>>>(
        *mem, q, q_stride, z, reinterpret_cast<__nv_bfloat16*>(phi), ld_phi, phi_stride, den, den_stride, rows, d_mem,
        nu);
  else
    dpfp_den_kernel<float><<<grid, 256, 0, as_stream(stream)>>>(*mem, q, q_stride, z, reinterpret_cast<float*>(phi),
                                                                ld_phi, phi_stride, den, den_stride, rows, d_mem, nu);
  ARMT_CHECK_LAUNCH("dpfp_den");
  return ARMT_OK;
}

int armt_cast(const void* src, int sd, void* dst, int dd, long long n, void* stream) {
  if (n <= 0) return ARMT_OK;
  const int blocks = (int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
  cudaStream_t s = as_stream(stream);
  if (sd == ARMT_F32 && dd == ARMT_BF16)
    cast_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const float*>(src), reinterpret_cast<__nv_bfloat16*>(dst), n);
  else if (sd == ARMT_BF16 && dd == ARMT_F32)
    cast_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const __nv_bfloat16*>(src), reinterpret_cast<float*>(dst), n);
  else if (sd == ARMT_F32 && dd == ARMT_F32)
    cast_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const float*>(src), reinterpret_cast<float*>(dst), n);
  else
    cast_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const __nv_bfloat16*>(src),
                                       reinterpret_cast<__nv_bfloat16*>(dst), n);
  ARMT_CHECK_LAUNCH("cast");
  return ARMT_OK;
}

int armt_logits_nll(const void* logits, int dtype, long long ld, const long long* targets, float* nll,
                    long long rows, int vocab, void* stream) {
  if (rows <= 0) return ARMT_OK;
  if (dtype == ARMT_BF16)
    nll_kernel<<<(unsigned)rows, 256, 0, as_stream(stream)>>>(reinterpret_cast<const __nv_bfloat16*>(logits), ld,
                                                              targets, nll, vocab);
  else
    nll_kernel<<<(unsigned)rows, 256, 0, as_stream(stream)>>>(reinterpret_cast<const float*>(logits), ld, targets,
                                                              nll, vocab);
  ARMT_CHECK_LAUNCH("nll");
  return ARMT_OK;
}

int armt_lse_finalize(const float* lse_part, long long lse_ld, int n_tiles, const float* tgt,
                      const long long* targets, float* nll, long long rows, void* stream) {
  if (rows <= 0) return ARMT_OK;
  lse_finalize_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float2*>(lse_part), lse_ld, n_tiles, tgt, targets, nll, rows);
  ARMT_CHECK_LAUNCH("lse_finalize");
  return ARMT_OK;
}

int armt_lse_reduce(const float* lse_part, long long lse_ld, int n_tiles, float* out, long long rows, void* stream) {
  if (rows <= 0) return ARMT_OK;
  ARMT_REQUIRE(lse_part && out && n_tiles >= 1, ARMT_ERR_INPUT, "lse_reduce: bad arguments");
  lse_reduce_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float2*>(lse_part), lse_ld, n_tiles, reinterpret_cast<float2*>(out), rows);
  ARMT_CHECK_LAUNCH("lse_reduce");
  return ARMT_OK;
}

const char* armt_last_error(void) { return g_err; }
const char* armt_version(void) { return "armt_b200 0.1.0 (sm_100a)"; }
int armt_num_sms(void) { return num_sms(); }
int armt_kernel_count(void) { return (int)launch_counter().load(); }
long long armt_abi_sizeof(int which) {
  switch (which) {
    case 0: return (long long)sizeof(ArmtGemmArgs);
    case 1: return (long long)sizeof(ArmtMembers);
    case 2: return (long long)offsetof(ArmtGemmArgs, a_slot);
  }
  return -1;
}

}  // extern "C"
