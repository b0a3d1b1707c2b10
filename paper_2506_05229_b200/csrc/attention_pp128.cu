// tcgen05 causal segment attention, ping-pong form for d_head 128 (bf16; the C5 head size).
//
// Reference: armt/layers.py:211-223 (scores = q k^T / sqrt(dh) + causal mask over all T rows,
// max-subtracted softmax, ctx = P v, heads merged).
//
// The d_head-64 kernel's structure (attention_pp.cu: persistent CTA, TMA producer warp, one
// MMA-issuing thread, two softmax warpgroups ping-ponging over a PAIR of query tiles that share
// every K/V tile, S / O / P in TMEM, thread = query row, lazy running max) with the K/V step cut
// to 64 keys so that both groups' S (64 columns), O (128) and P (32) fit TMEM (448 of 512
// columns). Q, K and V rows are 256 B, so every operand tile is two 64-column SW128 sub-tiles:
// the S MMA walks K = 128 as 2 x 4 K-steps, the PV MMA reads V as an MN-major operand whose two
// 64-column halves sit LBO = 8 KB apart.

#include "tc_ptx.cuh"

namespace armt {

int make_tma_map_bf16(CUtensorMap* map, const void* base, long long cols, long long rows, long long batches,
                      long long ld, long long batch_stride, int box_rows);

namespace attn_pp128 {

using namespace tcx;

constexpr int DH = 128, BQ = 128, BKV = 64, NG = 2, NTHREADS = 128 + NG * 128;
#ifndef ARMT_PP128_NST
#define ARMT_PP128_NST 4
#endif
constexpr int NST = ARMT_PP128_NST;               // K/V stages
constexpr int QTILE = BQ * DH * 2;                // 32 KB: two 64-column sub-tiles
constexpr int QSUB = BQ * 64 * 2;                 // 16 KB
constexpr int KVTILE = BKV * DH * 2;              // 16 KB: two 64-column sub-tiles
constexpr int KVSUB = BKV * 64 * 2;               // 8 KB
constexpr int Q_BYTES = NG * QTILE;               // one Q buffer (three tiles)
constexpr int KV_BYTES = 2 * KVTILE;              // K + V of one stage
constexpr int S_COL = 0, O_COL = NG * BKV, P_COL = O_COL + NG * DH, TMEM_COLS = 512;
constexpr int BAR_BYTES = 512;
#ifndef ARMT_PP128_QB
#define ARMT_PP128_QB 1
#endif
constexpr int QB = ARMT_PP128_QB;                 // Q buffers (items in flight)
constexpr int SMEM = QB * Q_BYTES + NST * KV_BYTES + BAR_BYTES;
static_assert(SMEM <= 227 * 1024, "attention (d_head 128) shared memory budget");
static_assert(P_COL + NG * BKV / 2 <= TMEM_COLS, "TMEM columns");
constexpr float RESCALE_LOG2 = 8.f;
#ifndef ARMT_PP128_CHUNKED
#define ARMT_PP128_CHUNKED 1
#endif
constexpr bool CHUNKED = ARMT_PP128_CHUNKED;

struct Params {
  __nv_bfloat16* ctx;
  long long ld_ctx, ctx_stride;
  int T, H, G, d, nq, npair, nkv_all, nctas, chunked_items;
  float scale_log2;
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ unsigned long long f2_u(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void u_f2(unsigned long long r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// D[tmem] (+)= A[tmem] . B[smem]: the TS form (A K-major in TMEM, lane = row)
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
      ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_ld64(uint32_t taddr, float* v) {
  uint32_t r[64];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld32f(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_st32u(uint32_t taddr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
               ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
               : "memory");
}

__device__ __forceinline__ void tmem_st32f(uint32_t taddr, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
               ::"r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])), "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])), "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])), "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])), "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])), "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
               : "memory");
}

struct Item {
  int qt[NG], n[NG], h, g, nmax;
};

// item w: round = w / HG walks pairs of query tiles from the last (heaviest) down; the
// (member, head) slots of a round are visited in alternating directions (K/V reuse in L2)
__device__ __forceinline__ Item decode(int w, const Params& p) {
  Item I;
  const int HG = p.H * p.G, P = p.nctas;
  int round, slot;
  if (CHUNKED && w < p.chunked_items) {
    // chunks of P (member, head) slots, all query-pair rounds of a chunk together, heaviest
    // first: with the persistent round-robin CTA b takes slot chunk * P + b in every round, so
    // each CTA walks one slot's query pairs back to back (its K/V stays in L2) and every CTA
    // gets the same work per chunk
    const int per = P * p.npair;
    const int c = w / per, x = w - c * per;
    round = x / P;
    slot = c * P + (x - round * P);
  } else {
    // the slots past the last whole chunk: rounds over all of them, alternating direction
    const int base = CHUNKED ? p.chunked_items / p.npair : 0, n = HG - base;
    const int x = w - (CHUNKED ? p.chunked_items : 0);
    round = x / n;
    int r = x - round * n;
    if (round & 1) r = n - 1 - r;
    slot = base + r;
  }
  const int trip = p.npair - 1 - round;
  I.h = slot % p.H;
  I.g = slot / p.H;
  I.nmax = 0;
#pragma unroll
  for (int s = 0; s < NG; ++s) {
    const int qt = NG * trip + s;
    I.qt[s] = qt;
    I.n[s] = qt < p.nq ? min(2 * (qt + 1), p.nkv_all) : 0;
    I.nmax = max(I.nmax, I.n[s]);
  }
  return I;
}

__global__ void __launch_bounds__(NTHREADS, 1)
attn_pp128_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV,
                const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem) & 1023) != 0) __trap();  // SW128 operand tiles need 1 KB alignment
  uint8_t* sQ = smem;                              // buffer qi: tile s at qi * Q_BYTES + s * QTILE
  uint8_t* sKV = sQ + QB * Q_BYTES;                // stage st: K at st * KV_BYTES, V at + KVTILE
  uint64_t* bar = reinterpret_cast<uint64_t*>(sKV + NST * KV_BYTES);
  uint64_t* q_full = bar;                    // [2]
  uint64_t* q_empty = bar + 2;               // [2]
  uint64_t* kv_full = bar + 4;               // [NST]
  uint64_t* kv_empty = kv_full + NST;        // [NST]
  uint64_t* s_full = kv_empty + NST;         // [NG]
  uint64_t* s_empty = s_full + NG;
  uint64_t* p_full = s_empty + NG;
  uint64_t* p_empty = p_full + NG;
  uint64_t* o_full = p_empty + NG;
  uint64_t* o_empty = o_full + NG;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + NG);
  static_assert((4 + 2 * NST + 6 * NG) * 8 + 4 <= BAR_BYTES, "barrier region");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = p.npair * p.H * p.G;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmQ)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmKV)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < 2; ++i) { mbar_init(&q_full[i], 1); mbar_init(&q_empty[i], 1); }
    for (int i = 0; i < NST; ++i) { mbar_init(&kv_full[i], 1); mbar_init(&kv_empty[i], 1); }
    for (int i = 0; i < NG; ++i) {
      mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 4);
      mbar_init(&p_full[i], 4); mbar_init(&p_empty[i], 1);
      mbar_init(&o_full[i], 1); mbar_init(&o_empty[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tmem_slot)), "r"(TMEM_COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_launch_dependents();
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int tt = 0, it = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++it) {
        const Item I = decode(w, p);
        const int qi = it % QB;
        mbar_wait_sleep(&q_empty[qi], ((it / QB) & 1) ^ 1);
        int nvalid = 0;
#pragma unroll
        for (int s = 0; s < NG; ++s) nvalid += I.n[s] > 0;
        mbar_expect_tx(&q_full[qi], nvalid * QTILE);
#pragma unroll
        for (int s = 0; s < NG; ++s)
          if (I.n[s])
#pragma unroll
            for (int u = 0; u < 2; ++u)
              tma_load_3d(sQ + qi * Q_BYTES + s * QTILE + u * QSUB, &tmQ, &q_full[qi], I.h * DH + 64 * u,
                          I.qt[s] * BQ, I.g);
        for (int j = 0; j < I.nmax; ++j, ++tt) {
          const int st = tt % NST;
          mbar_wait_sleep(&kv_empty[st], ((tt / NST) & 1) ^ 1);
          mbar_expect_tx(&kv_full[st], KV_BYTES);
          uint8_t* base = sKV + st * KV_BYTES;
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            tma_load_3d(base + u * KVSUB, &tmKV, &kv_full[st], p.d + I.h * DH + 64 * u, j * BKV, I.g);
            tma_load_3d(base + KVTILE + u * KVSUB, &tmKV, &kv_full[st], 2 * p.d + I.h * DH + 64 * u, j * BKV, I.g);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer: per KV step j, S_s(j) for every group, then PV_s(j-1)
      constexpr uint32_t idS = instr_desc<128, BKV, 0>();
      constexpr uint32_t idO = instr_desc<128, DH, 1>();
      int u[NG], io[NG];
#pragma unroll
      for (int s = 0; s < NG; ++s) { u[s] = 0; io[s] = 0; }
      int tt = 0, it = 0;
      auto issue_pv = [&](int s, int j, int v, int st, bool last) {
        mbar_wait(&p_full[s], v & 1);
        if (j == 0) mbar_wait(&o_empty[s], (io[s] & 1) ^ 1);
        tc_fence_after();
        const uint32_t vbase = smem_u32(sKV + st * KV_BYTES + KVTILE);
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k) {
          // B = V (MN-major SW128: +2048 B per 16 keys, LBO = 8 KB to the second 64 d_head
          // columns); A = P from TMEM (8 packed columns per 16 keys)
          const uint64_t b = (smem_desc_sw128(vbase) | ((uint64_t)(KVSUB >> 4) << 16)) + (uint64_t)((2048 * k) >> 4);
          mma_bf16_ts(tmem + O_COL + s * DH, tmem + P_COL + s * (BKV / 2) + 8 * k, b, idO, j > 0 || k > 0);
        }
        mma_commit(&p_empty[s]);
        if (last) { mma_commit(&o_full[s]); ++io[s]; }
      };
      for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++it) {
        const Item I = decode(w, p);
        const int qi = it % QB;
        mbar_wait(&q_full[qi], (it / QB) & 1);
        for (int j = 0; j < I.nmax; ++j) {
          const int st = (tt + j) % NST;
          mbar_wait(&kv_full[st], ((tt + j) / NST) & 1);
          const uint32_t kbase = smem_u32(sKV + st * KV_BYTES);
#pragma unroll
          for (int s = 0; s < NG; ++s) {
            if (j >= I.n[s]) continue;
            mbar_wait(&s_empty[s], ((u[s] + j) & 1) ^ 1);
            tc_fence_after();
            const uint32_t qbase = smem_u32(sQ + qi * Q_BYTES + s * QTILE);
#pragma unroll
            for (int k = 0; k < DH / 16; ++k)
              mma_bf16(tmem + S_COL + s * BKV, smem_desc_sw128(qbase + (k >> 2) * QSUB) + 2 * (k & 3),
                       smem_desc_sw128(kbase + (k >> 2) * KVSUB) + 2 * (k & 3), idS, k > 0);
            mma_commit(&s_full[s]);
          }
          if (j > 0) {
            const int pst = (tt + j - 1) % NST;
#pragma unroll
            for (int s = 0; s < NG; ++s)
              if (j - 1 < I.n[s]) issue_pv(s, j - 1, u[s] + j - 1, pst, j == I.n[s]);
            mma_commit(&kv_empty[pst]);
          }
        }
        mma_commit(&q_empty[qi]);   // every S MMA of this item has read its Q tiles
        const int lst = (tt + I.nmax - 1) % NST;
#pragma unroll
        for (int s = 0; s < NG; ++s)
          if (I.n[s] == I.nmax) issue_pv(s, I.nmax - 1, u[s] + I.nmax - 1, lst, true);
        mma_commit(&kv_empty[lst]);
#pragma unroll
        for (int s = 0; s < NG; ++s) u[s] += I.n[s];
        tt += I.nmax;
      }
    }
  } else if (warp >= 4) {
    // ---------------- softmax: group s, thread = query row r (TMEM lane)
    const int s = (warp - 4) >> 2;
    const int ew = warp & 3;
    const int r = ew * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(ew * 32) << 16);
    const uint32_t tS = tl + S_COL + s * BKV, tO = tl + O_COL + s * DH, tP = tl + P_COL + s * (BKV / 2);
    const float sl2 = p.scale_log2;
    int v = 0, io = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
      const Item I = decode(w, p);
      const int nk = s == 0 ? I.n[0] : I.n[1];
      if (nk == 0) continue;
      const int qt = s == 0 ? I.qt[0] : I.qt[1];
      const int qrow = qt * BQ + r;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < nk; ++j, ++v) {
        const int k0 = j * BKV;
        const int lim = min(qrow, p.T - 1) - k0;   // valid keys of this row: c <= lim
        mbar_wait(&s_full[s], v & 1);
        tc_fence_after();
        float sv[BKV];
        tmem_ld64(tS, sv);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[s]);
        if (k0 + BKV - 1 > qt * BQ || k0 + BKV > p.T) {   // reaches the diagonal or ragged (warp-uniform)
#pragma unroll
          for (int c = 0; c < BKV; ++c) sv[c] = c <= lim ? sv[c] : -INFINITY;
        }
        float mc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mc[i] = fmaxf(sv[i], sv[i + 8]);
#pragma unroll
        for (int c = 16; c < BKV; c += 16)
#pragma unroll
          for (int i = 0; i < 8; i += 2) {
            mc[i] = fmaxf(mc[i], fmaxf(sv[c + i], sv[c + i + 8]));
            mc[i + 1] = fmaxf(mc[i + 1], fmaxf(sv[c + i + 1], sv[c + i + 9]));
          }
        const float mx = fmaxf(fmaxf(fmaxf(mc[0], mc[1]), fmaxf(mc[2], mc[3])),
                               fmaxf(fmaxf(mc[4], mc[5]), fmaxf(mc[6], mc[7])));
        const bool raise = (mx - m) * sl2 > RESCALE_LOG2;
        const float corr = raise ? ex2((m - mx) * sl2) : 1.f;   // first step: m = -inf -> 0
        if (raise) m = mx;
        const float nm = -m * sl2;
        const unsigned long long sc2 = f2_u(sl2, sl2), nm2 = f2_u(nm, nm);
        unsigned long long sum2[4];
        uint32_t pk[BKV / 2];
#pragma unroll
        for (int c = 0; c < BKV; c += 2) {
          const unsigned long long e = ffma2(f2_u(sv[c], sv[c + 1]), sc2, nm2);
          float a, b;
          u_f2(e, a, b);
          a = ex2(a);
          b = ex2(b);
          pk[c >> 1] = pack_bf16x2(a, b);
          const int q = (c >> 1) & 3;
          sum2[q] = c < 8 ? f2_u(a, b) : fadd2(sum2[q], f2_u(a, b));
        }
        float ra, rb;
        u_f2(fadd2(fadd2(sum2[0], sum2[1]), fadd2(sum2[2], sum2[3])), ra, rb);
        mbar_wait(&p_empty[s], (v & 1) ^ 1);   // PV(v-1) done: P free, O stable
        tc_fence_after();
        tmem_st32u(tP, pk);
        if (j > 0 && __any_sync(0xffffffffu, raise)) {
#pragma unroll
          for (int c0 = 0; c0 < DH; c0 += 32) {
            float o[32];
            tmem_ld32f(tO + c0, o);
#pragma unroll
            for (int c = 0; c < 32; ++c) o[c] *= corr;
            tmem_st32f(tO + c0, o);
          }
        }
        l = l * corr + (ra + rb);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[s]);
      }
      // epilogue: O of this query tile complete in TMEM
      mbar_wait(&o_full[s], io & 1);
      ++io;
      tc_fence_after();
      const float inv = 1.f / l;
      __nv_bfloat16* out = p.ctx + (long long)I.g * p.ctx_stride + (long long)qrow * p.ld_ctx + I.h * DH;
#pragma unroll
      for (int c0 = 0; c0 < DH; c0 += 64) {
        float o[64];
        tmem_ld64(tO + c0, o);
        if (qrow < p.T) {
#pragma unroll
          for (int c = 0; c < 64; c += 8)
            *reinterpret_cast<uint4*>(out + c0 + c) =
                make_uint4(pack_bf16x2(o[c] * inv, o[c + 1] * inv), pack_bf16x2(o[c + 2] * inv, o[c + 3] * inv),
                           pack_bf16x2(o[c + 4] * inv, o[c + 5] * inv), pack_bf16x2(o[c + 6] * inv, o[c + 7] * inv));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[s]);
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
}

}  // namespace attn_pp128

int attention_pp128(int G, const void* qkv, long long ld_qkv, long long qkv_stride, void* ctx, long long ld_ctx,
                  long long ctx_stride, int T, int H, float scale, cudaStream_t s) {
  using namespace attn_pp128;
  CUtensorMap tmQ, tmKV;
  int rc = make_tma_map_bf16(&tmQ, qkv, ld_qkv, T, G, ld_qkv, qkv_stride, BQ);
  if (!rc) rc = make_tma_map_bf16(&tmKV, qkv, ld_qkv, T, G, ld_qkv, qkv_stride, BKV);
  if (rc) return rc;
  Params p;
  p.ctx = reinterpret_cast<__nv_bfloat16*>(ctx);
  p.ld_ctx = ld_ctx; p.ctx_stride = ctx_stride;
  p.T = T; p.H = H; p.G = G; p.d = H * DH;
  p.nq = (T + BQ - 1) / BQ;
  p.npair = (p.nq + NG - 1) / NG;
  p.nkv_all = (T + BKV - 1) / BKV;
  p.scale_log2 = scale * 1.4426950408889634f;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_pp128_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    attr = true;
  }
  const int items = p.npair * H * G;
  const int grid = items < num_sms() ? items : num_sms();
  p.nctas = grid;
  p.chunked_items = ((H * G) / grid) * grid * p.npair;
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = la;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, attn_pp128_kernel, tmQ, tmKV, p);
  ARMT_CHECK_LAUNCH("attention tcgen05 ping-pong d_head 128");
  return ARMT_OK;
}

}  // namespace armt
