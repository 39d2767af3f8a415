// Tensor-core (tcgen05 + TMEM) sum-layer contractions for sm_100a.
//
// All three kernels share one recipe: fp32 log-domain inputs are shifted by a
// per-sample maximum, exponentiated, split into bf16 hi + lo and contracted
// as hi*hi + hi*lo + lo*hi with fp32 accumulation in TMEM (three kind::f16
// MMAs; ~2^-16 relative operand precision, well inside the 1e-4 parity bar).
// The per-sample maxima come from side outputs (bmax of the product kernel,
// rmax of the ratio-max pass), so each operand is read from HBM once.
// Parameter operands are the pre-split bf16 tiles (k_theta_to_mma) copied
// into shared memory with cp.async — one MMA per stacked tile.
//
//   sum forward  (engine.py:74-102):  D[b, n] = sum_j e^{child[j,b]-g_b} theta[n, j]
//   child flows  (engine.py:129-165): D[b, j] = sum_m e^{lnf[m,b]-g_b} theta[m, j]
//   param flows  (engine.py:105-126): D[m, j] = sum_b e^{lnf[m,b]-c_b} e^{child[j,b]+c_b}
#include <math.h>

#include "pcb_internal.cuh"
#include "pcb_tc.cuh"

#ifndef PCB_MN_VARIANT
#define PCB_MN_VARIANT 0  // MN-major descriptor: LBO = K-adjacent core stride
#endif

namespace pcb {

using namespace tc;

constexpr int TC_M = 128;      // samples (or sums) per MMA tile
constexpr int TC_NMAX = 256;   // max stacked N per CTA
constexpr int TC_THREADS = 256;

__device__ __forceinline__ float lnf_of(float f, float l) {
  return (l == PCB_NEG_INF) ? PCB_NEG_INF : (__logf(f) - l);
}

// store 8 consecutive K-elements (split hi/lo) of one A row
__device__ __forceinline__ void store_split8(uint8_t* sh, uint8_t* sl, uint32_t off,
                                             const float (&v)[8]) {
  uint32_t hi[4], lo[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    __nv_bfloat16 h0, l0, h1, l1;
    split_bf16(v[2 * e], h0, l0);
    split_bf16(v[2 * e + 1], h1, l1);
    hi[e] = pack2(h0, h1);
    lo[e] = pack2(l0, l1);
  }
  *reinterpret_cast<uint4*>(sh + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
  *reinterpret_cast<uint4*>(sl + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
}

// cp.async the stacked bf16 tiles of one stage: tile s (k_rows x k_cols,
// hi plane then lo plane, 4 * k_rows * k_cols bytes) lands at dst + s * bytes
__device__ __forceinline__ void copy_tiles(uint8_t* dst, const __nv_bfloat16* __restrict__ mma,
                                           const int32_t* __restrict__ slab_row0, int64_t stride,
                                           const int32_t* __restrict__ members, int m0, int S,
                                           int col, int tile_bytes, int tid) {
  const int chunks = tile_bytes >> 4;
  for (int q = tid; q < S * chunks; q += TC_THREADS) {
    const int s = q / chunks, o = q - s * chunks;
    const int slab = slab_row0[(int64_t)members[m0 + s] * stride + col];
    cp_async16(smem_u32(dst + s * tile_bytes + o * 16),
               reinterpret_cast<const uint8_t*>(mma + slab) + o * 16);
  }
}

// --------------------------------------------------------------- sum forward
template <int KN>
struct FwdSmem {
  static constexpr int kA = TC_M * KN * 2;           // one bf16 A plane
  static constexpr int kB = TC_NMAX * KN * 4;        // stacked tiles, hi+lo
  static constexpr int kStage = 2 * kA + kB;
  static constexpr int kBytes = 2 * kStage;
};

template <int KN>
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_sum_fwd_tc(int cap, int k_m, int B, int ldb, const int32_t* __restrict__ row_off,
                 const int32_t* __restrict__ members, const int32_t* __restrict__ sum_ids,
                 const int32_t* __restrict__ prod_ids, const int32_t* __restrict__ param_ids,
                 const int32_t* __restrict__ param_slab, const __nv_bfloat16* __restrict__ mma,
                 const float* __restrict__ scratch, const float* __restrict__ bmax,
                 float* __restrict__ values) {
  using SM = FwdSmem<KN>;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int row = tid & (TC_M - 1);  // sample within the tile
  const int half = tid >> 7;         // which half of the K chunk this thread converts
  const int sr = blockIdx.x;
  const int b = blockIdx.y * TC_M + row;
  const bool live = b < B;
  const int m0 = row_off[sr];
  const int S = row_off[sr + 1] - m0;
  const int N = S * k_m;
  const int r0 = members[m0];
  const int32_t* prow = prod_ids + (int64_t)r0 * cap;
  const int32_t* trow = param_ids + (int64_t)r0 * cap;

  float gm = PCB_NEG_INF;  // per-sample max over all children of the super-row
  if (live)
    for (int c = 0; c < cap; ++c)
      if (trow[c] != 0) gm = fmaxf(gm, bmax[(int64_t)(prow[c] / KN) * ldb + b]);
  const bool dead = (gm == PCB_NEG_INF);

  const uint32_t ncols = tmem_cols_for(N);
  if (tid == 0) {
    mbar_init(smem_u32(&mbar[0]), 1);
    mbar_init(smem_u32(&mbar[1]), 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(smem_u32(&tmem_base), ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = idesc_bf16(TC_M, k_m);
  constexpr uint32_t SBO = (KN / 8) * 128;
  const int tile_bytes = k_m * KN * 4;

  int it = 0;
  for (int c = 0; c < cap; ++c) {
    if (trow[c] == 0) continue;  // padded child column (uniform across the CTA)
    const int stage = it & 1;
    if (it >= 2) mbar_wait(smem_u32(&mbar[stage]), ((it - 2) >> 1) & 1);
    uint8_t* sAh = smem + stage * SM::kStage;
    uint8_t* sAl = sAh + SM::kA;
    uint8_t* sB = sAl + SM::kA;
    copy_tiles(sB, mma, param_slab, cap, members, m0, S, c, tile_bytes, tid);
    const float* src = scratch + (int64_t)prow[c] * ldb + b;
#pragma unroll
    for (int jq = half * (KN / 16); jq < (half + 1) * (KN / 16); ++jq) {
      float x[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) x[e] = live ? src[(int64_t)(jq * 8 + e) * ldb] : PCB_NEG_INF;
#pragma unroll
      for (int e = 0; e < 8; ++e) x[e] = dead ? 0.f : __expf(x[e] - gm);
      store_split8(sAh, sAl, kmajor_off(row, jq * 8, KN), x);
    }
    cp_async_wait_all();
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t aH = smem_u32(sAh), aL = smem_u32(sAl), bB = smem_u32(sB);
      for (int s = 0; s < S; ++s) {
        const uint32_t bH = bB + s * tile_bytes, bL = bH + tile_bytes / 2;
        const uint32_t d = tmem + s * k_m;
#pragma unroll
        for (int ks = 0; ks < KN / 16; ++ks) {
          const uint32_t o = ks * 256;
          mma_bf16(d, make_desc(aH + o, 128, SBO), make_desc(bH + o, 128, SBO), idesc,
                   (it > 0 || ks > 0) ? 1u : 0u);
          mma_bf16(d, make_desc(aH + o, 128, SBO), make_desc(bL + o, 128, SBO), idesc, 1u);
          mma_bf16(d, make_desc(aL + o, 128, SBO), make_desc(bH + o, 128, SBO), idesc, 1u);
        }
      }
      mma_commit(smem_u32(&mbar[stage]));
    }
    __syncwarp();
    ++it;
  }
  if (it > 0) {
    mbar_wait(smem_u32(&mbar[(it - 1) & 1]), ((it - 1) >> 1) & 1);
    tc_fence_after();
  }
  // epilogue: warps w and w+4 share TMEM lanes; they split the 16-column chunks
  const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
  for (int c0 = (warp >> 2) * 16; c0 < N; c0 += 32) {
    float v[16];
    tmem_ld16(tmem + lane_base + c0, v);
    if (!live) continue;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int n = c0 + i;
      if (n >= N) break;
      const int s = n / k_m, mm = n - s * k_m;
      const int sid = sum_ids[members[m0 + s]] + mm;
      const float d = (it > 0) ? v[i] : 0.f;
      values[(int64_t)sid * ldb + b] = (dead || !(d > 0.f)) ? PCB_NEG_INF : (__logf(d) + gm);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free(tmem, ncols);
}

// --------------------------------------------------------------- child flows
template <int KM>
struct CfSmem {
  static constexpr int kA = TC_M * KM * 2;
  static constexpr int kB = TC_NMAX * KM * 4;
  static constexpr int kStage = 2 * kA + kB;
  static constexpr int kBytes = 2 * kStage;
};

template <int KM>
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_child_flow_tc(int cap, int k_n, int B, int ldb, const int32_t* __restrict__ row_off,
                    const int32_t* __restrict__ members, const int32_t* __restrict__ ch_ids,
                    const int32_t* __restrict__ par_ids, const int32_t* __restrict__ ppids,
                    const int32_t* __restrict__ par_slab, const __nv_bfloat16* __restrict__ mma,
                    const float* __restrict__ values, const float* __restrict__ flows,
                    const float* __restrict__ scratch, const float* __restrict__ rmax,
                    int64_t sb_base, float* __restrict__ flow_scratch) {
  using SM = CfSmem<KM>;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int row = tid & (TC_M - 1);
  const int half = tid >> 7;
  const int sr = blockIdx.x;
  const int b = blockIdx.y * TC_M + row;
  const bool live = b < B;
  const int m0 = row_off[sr];
  const int S = row_off[sr + 1] - m0;
  const int N = S * k_n;
  const int r0 = members[m0];
  const int32_t* parow = par_ids + (int64_t)r0 * cap;
  const int32_t* pprow = ppids + (int64_t)r0 * cap;

  float gm = PCB_NEG_INF;  // per-sample max of lnf over every parent sum
  if (live)
    for (int p = 0; p < cap; ++p)
      if (pprow[p] != 0) gm = fmaxf(gm, rmax[((int64_t)parow[p] - sb_base) / KM * ldb + b]);
  const bool dead = (gm == PCB_NEG_INF);

  const uint32_t ncols = tmem_cols_for(N);
  if (tid == 0) {
    mbar_init(smem_u32(&mbar[0]), 1);
    mbar_init(smem_u32(&mbar[1]), 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(smem_u32(&tmem_base), ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = idesc_bf16_bmn(TC_M, k_n);
  constexpr uint32_t SBO_A = (KM / 8) * 128;
  const uint32_t kstride = (uint32_t)(k_n / 8) * 128;  // K-adjacent cores of a tile
  const uint32_t lbo = PCB_MN_VARIANT == 0 ? kstride : 128u;
  const uint32_t sbo = PCB_MN_VARIANT == 0 ? 128u : kstride;
  const int tile_bytes = KM * k_n * 4;

  int it = 0;
  for (int p = 0; p < cap; ++p) {
    if (pprow[p] == 0) continue;
    const int stage = it & 1;
    if (it >= 2) mbar_wait(smem_u32(&mbar[stage]), ((it - 2) >> 1) & 1);
    uint8_t* sAh = smem + stage * SM::kStage;
    uint8_t* sAl = sAh + SM::kA;
    uint8_t* sB = sAl + SM::kA;
    copy_tiles(sB, mma, par_slab, cap, members, m0, S, p, tile_bytes, tid);
    const int64_t base = (int64_t)parow[p] * ldb + b;
#pragma unroll
    for (int kq = half * (KM / 16); kq < (half + 1) * (KM / 16); ++kq) {
      float f[8], l[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int64_t o = base + (int64_t)(kq * 8 + e) * ldb;
        f[e] = live ? flows[o] : 0.f;
        l[e] = live ? values[o] : PCB_NEG_INF;
      }
      float x[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float a = lnf_of(f[e], l[e]);
        x[e] = (dead || a == PCB_NEG_INF) ? 0.f : __expf(a - gm);
      }
      store_split8(sAh, sAl, kmajor_off(row, kq * 8, KM), x);
    }
    cp_async_wait_all();
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t aH = smem_u32(sAh), aL = smem_u32(sAl), bB = smem_u32(sB);
      for (int s = 0; s < S; ++s) {
        const uint32_t bH = bB + s * tile_bytes, bL = bH + tile_bytes / 2;
        const uint32_t d = tmem + s * k_n;
#pragma unroll
        for (int ks = 0; ks < KM / 16; ++ks) {
          const uint32_t oa = ks * 256, ob = ks * 2 * kstride;
          mma_bf16(d, make_desc(aH + oa, 128, SBO_A), make_desc(bH + ob, lbo, sbo), idesc,
                   (it > 0 || ks > 0) ? 1u : 0u);
          mma_bf16(d, make_desc(aH + oa, 128, SBO_A), make_desc(bL + ob, lbo, sbo), idesc, 1u);
          mma_bf16(d, make_desc(aL + oa, 128, SBO_A), make_desc(bH + ob, lbo, sbo), idesc, 1u);
        }
      }
      mma_commit(smem_u32(&mbar[stage]));
    }
    __syncwarp();
    ++it;
  }
  if (it > 0) {
    mbar_wait(smem_u32(&mbar[(it - 1) & 1]), ((it - 1) >> 1) & 1);
    tc_fence_after();
  }
  const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
  for (int c0 = (warp >> 2) * 16; c0 < N; c0 += 32) {
    float v[16];
    tmem_ld16(tmem + lane_base + c0, v);
    if (!live) continue;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int n = c0 + i;
      if (n >= N) break;
      const int s = n / k_n, j = n - s * k_n;
      const int64_t o = (int64_t)(ch_ids[members[m0 + s]] + j) * ldb + b;
      const float d = (it > 0) ? v[i] : 0.f;
      flow_scratch[o] = (dead || !(d > 0.f)) ? 0.f : __expf(__logf(d) + gm + scratch[o]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free(tmem, ncols);
}

// --------------------------------------------------------------- param flows
// One CTA = one super-row (all of its <= 256 sums as up to two 128-row M
// tiles, two TMEM accumulators) x up to 256 product columns; K = samples
// streamed 32 at a time.  Each product operand chunk is converted once and
// feeds both M tiles.  c_b = per-sample max of rmax over the super-row.
constexpr int PF_KC = 32;

struct PfSmem {
  static constexpr int kA = 2 * TC_M * PF_KC * 2;  // 256 rows, one plane
  static constexpr int kB = TC_NMAX * PF_KC * 2;
  static constexpr int kStage = 2 * kA + 2 * kB;
  static constexpr int kBytes = 2 * kStage;
};

template <int KN>
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_param_flow_tc(int cap, int k_m, int B, int ldb, const int32_t* __restrict__ row_off,
                    const int32_t* __restrict__ members, const int32_t* __restrict__ sum_ids,
                    const int32_t* __restrict__ prod_ids, const int32_t* __restrict__ param_ids,
                    const int32_t* __restrict__ flow_ids, const float* __restrict__ theta,
                    const float* __restrict__ values, const float* __restrict__ flows,
                    const float* __restrict__ scratch, const float* __restrict__ rmax,
                    int64_t sb_base, float* __restrict__ f_params) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[2];
  __shared__ uint32_t tmem_base;
  __shared__ float cb[PF_KC];
  __shared__ int cols[TC_NMAX / 16];
  __shared__ int ncols_s;
  constexpr int CPG = TC_NMAX / KN;  // child columns per CTA
  const int tid = threadIdx.x, warp = tid >> 5;
  const int sr = blockIdx.x;
  const int cg = blockIdx.y;
  const int m0 = row_off[sr];
  const int S = row_off[sr + 1] - m0;
  const int Nsum = S * k_m;
  const int MT = (Nsum + TC_M - 1) / TC_M;  // 1 or 2 M tiles
  const int r0 = members[m0];
  const int32_t* trow = param_ids + (int64_t)r0 * cap;
  if (tid == 0) {
    int seen = 0, n = 0;
    for (int c = 0; c < cap; ++c) {
      if (trow[c] == 0) continue;
      if (seen >= cg * CPG && n < CPG) cols[n++] = c;
      ++seen;
    }
    ncols_s = n;
  }
  __syncthreads();
  const int ncol = ncols_s;
  if (ncol == 0) return;
  const int Npad = ncol * KN;
  const int ms = tid;  // A row (sum index within the super-row)
  const bool row_live = ms < Nsum;
  int sum_slot = 0;
  if (row_live) sum_slot = sum_ids[members[m0 + ms / k_m]] + (ms % k_m);

  const uint32_t ncols_t = MT > 1 ? 512u : tmem_cols_for(Npad);
  if (tid == 0) {
    mbar_init(smem_u32(&mbar[0]), 1);
    mbar_init(smem_u32(&mbar[1]), 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(smem_u32(&tmem_base), ncols_t);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = idesc_bf16(TC_M, Npad);
  constexpr uint32_t SBO = (PF_KC / 8) * 128;
  const int32_t* prow = prod_ids + (int64_t)r0 * cap;

  int it = 0;
  for (int b0 = 0; b0 < B; b0 += PF_KC, ++it) {
    const int stage = it & 1;
    float ln[PF_KC];
    if (row_live) {
      const float4* fp = reinterpret_cast<const float4*>(flows + (int64_t)sum_slot * ldb + b0);
      const float4* vp = reinterpret_cast<const float4*>(values + (int64_t)sum_slot * ldb + b0);
#pragma unroll
      for (int q = 0; q < PF_KC / 4; ++q) {
        const float4 f = fp[q], v = vp[q];
        ln[4 * q + 0] = lnf_of(f.x, v.x);
        ln[4 * q + 1] = lnf_of(f.y, v.y);
        ln[4 * q + 2] = lnf_of(f.z, v.z);
        ln[4 * q + 3] = lnf_of(f.w, v.w);
      }
    } else {
#pragma unroll
      for (int q = 0; q < PF_KC; ++q) ln[q] = PCB_NEG_INF;
    }
    if (it >= 2) mbar_wait(smem_u32(&mbar[stage]), ((it - 2) >> 1) & 1);
    __syncthreads();  // previous chunk's readers of cb are done
    if (tid < PF_KC) {
      float v = PCB_NEG_INF;
      if (b0 + tid < B)
        for (int s = 0; s < S; ++s) {
          const int64_t blk = (sum_ids[members[m0 + s]] - sb_base) / k_m;
          v = fmaxf(v, rmax[blk * ldb + b0 + tid]);
        }
      cb[tid] = v;
    }
    __syncthreads();
    uint8_t* sAh = smem + stage * PfSmem::kStage;
    uint8_t* sAl = sAh + PfSmem::kA;
    uint8_t* sBh = sAl + PfSmem::kA;
    uint8_t* sBl = sBh + PfSmem::kB;
#pragma unroll
    for (int kq = 0; kq < PF_KC / 8; ++kq) {
      float x[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int q = kq * 8 + e;
        const float c = cb[q];
        x[e] = (c == PCB_NEG_INF || ln[q] == PCB_NEG_INF || b0 + q >= B) ? 0.f
                                                                           : __expf(ln[q] - c);
      }
      store_split8(sAh, sAl, kmajor_off(ms, kq * 8, PF_KC), x);
    }
    for (int q = tid; q < Npad * (PF_KC / 8); q += TC_THREADS) {
      const int n = q / (PF_KC / 8), kq = q - n * (PF_KC / 8);
      const int c = cols[n / KN], j = n % KN;
      const float* src = scratch + (int64_t)(prow[c] + j) * ldb + b0 + kq * 8;
      const float4 x0 = *reinterpret_cast<const float4*>(src);
      const float4 x1 = *reinterpret_cast<const float4*>(src + 4);
      const float xs[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
      float x[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float c = cb[kq * 8 + e];
        x[e] = (c == PCB_NEG_INF) ? 0.f : fminf(__expf(xs[e] + c), 1e37f);
      }
      store_split8(sBh, sBl, kmajor_off(n, kq * 8, PF_KC), x);
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t bH = smem_u32(sBh), bL = smem_u32(sBl);
      for (int mt = 0; mt < MT; ++mt) {
        // M tile mt = A rows [128 mt, 128 mt + 128): 16 row-groups further on
        const uint32_t aH = smem_u32(sAh) + mt * 16 * SBO, aL = smem_u32(sAl) + mt * 16 * SBO;
        const uint32_t d = tmem + mt * 256;
#pragma unroll
        for (int ks = 0; ks < PF_KC / 16; ++ks) {
          const uint32_t o = ks * 256;
          mma_bf16(d, make_desc(aH + o, 128, SBO), make_desc(bH + o, 128, SBO), idesc,
                   (it > 0 || ks > 0) ? 1u : 0u);
          mma_bf16(d, make_desc(aH + o, 128, SBO), make_desc(bL + o, 128, SBO), idesc, 1u);
          mma_bf16(d, make_desc(aL + o, 128, SBO), make_desc(bH + o, 128, SBO), idesc, 1u);
        }
      }
      mma_commit(smem_u32(&mbar[stage]));
    }
    __syncwarp();
  }
  mbar_wait(smem_u32(&mbar[(it - 1) & 1]), ((it - 1) >> 1) & 1);
  tc_fence_after();
  // epilogue: warp w -> M tile w/4, TMEM lanes 32 (w%4) ..; one sum row per thread
  const int mt = warp >> 2;
  const int er = mt * TC_M + (warp & 3) * 32 + (tid & 31);
  const bool live = (mt < MT) && er < Nsum;
  int s = 0, mm = 0;
  if (live) {
    s = er / k_m;
    mm = er - s * k_m;
  }
  const int64_t rowbase = (int64_t)members[m0 + (live ? s : 0)] * cap;
  if (mt < MT)
    for (int c0 = 0; c0 < Npad; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + ((uint32_t)((warp & 3) * 32) << 16) + mt * 256 + c0, v);
      if (!live) continue;
      const int c = cols[c0 / KN];
      const int tile = param_ids[rowbase + c];
      const int flow = flow_ids[rowbase + c];
      const int j0 = c0 % KN;
      const float* th = theta + tile + mm * KN + j0;
      float* dst = f_params + flow + mm * KN + j0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float t = __ldg(th + i);
        if (t != 0.f && v[i] != 0.f) atomicAdd(dst + i, t * v[i]);
      }
    }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free(tmem, ncols_t);
}

// --------------------------------------------------------------- launchers
static bool tc_k(int64_t k) { return k == 16 || k == 32 || k == 64; }

bool tc_supported(const Layer& L) { return tc_k(L.k_m) && tc_k(L.k_n); }
bool tc_bwd_supported(const Layer& L) { return tc_k(L.k_m) && tc_k(L.k_n); }

template <typename K>
static int set_smem(K kernel, int bytes, bool& done) {
  if (done) return PCB_OK;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) !=
      cudaSuccess)
    return PCB_CUDA;
  done = true;
  return PCB_OK;
}

template <int KN>
static int fwd_kn(const pcb_plan* P, const Layer& L, const FwdGroup& g, const TcRows& tc,
                  cudaStream_t s, int B, int ldb, const float* scratch, const float* bmax,
                  float* values) {
  static bool done = false;
  if (set_smem(k_sum_fwd_tc<KN>, FwdSmem<KN>::kBytes, done)) return PCB_CUDA;
  dim3 grid((unsigned)tc.count, (unsigned)((B + TC_M - 1) / TC_M));
  k_sum_fwd_tc<KN><<<grid, TC_THREADS, FwdSmem<KN>::kBytes, s>>>(
      (int)g.cap, (int)L.k_m, B, ldb, tc.row_off, tc.members, g.sum_ids, g.prod_ids,
      g.param_ids, g.param_slab, P->mma, scratch, bmax, values);
  return check_launch();
}

int launch_sum_fwd_tc(const pcb_plan* P, const Layer& L, const FwdGroup& g, const TcRows& tc,
                      cudaStream_t s, int B, int ldb, const float* scratch, const float* bmax,
                      float* values) {
  ProfScope prof_(KC_SUM_FWD_TC, s);
  if (!tc.count || !B) return PCB_OK;
  switch (L.k_n) {
    case 16: return fwd_kn<16>(P, L, g, tc, s, B, ldb, scratch, bmax, values);
    case 32: return fwd_kn<32>(P, L, g, tc, s, B, ldb, scratch, bmax, values);
    case 64: return fwd_kn<64>(P, L, g, tc, s, B, ldb, scratch, bmax, values);
    default: return PCB_USAGE;
  }
}

template <int KM>
static int cf_km(const pcb_plan* P, const Layer& L, const BwdGroup& g, const TcRows& tc,
                 cudaStream_t s, int B, int ldb, const float* values, const float* flows,
                 const float* scratch, const float* rmax, float* flow_scratch) {
  static bool done = false;
  if (set_smem(k_child_flow_tc<KM>, CfSmem<KM>::kBytes, done)) return PCB_CUDA;
  dim3 grid((unsigned)tc.count, (unsigned)((B + TC_M - 1) / TC_M));
  k_child_flow_tc<KM><<<grid, TC_THREADS, CfSmem<KM>::kBytes, s>>>(
      (int)g.cap, (int)L.k_n, B, ldb, tc.row_off, tc.members, g.ch_ids, g.par_ids,
      g.par_param_ids, g.par_slab, P->mma, values, flows, scratch, rmax, L.sb_base,
      flow_scratch);
  return check_launch();
}

int launch_child_flow_tc(const pcb_plan* P, const Layer& L, const BwdGroup& g, const TcRows& tc,
                         cudaStream_t s, int B, int ldb, const float* values, const float* flows,
                         const float* scratch, const float* rmax, float* flow_scratch) {
  ProfScope prof_(KC_CHILD_FLOW, s);
  if (!tc.count || !B) return PCB_OK;
  switch (L.k_m) {
    case 16: return cf_km<16>(P, L, g, tc, s, B, ldb, values, flows, scratch, rmax, flow_scratch);
    case 32: return cf_km<32>(P, L, g, tc, s, B, ldb, values, flows, scratch, rmax, flow_scratch);
    case 64: return cf_km<64>(P, L, g, tc, s, B, ldb, values, flows, scratch, rmax, flow_scratch);
    default: return PCB_USAGE;
  }
}

template <int KN>
static int pf_kn(const Layer& L, const FwdGroup& g, const TcRows& tc, cudaStream_t s, int B,
                 int ldb, const float* theta, const float* values, const float* flows,
                 const float* scratch, const float* rmax, float* f_params) {
  static bool done = false;
  if (set_smem(k_param_flow_tc<KN>, PfSmem::kBytes, done)) return PCB_CUDA;
  const int cgroups = (int)((g.cap * KN + TC_NMAX - 1) / TC_NMAX);
  dim3 grid((unsigned)tc.count, (unsigned)cgroups);
  k_param_flow_tc<KN><<<grid, TC_THREADS, PfSmem::kBytes, s>>>(
      (int)g.cap, (int)L.k_m, B, ldb, tc.row_off, tc.members, g.sum_ids, g.prod_ids,
      g.param_ids, g.flow_ids, theta, values, flows, scratch, rmax, L.sb_base, f_params);
  return check_launch();
}

int launch_param_flow_tc(const Layer& L, const FwdGroup& g, const TcRows& tc, cudaStream_t s,
                         int B, int ldb, const float* theta, const float* values,
                         const float* flows, const float* scratch, const float* rmax,
                         float* f_params) {
  ProfScope prof_(KC_PARAM_FLOW, s);
  if (!tc.count || !B) return PCB_OK;
  switch (L.k_n) {
    case 16: return pf_kn<16>(L, g, tc, s, B, ldb, theta, values, flows, scratch, rmax, f_params);
    case 32: return pf_kn<32>(L, g, tc, s, B, ldb, theta, values, flows, scratch, rmax, f_params);
    case 64: return pf_kn<64>(L, g, tc, s, B, ldb, theta, values, flows, scratch, rmax, f_params);
    default: return PCB_USAGE;
  }
}

}  // namespace pcb
