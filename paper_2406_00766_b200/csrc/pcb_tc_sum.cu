// Tensor-core (tcgen05 + TMEM) sum-layer contractions for sm_100a.
//
// All three kernels share one recipe: fp32 log-domain inputs are shifted by a
// per-sample maximum, exponentiated (MUFU ex2 with the shift folded into one
// FFMA), split into bf16 hi + lo (packed cvt) and contracted as
// hi*hi + hi*lo + lo*hi with fp32 accumulation in TMEM (three kind::f16
// MMAs; ~2^-16 relative operand precision, well inside the 1e-4 parity bar).
// The per-sample maxima come from side outputs (bmax of the product kernel,
// rmax of the ratio-max pass), so each operand is read from HBM once.
// Parameter operands are the pre-split bf16 tiles (k_theta_to_mma), moved
// into shared memory by 1-D TMA bulk copies that complete on an mbarrier —
// one MMA per stacked tile.  Two smem stages: the conversion of stage s+1
// overlaps the MMAs of stage s, and every thread issues the global loads of
// stage s+1 into registers before converting stage s (the kernels are
// load-latency bound otherwise).
//
//   sum forward  (engine.py:74-102):  D[b, n] = sum_j e^{child[j,b]-g_b} theta[n, j]
//   child flows  (engine.py:129-165): D[b, j] = sum_m e^{lnf[m,b]-g_b} theta[m, j]
//   param flows  (engine.py:105-126): D[m, j] = sum_b e^{lnf[m,b]-c_b} e^{child[j,b]+c_b}
#include <math.h>

#include "pcb_internal.cuh"
#include "pcb_tc.cuh"

namespace pcb {

using namespace tc;

constexpr int TC_M = 128;      // samples (or sums) per MMA tile
constexpr int TC_NMAX = 256;   // max stacked N per CTA
constexpr int TC_THREADS = 256;

// store 8 consecutive K-elements (split hi/lo) of one operand row
__device__ __forceinline__ void store_split8(uint8_t* sh, uint8_t* sl, uint32_t off,
                                             const float* v) {
  float t[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) t[e] = v[e];
  uint4 hi, lo;
  split_pack8(t, hi, lo);
  *reinterpret_cast<uint4*>(sh + off) = hi;
  *reinterpret_cast<uint4*>(sl + off) = lo;
}

// one thread: TMA-bulk-copy the S stacked bf16 tiles of one stage (each
// `tile_bytes`: hi plane at slab, lo plane one plane region later) into dst
// as [hi | lo] per tile, completing on `full`
__device__ __forceinline__ void issue_tiles(uint8_t* dst, const __nv_bfloat16* __restrict__ mma,
                                            int64_t plane, const int32_t* __restrict__ slab_rows,
                                            int64_t stride, const int32_t* __restrict__ members,
                                            int m0, int S, int col, int tile_bytes, uint32_t full) {
  mbar_arrive_expect_tx(full, (uint32_t)(S * tile_bytes));
  for (int s = 0; s < S; ++s) {
    const int64_t slab = slab_rows[(int64_t)members[m0 + s] * stride + col];
    const uint32_t d = smem_u32(dst + s * tile_bytes);
    bulk_g2s(d, mma + slab, (uint32_t)tile_bytes / 2, full);
    bulk_g2s(d + tile_bytes / 2, mma + slab + plane, (uint32_t)tile_bytes / 2, full);
  }
}

__device__ __forceinline__ int next_real(const int32_t* __restrict__ ids, int cap, int c) {
  while (c < cap && ids[c] == 0) ++c;
  return c;
}

// exp(log(f) - l - g) in the log2 domain; 0 for impossible sums or zero flow
__device__ __forceinline__ float scaled_ratio(float f, float l, float gl2) {
  return (l == PCB_NEG_INF || !(f > 0.f)) ? 0.f : ex2(lg2(f) - fmaf(l, kL2E, gl2));
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
__global__ void __launch_bounds__(TC_THREADS, (KN <= 32) ? 2 : 1)
    k_sum_fwd_tc(int cap, int k_m, int B, int ldb, const int32_t* __restrict__ row_off,
                 const int32_t* __restrict__ members, const int32_t* __restrict__ sum_ids,
                 const int32_t* __restrict__ prod_ids, const int32_t* __restrict__ param_ids,
                 const int32_t* __restrict__ param_slab, const __nv_bfloat16* __restrict__ mma,
                 int64_t plane,
                 const float* __restrict__ scratch, const float* __restrict__ bmax,
                 float* __restrict__ values) {
  using SM = FwdSmem<KN>;
  constexpr int HALF = KN / 2;  // child rows converted per thread per stage
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t done[2], full[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int row = tid & (TC_M - 1);  // sample within the tile
  const int half = tid >> 7;         // which half of the K chunk this thread converts
  // 1-D grid, batch tiles of one super-row adjacent so its theta tiles are
  // fetched from HBM once and re-read from L2
  const int ntiles = (B + TC_M - 1) / TC_M;
  const int sr = blockIdx.x / ntiles;
  const int b = (blockIdx.x - sr * ntiles) * TC_M + row;
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
  const float gml = dead ? 0.f : gm * kL2E;

  const uint32_t ncols = tmem_cols_for(N);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&done[i]), 1);
      mbar_init(smem_u32(&full[i]), 1);
    }
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

  auto load = [&](int c, float* xr) {
    const float* src = scratch + ((int64_t)prow[c] + half * HALF) * ldb + b;
#pragma unroll
    for (int e = 0; e < HALF; ++e) xr[e] = live ? src[(int64_t)e * ldb] : PCB_NEG_INF;
  };
  float xn[HALF];
  int c = next_real(trow, cap, 0);
  if (c < cap) load(c, xn);
  int it = 0;
  while (c < cap) {
    float x[HALF];
#pragma unroll
    for (int e = 0; e < HALF; ++e) x[e] = xn[e];
    const int cn = next_real(trow, cap, c + 1);
    if (cn < cap) load(cn, xn);  // prefetch the next stage's children
    const int stage = it & 1;
    if (it >= 2) mbar_wait(smem_u32(&done[stage]), ((it - 2) >> 1) & 1);
    uint8_t* sAh = smem + stage * SM::kStage;
    uint8_t* sAl = sAh + SM::kA;
    uint8_t* sB = sAl + SM::kA;
    if (tid == 0)
      issue_tiles(sB, mma, plane, param_slab, cap, members, m0, S, c, tile_bytes,
                  smem_u32(&full[stage]));
#pragma unroll
    for (int e = 0; e < HALF; ++e) x[e] = dead ? 0.f : ex2(fmaf(x[e], kL2E, -gml));
#pragma unroll
    for (int q = 0; q < HALF / 8; ++q)
      store_split8(sAh, sAl, kmajor_off(row, half * HALF + q * 8, KN), x + q * 8);
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      mbar_wait(smem_u32(&full[stage]), (it >> 1) & 1);
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
      mma_commit(smem_u32(&done[stage]));
    }
    __syncwarp();
    ++it;
    c = cn;
  }
  if (it > 0) {
    mbar_wait(smem_u32(&done[(it - 1) & 1]), ((it - 1) >> 1) & 1);
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
      values[(int64_t)sid * ldb + b] = (dead || !(d > 0.f)) ? PCB_NEG_INF
                                                             : fmaf(lg2(d), kLN2, gm);
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
__global__ void __launch_bounds__(TC_THREADS, (KM <= 32) ? 2 : 1)
    k_child_flow_tc(int cap, int k_n, int B, int ldb, const int32_t* __restrict__ row_off,
                    const int32_t* __restrict__ members, const int32_t* __restrict__ ch_ids,
                    const int32_t* __restrict__ par_ids, const int32_t* __restrict__ ppids,
                    const int32_t* __restrict__ par_slab, const __nv_bfloat16* __restrict__ mma,
                    int64_t plane,
                    const float* __restrict__ values, const float* __restrict__ flows,
                    const float* __restrict__ scratch, const float* __restrict__ rmax,
                    int64_t sb_base, float* __restrict__ flow_scratch) {
  using SM = CfSmem<KM>;
  constexpr int HALF = KM / 2;  // parent sums converted per thread per stage
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t done[2], full[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int row = tid & (TC_M - 1);
  const int half = tid >> 7;
  // 1-D grid, batch tiles of one super-row adjacent so its theta tiles are
  // fetched from HBM once and re-read from L2
  const int ntiles = (B + TC_M - 1) / TC_M;
  const int sr = blockIdx.x / ntiles;
  const int b = (blockIdx.x - sr * ntiles) * TC_M + row;
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
  const float gl2 = dead ? 0.f : gm;  // rmax is in log2 units

  const uint32_t ncols = tmem_cols_for(N);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&done[i]), 1);
      mbar_init(smem_u32(&full[i]), 1);
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(smem_u32(&tmem_base), ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = idesc_bf16_bmn(TC_M, k_n);
  constexpr uint32_t SBO_A = (KM / 8) * 128;
  // MN-major B read from the theta-tile layout: LBO = K-adjacent core stride,
  // SBO = MN-adjacent (pinned by test_tcgen05_mn_major_b_selftest)
  const uint32_t lbo = (uint32_t)(k_n / 8) * 128, sbo = 128u;
  const int tile_bytes = KM * k_n * 4;

  auto load = [&](int p, float* fr, float* lr) {
    const int64_t base = ((int64_t)parow[p] + half * HALF) * ldb + b;
#pragma unroll
    for (int e = 0; e < HALF; ++e) {
      fr[e] = live ? flows[base + (int64_t)e * ldb] : 0.f;
      lr[e] = live ? values[base + (int64_t)e * ldb] : PCB_NEG_INF;
    }
  };
  float fn[HALF], ln[HALF];
  int p = next_real(pprow, cap, 0);
  if (p < cap) load(p, fn, ln);
  int it = 0;
  while (p < cap) {
    float x[HALF];
#pragma unroll
    for (int e = 0; e < HALF; ++e) x[e] = dead ? 0.f : scaled_ratio(fn[e], ln[e], gl2);
    const int pn = next_real(pprow, cap, p + 1);
    if (pn < cap) load(pn, fn, ln);  // prefetch the next parent block
    const int stage = it & 1;
    if (it >= 2) mbar_wait(smem_u32(&done[stage]), ((it - 2) >> 1) & 1);
    uint8_t* sAh = smem + stage * SM::kStage;
    uint8_t* sAl = sAh + SM::kA;
    uint8_t* sB = sAl + SM::kA;
    if (tid == 0)
      issue_tiles(sB, mma, plane, par_slab, cap, members, m0, S, p, tile_bytes,
                  smem_u32(&full[stage]));
#pragma unroll
    for (int q = 0; q < HALF / 8; ++q)
      store_split8(sAh, sAl, kmajor_off(row, half * HALF + q * 8, KM), x + q * 8);
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      mbar_wait(smem_u32(&full[stage]), (it >> 1) & 1);
      tc_fence_after();
      const uint32_t aH = smem_u32(sAh), aL = smem_u32(sAl), bB = smem_u32(sB);
      for (int s = 0; s < S; ++s) {
        const uint32_t bH = bB + s * tile_bytes, bL = bH + tile_bytes / 2;
        const uint32_t d = tmem + s * k_n;
#pragma unroll
        for (int ks = 0; ks < KM / 16; ++ks) {
          const uint32_t oa = ks * 256, ob = ks * 2 * lbo;
          mma_bf16(d, make_desc(aH + oa, 128, SBO_A), make_desc(bH + ob, lbo, sbo), idesc,
                   (it > 0 || ks > 0) ? 1u : 0u);
          mma_bf16(d, make_desc(aH + oa, 128, SBO_A), make_desc(bL + ob, lbo, sbo), idesc, 1u);
          mma_bf16(d, make_desc(aL + oa, 128, SBO_A), make_desc(bH + ob, lbo, sbo), idesc, 1u);
        }
      }
      mma_commit(smem_u32(&done[stage]));
    }
    __syncwarp();
    ++it;
    p = pn;
  }
  if (it > 0) {
    mbar_wait(smem_u32(&done[(it - 1) & 1]), ((it - 1) >> 1) & 1);
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
      // flow = D * 2^g * exp(l_child), evaluated as 2^(log2 D + l log2 e + g)
      flow_scratch[o] = (dead || !(d > 0.f)) ? 0.f
                                              : ex2(lg2(d) + fmaf(scratch[o], kL2E, gm));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free(tmem, ncols);
}

// --------------------------------------------------------------- param flows
// One CTA = one 128-sum M tile of a super-row x up to 256 product columns x
// one slice of the batch (blockIdx.z = mtile + mtiles * kslice; slices
// split the contraction so small layers still fill the machine — the
// epilogue's red.add into f_params sums them).  K = samples streamed 32 at a
// time, two threads per sum row (16 samples each).  c_b = per-sample max of
// rmax over the tile's sum blocks.  Every address is resolved once per CTA
// (shared-memory tables / registers); each chunk's flows, values, child
// values and shifts are loaded into registers one chunk ahead.
constexpr int PF_KC = 32;
constexpr int PF_MAXSB = TC_M / 16 + 1;  // sum blocks a 128-row tile can touch (k_m >= 16)

struct PfSmem {
  static constexpr int kA = TC_M * PF_KC * 2;
  static constexpr int kB = TC_NMAX * PF_KC * 2;
  static constexpr int kStage = 2 * kA + 2 * kB;
  static constexpr int kBytes = 2 * kStage;
};

template <int KN>
__global__ void __launch_bounds__(TC_THREADS, 2)
    k_param_flow_tc(int cap, int k_m, int B, int ldb, int mtiles, int kslices,
                    const int32_t* __restrict__ row_off, const int32_t* __restrict__ members,
                    const int32_t* __restrict__ sum_ids, const int32_t* __restrict__ prod_ids,
                    const int32_t* __restrict__ param_ids, const int32_t* __restrict__ flow_ids,
                    const float* __restrict__ theta, const float* __restrict__ values,
                    const float* __restrict__ flows, const float* __restrict__ scratch,
                    const float* __restrict__ rmax, int64_t sb_base, float* __restrict__ f_params) {
  constexpr int HS = PF_KC / 2;               // samples per thread per chunk (A side)
  constexpr int BQ = TC_NMAX * (PF_KC / 8) / TC_THREADS;  // B items per thread (max)
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t done[2];
  __shared__ uint32_t tmem_base;
  __shared__ float cb[2][PF_KC];
  __shared__ int cols[TC_NMAX / 16];
  __shared__ int64_t rblk[PF_MAXSB];
  __shared__ int ncols_s, nrblk_s;
  constexpr int CPG = TC_NMAX / KN;  // child columns per CTA
  const int tid = threadIdx.x, warp = tid >> 5;
  const int sr = blockIdx.x;
  const int cg = blockIdx.y;
  const int mt = blockIdx.z % mtiles;
  const int ks = blockIdx.z / mtiles;
  const int m0 = row_off[sr];
  const int S = row_off[sr + 1] - m0;
  const int Nsum = S * k_m;
  if (mt * TC_M >= Nsum) return;
  // this CTA's batch slice, in whole chunks
  const int nchunks = (B + PF_KC - 1) / PF_KC;
  const int per = (nchunks + kslices - 1) / kslices;
  const int kc0 = ks * per, kc1 = min(nchunks, kc0 + per);
  if (kc0 >= kc1) return;
  const int r0 = members[m0];
  const int32_t* trow = param_ids + (int64_t)r0 * cap;
  const int s_lo = (mt * TC_M) / k_m;
  const int s_hi = (min(mt * TC_M + TC_M, Nsum) - 1) / k_m;
  if (tid == 0) {
    int seen = 0, n = 0;
    for (int c = 0; c < cap; ++c) {
      if (trow[c] == 0) continue;
      if (seen >= cg * CPG && n < CPG) cols[n++] = c;
      ++seen;
    }
    ncols_s = n;
    for (int s = s_lo; s <= s_hi; ++s)
      rblk[s - s_lo] = (int64_t)(sum_ids[members[m0 + s]] - sb_base) / k_m * ldb;
    nrblk_s = s_hi - s_lo + 1;
  }
  __syncthreads();
  const int ncol = ncols_s;
  if (ncol == 0) return;
  const int Npad = ncol * KN;
  const int arow = tid & (TC_M - 1);     // A row within the tile
  const int ahalf = tid >> 7;            // which 16 samples of the chunk
  const int ms = mt * TC_M + arow;       // sum index within the super-row
  const bool row_live = ms < Nsum;
  int sum_slot = 0;
  if (row_live) sum_slot = sum_ids[members[m0 + ms / k_m]] + (ms % k_m);
  const int nrb = nrblk_s;

  const uint32_t ncols_t = tmem_cols_for(Npad);
  if (tid == 0) {
    mbar_init(smem_u32(&done[0]), 1);
    mbar_init(smem_u32(&done[1]), 1);
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
  const int nitems = Npad * (PF_KC / 8);

  // per-thread B items: the scratch row (constant over chunks) and smem slot
  const float* bsrc[BQ];
  int bn[BQ], bk[BQ];
#pragma unroll
  for (int u = 0; u < BQ; ++u) {
    const int q = tid + u * TC_THREADS;
    const int n = q / (PF_KC / 8), kq = q - n * (PF_KC / 8);
    bn[u] = n;
    bk[u] = kq;
    bsrc[u] = (q < nitems) ? scratch + (int64_t)(prow[cols[n / KN]] + n % KN) * ldb + kq * 8
                           : nullptr;
  }
  const float* fsrc = flows + (int64_t)sum_slot * ldb + ahalf * HS;
  const float* vsrc = values + (int64_t)sum_slot * ldb + ahalf * HS;

  float fn[HS], ln[HS], ev[BQ][8], cbn = PCB_NEG_INF;
  auto load_chunk = [&](int b0) {
    if (row_live) {
      const float4* fp = reinterpret_cast<const float4*>(fsrc + b0);
      const float4* vp = reinterpret_cast<const float4*>(vsrc + b0);
#pragma unroll
      for (int q = 0; q < HS / 4; ++q) {
        const float4 f = fp[q], v = vp[q];
        fn[4 * q] = f.x, fn[4 * q + 1] = f.y, fn[4 * q + 2] = f.z, fn[4 * q + 3] = f.w;
        ln[4 * q] = v.x, ln[4 * q + 1] = v.y, ln[4 * q + 2] = v.z, ln[4 * q + 3] = v.w;
      }
    }
#pragma unroll
    for (int u = 0; u < BQ; ++u) {
      if (bsrc[u]) {
        const float4 x0 = *reinterpret_cast<const float4*>(bsrc[u] + b0);
        const float4 x1 = *reinterpret_cast<const float4*>(bsrc[u] + b0 + 4);
        ev[u][0] = x0.x, ev[u][1] = x0.y, ev[u][2] = x0.z, ev[u][3] = x0.w;
        ev[u][4] = x1.x, ev[u][5] = x1.y, ev[u][6] = x1.z, ev[u][7] = x1.w;
      }
    }
    if (tid < PF_KC) {  // per-sample shift of this chunk
      float v = PCB_NEG_INF;
      if (b0 + tid < B)
        for (int i = 0; i < nrb; ++i) v = fmaxf(v, rmax[rblk[i] + b0 + tid]);
      cbn = v;
    }
  };
  load_chunk(kc0 * PF_KC);
  int it = 0;
  for (int kc = kc0; kc < kc1; ++kc, ++it) {
    const int b0 = kc * PF_KC;
    const int stage = it & 1;
    if (it >= 2) mbar_wait(smem_u32(&done[stage]), ((it - 2) >> 1) & 1);
    if (tid < PF_KC) cb[stage][tid] = cbn;
    __syncthreads();
    uint8_t* sAh = smem + stage * PfSmem::kStage;
    uint8_t* sAl = sAh + PfSmem::kA;
    uint8_t* sBh = sAl + PfSmem::kA;
    uint8_t* sBl = sBh + PfSmem::kB;
    const float* cbs = cb[stage];
    {
      float x[HS];
#pragma unroll
      for (int e = 0; e < HS; ++e) {
        const int q = ahalf * HS + e;
        const float c = cbs[q];
        x[e] = (!row_live || c == PCB_NEG_INF || b0 + q >= B)
                   ? 0.f
                   : scaled_ratio(fn[e], ln[e], c);
      }
#pragma unroll
      for (int kq = 0; kq < HS / 8; ++kq)
        store_split8(sAh, sAl, kmajor_off(arow, ahalf * HS + kq * 8, PF_KC), x + kq * 8);
    }
#pragma unroll
    for (int u = 0; u < BQ; ++u) {
      if (bsrc[u]) {
        float x[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float c = cbs[bk[u] * 8 + e];
          x[e] = (c == PCB_NEG_INF) ? 0.f : fminf(ex2(fmaf(ev[u][e], kL2E, c)), 1e37f);
        }
        store_split8(sBh, sBl, kmajor_off(bn[u], bk[u] * 8, PF_KC), x);
      }
    }
    if (kc + 1 < kc1) load_chunk(b0 + PF_KC);  // next chunk's operands, in flight during the MMA
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t aH = smem_u32(sAh), aL = smem_u32(sAl);
      const uint32_t bH = smem_u32(sBh), bL = smem_u32(sBl);
#pragma unroll
      for (int kk = 0; kk < PF_KC / 16; ++kk) {
        const uint32_t o = kk * 256;
        mma_bf16(tmem, make_desc(aH + o, 128, SBO), make_desc(bH + o, 128, SBO), idesc,
                 (it > 0 || kk > 0) ? 1u : 0u);
        mma_bf16(tmem, make_desc(aH + o, 128, SBO), make_desc(bL + o, 128, SBO), idesc, 1u);
        mma_bf16(tmem, make_desc(aL + o, 128, SBO), make_desc(bH + o, 128, SBO), idesc, 1u);
      }
      mma_commit(smem_u32(&done[stage]));
    }
    __syncwarp();
  }
  mbar_wait(smem_u32(&done[(it - 1) & 1]), ((it - 1) >> 1) & 1);
  tc_fence_after();
  // epilogue: warps w and w+4 share TMEM lanes 32 (w%4) ..; they split the chunks
  const int er = mt * TC_M + (warp & 3) * 32 + (tid & 31);
  const bool live = er < Nsum;
  int s = 0, mm = 0;
  if (live) {
    s = er / k_m;
    mm = er - s * k_m;
  }
  const int64_t rowbase = (int64_t)members[m0 + (live ? s : 0)] * cap;
  for (int c0 = (warp >> 2) * 16; c0 < Npad; c0 += 32) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)((warp & 3) * 32) << 16) + c0, v);
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
  const unsigned grid = (unsigned)(tc.count * ((B + TC_M - 1) / TC_M));
  k_sum_fwd_tc<KN><<<grid, TC_THREADS, FwdSmem<KN>::kBytes, s>>>(
      (int)g.cap, (int)L.k_m, B, ldb, tc.row_off, tc.members, g.sum_ids, g.prod_ids,
      g.param_ids, g.param_slab, P->mma, P->mma_plane, scratch, bmax, values);
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
  const unsigned grid = (unsigned)(tc.count * ((B + TC_M - 1) / TC_M));
  k_child_flow_tc<KM><<<grid, TC_THREADS, CfSmem<KM>::kBytes, s>>>(
      (int)g.cap, (int)L.k_n, B, ldb, tc.row_off, tc.members, g.ch_ids, g.par_ids,
      g.par_param_ids, g.par_slab, P->mma, P->mma_plane, values, flows, scratch, rmax, L.sb_base,
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
  const int mtiles = (int)((TC_NMAX + TC_M - 1) / TC_M);  // super-rows hold <= 256 sums
  // split the batch so a layer launches >= ~2 waves of 2 CTAs/SM; each slice
  // keeps >= 2 chunks so the register prefetch still has something to hide
  const int64_t base = (int64_t)tc.count * cgroups * mtiles;
  const int nchunks = (B + PF_KC - 1) / PF_KC;
  int kslices = (int)((4 * 148 + base - 1) / base);
  kslices = max(1, min(kslices, nchunks / 2));
  dim3 grid((unsigned)tc.count, (unsigned)cgroups, (unsigned)(mtiles * kslices));
  k_param_flow_tc<KN><<<grid, TC_THREADS, PfSmem::kBytes, s>>>(
      (int)g.cap, (int)L.k_m, B, ldb, mtiles, kslices, tc.row_off, tc.members, g.sum_ids,
      g.prod_ids, g.param_ids, g.flow_ids, theta, values, flows, scratch, rmax, L.sb_base,
      f_params);
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
