// Warp-specialised, persistent tcgen05 sum-layer kernels for sm_100a:
// the sum forward (engine.py:74-102) and the child flows (engine.py:129-165).
//
// Both are "transform + GEMM" over node-major fp32 rows:
//   forward     D[b, n] = sum_j e^{child[j,b] - g_b} theta[n, j]      (A = children)
//   child flow  D[b, j] = sum_m e^{lnf[m,b] - g_b} theta[m, j]         (A = parent ratios)
// Log values are (integer block base, fp32 offset) pairs (pcb_internal.cuh):
// the forward shift g_b is the max of the K blocks' bases G (the output
// base; a K block enters as offset + (base - G)); the child flows move
// every parent block's ratio onto a common base Gr (max of the parents'
// bases) and every product block's offset back onto its own base in the
// epilogue.  All base arithmetic is exact integer differences.
// with M = 128 samples per work item, N = a stacked super-row (<= 256) and K
// streamed one child (parent) block at a time.  A work item is one
// (super-row, 128-sample tile); CTAs are persistent (one per SM, TMEM
// 2 x 256 columns double-buffers the accumulator) and take items round-robin
// so the batch tiles of one super-row run side by side and share its theta
// tiles through L2.
//
// Warp roles (20 warps):
//   warp 0      raw producer: one 2-D TMA box (cp.async.bulk.tensor) of the
//               K block's fp32 rows x 128 samples per source array into the
//               raw ring;
//   warp 18     theta producer: 1-D bulk copies of the stacked pre-split bf16
//               theta planes into the theta ring (4 stages at block 32);
//   warp 1      MMA issuer: three kind::f16 MMAs per 16-wide K step
//               (hi*hi + hi*lo + lo*hi, fp32 accumulation in TMEM; A_hi kept
//               in the operand collector for the second), commits free A and
//               theta stages and publishes finished accumulators;
//   warps 2-9   converters: thread = (sample, K half); raw row values -> shifted
//               exponential (MUFU ex2, shift folded into one FFMA) -> packed
//               bf16 hi/lo planes in the K-major core-matrix layout (A ring);
//   warp 19     shift warp: per-sample shift g_b of the next item (max of the
//               block bases / ratio shifts over its K blocks), live-K count,
//               output rows -- for long K with one item per CTA computed at
//               kernel start by warps 2-17 and 19 together;
//   warps 10-17 epilogue: TMEM -> registers -> log-domain result -> coalesced
//               fp32 row stores (two warps per TMEM lane quarter, alternate
//               16-column chunks); split K: partial sums reduced in L2, then
//               the co-resident slices each finish a share of the columns (or
//               the last arrival finishes the item).
// Every hand-off is an mbarrier: raw full/empty, A full/empty, theta
// full/empty, accumulator full/empty, shift full/empty.
#include <math.h>
#include <stdlib.h>

#include "pcb_internal.cuh"
#include "pcb_tc.cuh"
#include "pcb_ws.cuh"

namespace pcb {

using namespace tc;
using namespace ws;

namespace {

constexpr int WS_M = 128;           // samples per item
constexpr int WS_NMAX = 256;        // stacked N per item
constexpr int WS_PRODUCER = 0, WS_MMA = 1, WS_CONV0 = 2;

// warp layout: producer, MMA, NCONV converter warps (128 / 256 threads: one
// or two per sample, splitting each K block), 8 epilogue warps, the theta
// producer and the shift warp
template <int NCONV>
struct WsWarps {
  static constexpr int kConv = NCONV;
  static constexpr int kEpi0 = WS_CONV0 + NCONV;
  static constexpr int kTheta = kEpi0 + 8;
  static constexpr int kShift = kTheta + 1;
  static constexpr int kThreads = (kShift + 1) * 32;
};

enum { MODE_FWD = 0, MODE_CF = 1 };

struct WsArgs {
  int cap;        // K blocks per group row
  int nb;         // N of one stacked tile (k_m forward, k_n child flow)
  int B, ldb;
  int n_items, ntiles;
  int kslices, kper;               // K split: slice ks covers real columns [ks * kper, +kper)
  int64_t sb_base;                 // shift-row base (child flow: first sum-block slot)
  const int32_t* row_off;          // super-row -> members
  const int32_t* members;          // group rows
  const int32_t* out_ids;          // sum_ids (fwd) / ch_ids (cf): first output row per member
  const int32_t* src_ids;          // prod_ids (fwd) / par_ids (cf): first source row per column
  const int32_t* real_ids;         // param_ids (fwd) / par_param_ids (cf): 0 = padding column
  const int32_t* slab;             // bf16 hi-plane offset per (member, column); lo = + plane
  const int32_t* flags;            // per super-row: bit 2 = stacked tiles contiguous
  int64_t plane;                   // elements per plane region of the bf16 theta copy
  const __nv_bfloat16* mma;
  const float* src0;               // scratch (fwd) / ratio rows r (cf, from sb_base)
  const float* shift;              // pbase (fwd) / rmax R (cf), layer rows
  const float* aux;                // - / scratch (cf epilogue: child log values)
  float* out;                      // values (fwd) / flow_scratch (cf)
  float* vbase;                    // fwd: the layer's sum-block base rows (written)
  const float* vbase_in;           // cf: the layer's sum-block base rows
  const float* pbase_in;           // cf: the layer's product-block base rows
  int64_t out_base;                // fwd: first sum slot of the layer (vbase row of a slot)
  int32_t* counters;               // split-K arrivals per (super-row, tile)
  const float* gshift;             // precomputed per-(super-row, sample) shifts, or null
  const float* gbase;              // cf: precomputed per-(super-row, sample) common bases Gr
  int64_t gshift_stride;           // ldb, or 0 when every super-row shares one shift row
  int coop;                        // long K, one item per CTA: shifts computed in-kernel
  int split_finish;                // coop split K: every slice finishes a share of the columns
  float* part;                     // coop split K: this launch's partial-sum slab (or null)
};

struct WsItem {
  int sr, tile, ks, b0, m0, S, r0;
};

// item = tile + ntiles * (slice + kslices * super-row): the tiles and slices of
// one super-row run side by side (theta tiles shared through L2)
__device__ __forceinline__ WsItem ws_item(const WsArgs& a, int item) {
  WsItem it;
  it.tile = item % a.ntiles;
  const int q = item / a.ntiles;
  it.ks = q % a.kslices;
  it.sr = q / a.kslices;
  it.b0 = it.tile * WS_M;
  it.m0 = a.row_off[it.sr];
  it.S = a.row_off[it.sr + 1] - it.m0;
  it.r0 = a.members[it.m0];
  return it;
}

// the first real column of the item's K slice
__device__ __forceinline__ int slice_first(const int32_t* __restrict__ real, int cap, int skip) {
  int c = next_real(real, cap, 0);
  for (int k = 0; k < skip && c < cap; ++k) c = next_real(real, cap, c + 1);
  return c;
}

// rows whose columns are all real (TcRows flags bit 3) step arithmetically
__device__ __forceinline__ bool dense_row(const WsArgs& a, const WsItem& it) {
  return a.flags && (__ldg(a.flags + it.sr) & 8);
}
__device__ __forceinline__ int col_first(const int32_t* __restrict__ real, int cap, int skip,
                                         bool dense) {
  return dense ? min(skip, cap) : slice_first(real, cap, skip);
}
__device__ __forceinline__ int col_next(const int32_t* __restrict__ real, int cap, int c,
                                        bool dense) {
  return dense ? c : next_real(real, cap, c);
}

template <int MODE, int KC>
struct WsCfg {
  // raw rows per stage: the K block's rows (forward: child offsets; child
  // flow: shifted log2 flow ratios r) + the block's base row (forward) / its
  // shift row R and base row (child flow)
  static constexpr int kRows = KC + (MODE == MODE_CF ? 2 : 1);
  static constexpr int kRaw = kRows * WS_M * 4;               // raw stage bytes
  static constexpr int kA = WS_M * KC * 2;                    // one bf16 A plane
  static constexpr int kBPlane = WS_NMAX * KC * 2;            // stacked theta hi (or lo) plane
  static constexpr int kB = 2 * kBPlane;
#ifndef PCB_WS_BUDGET
#define PCB_WS_BUDGET 220
#endif
  static constexpr int kBudget = PCB_WS_BUDGET * 1024;
  // separate rings for the converted A planes (converters -> MMA) and the
  // theta planes (bulk copies -> MMA): the theta stream gets the depth to
  // cover its L2 / HBM latency (4 stages of 32 KB at KC = 32, was 2 shared
  // stages: HMM-4096 sum forward 1.75 -> 1.63 ms, child flows 2.24 -> 2.03),
  // the converters' A ring stays shallow (its input is the raw ring)
#ifndef PCB_WS_AS
#define PCB_WS_AS 2
#endif
#ifndef PCB_WS_BS
#define PCB_WS_BS 4
#endif
  static constexpr int kAS = (KC <= 16) ? 4 : PCB_WS_AS;
  static constexpr int kBS = (KC <= 16) ? 4 : PCB_WS_BS;
  static constexpr int kRSmax = (kBudget - kAS * 2 * kA - kBS * kB) / kRaw;
  static constexpr int kRS = kRSmax > 8 ? 8 : kRSmax;
  static constexpr int kBytes = kRS * kRaw + kAS * 2 * kA + kBS * kB;
  static_assert(kRS >= 2, "raw ring too small");
  static constexpr int kNConv = 8;  // converter warps: two threads per sample
};

}  // namespace

template <int MODE, int KC>
__global__ void __launch_bounds__(WsWarps<WsCfg<MODE, KC>::kNConv>::kThreads, 1)
    k_sum_ws(const WsArgs a, const __grid_constant__ CUtensorMap tm0,
             const __grid_constant__ CUtensorMap tm1, const __grid_constant__ CUtensorMap tm2) {
  pdl_enter();
  using C = WsCfg<MODE, KC>;
  using W = WsWarps<C::kNConv>;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t raw_full[C::kRS], raw_empty[C::kRS];
  __shared__ uint64_t a_full[C::kAS], a_empty[C::kAS], b_full[C::kBS], b_empty[C::kBS];
  __shared__ uint64_t acc_full[2], acc_empty[2], g_full[2], g_empty[2];
  __shared__ float g_s[2][WS_M];
  __shared__ float gr_s[2][WS_M];        // child flow: the common parent base Gr
  __shared__ int g_nk[2];                // real K blocks of the item (0: dead)
  __shared__ int g_orow[2][WS_NMAX / 16];  // first output row of every 16 columns
  __shared__ bool g_last;
  __shared__ uint32_t tmem_base;
  __shared__ int cs_g[WS_M], cs_gr[WS_M];  // coop shifts: order-preserving ints
  uint8_t* raw = smem;
  uint8_t* aops = smem + C::kRS * C::kRaw;       // A ring: hi plane, lo plane per stage
  uint8_t* bops = aops + C::kAS * 2 * C::kA;       // theta ring: hi planes, lo planes

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < C::kRS; ++i) {
      mbar_init(smem_u32(&raw_full[i]), 1);
      mbar_init(smem_u32(&raw_empty[i]), W::kConv);
    }
    for (int i = 0; i < C::kAS; ++i) {
      mbar_init(smem_u32(&a_full[i]), W::kConv);  // converter warps
      mbar_init(smem_u32(&a_empty[i]), 1);
    }
    for (int i = 0; i < C::kBS; ++i) {
      mbar_init(smem_u32(&b_full[i]), 1);  // theta producer (+ tx)
      mbar_init(smem_u32(&b_empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&acc_full[i]), 1);
      mbar_init(smem_u32(&acc_empty[i]), 8);
      mbar_init(smem_u32(&g_full[i]), 1);               // the shift warp
      mbar_init(smem_u32(&g_empty[i]), W::kConv + 8);   // converters + epilogue warps
    }
    fence_mbar_init();
  }
  if (warp == WS_MMA) tmem_alloc(smem_u32(&tmem_base), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const int plane_bytes = a.nb * KC * 2;  // one bf16 plane of one theta tile

  // Long K with one item per CTA: the item's per-sample shifts (what
  // k_group_shift would precompute) come from the 17 converter, epilogue and
  // shift warps together while the producers start streaming -- one round of
  // loads per warp (lane = sample, 8 K blocks per warp), then order-preserving
  // integer max reductions in shared memory.  Child flow: each thread keeps
  // (gr, g) online; the partial g are moved onto the common gr before the
  // second reduction.
  const bool coop = a.coop && warp >= WS_CONV0 && warp != W::kTheta;
  if (coop) {
    constexpr int NW = W::kShift - WS_CONV0;  // converters + epilogue + shift (theta excluded)
    const int wr = (warp == W::kShift) ? NW - 1 : warp - WS_CONV0;
    const int ct = wr * 32 + lane;
    auto ord = [](float f) {
      const int i = __float_as_int(f);
      return i >= 0 ? i : i ^ 0x7fffffff;
    };
    auto unord = [](int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); };
    for (int q = ct; q < WS_M; q += NW * 32) cs_g[q] = cs_gr[q] = ord(PCB_NEG_INF);
    asm volatile("bar.sync 3, %0;" ::"n"(NW * 32) : "memory");
    const WsItem it = ws_item(a, blockIdx.x);
    const int32_t* src = a.src_ids + (int64_t)it.r0 * a.cap;
    const int32_t* real = a.real_ids + (int64_t)it.r0 * a.cap;
    constexpr int SPL = WS_M / 32;
    float g[SPL], gr[SPL];
#pragma unroll
    for (int u = 0; u < SPL; ++u) g[u] = gr[u] = PCB_NEG_INF;
    for (int c0 = wr; c0 < a.cap; c0 += NW * 4) {
      float v[4][SPL], w[4][SPL];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int c = c0 + NW * e;
        const int sc = (c < a.cap && __ldg(real + c) != 0) ? __ldg(src + c) : -1;
#pragma unroll
        for (int u = 0; u < SPL; ++u) {
          const int b = it.b0 + lane + 32 * u;
          const bool ok = sc >= 0 && b < a.B;
          const int64_t o = (int64_t)(sc - a.sb_base) / KC * a.ldb + b;
          v[e][u] = ok ? __ldg(a.shift + o) : PCB_NEG_INF;
          w[e][u] = (MODE == MODE_CF && ok) ? __ldg(a.vbase_in + o) : PCB_NEG_INF;
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e)
#pragma unroll
        for (int u = 0; u < SPL; ++u) {
          if (MODE == MODE_FWD) {
            g[u] = fmaxf(g[u], v[e][u]);
          } else if (w[e][u] != PCB_NEG_INF) {
            if (w[e][u] > gr[u]) {
              if (g[u] != PCB_NEG_INF) g[u] += (w[e][u] - gr[u]) * kL2E;
              gr[u] = w[e][u];
            }
            g[u] = fmaxf(g[u], fmaf(gr[u] - w[e][u], kL2E, v[e][u]));
          }
        }
    }
    if (MODE == MODE_CF) {
#pragma unroll
      for (int u = 0; u < SPL; ++u)
        if (gr[u] != PCB_NEG_INF) atomicMax(&cs_gr[lane + 32 * u], ord(gr[u]));
      asm volatile("bar.sync 3, %0;" ::"n"(NW * 32) : "memory");
#pragma unroll
      for (int u = 0; u < SPL; ++u) {
        const float G = unord(cs_gr[lane + 32 * u]);
        if (g[u] != PCB_NEG_INF) g[u] += (G - gr[u]) * kL2E;  // onto the common base
      }
    }
#pragma unroll
    for (int u = 0; u < SPL; ++u)
      if (g[u] != PCB_NEG_INF) atomicMax(&cs_g[lane + 32 * u], ord(g[u]));
    asm volatile("bar.sync 3, %0;" ::"n"(NW * 32) : "memory");
    for (int q = ct; q < WS_M; q += NW * 32) {
      g_s[0][q] = unord(cs_g[q]);
      gr_s[0][q] = unord(cs_gr[q]);
    }
    asm volatile("bar.sync 3, %0;" ::"n"(NW * 32) : "memory");
  }

  if (warp == WS_PRODUCER) {
    // ------------------------------------------------------------ raw producer
    // one 2-D TMA box [KC rows x 128 samples] per source array and K block;
    // samples past ldb are zero-filled by the TMA unit
    if (lane == 0) {
      prefetch_tmap(&tm0);
      prefetch_tmap(&tm1);
      if (MODE == MODE_CF) prefetch_tmap(&tm2);
      Ring<C::kRS> rr;
      for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
        const WsItem it = ws_item(a, item);
        const int b0 = it.b0;
        const int32_t* src = a.src_ids + (int64_t)it.r0 * a.cap;
        const int32_t* real = a.real_ids + (int64_t)it.r0 * a.cap;
        const bool dn = dense_row(a, it);
      int c = col_first(real, a.cap, it.ks * a.kper, dn);
        for (int k = 0; c < a.cap && k < a.kper; ++k, c = col_next(real, a.cap, c + 1, dn)) {
          const int row0 = __ldg(src + c) - (int)a.sb_base;
          mbar_wait(smem_u32(&raw_empty[rr.slot()]), rr.empty_par());
          const uint32_t rf = smem_u32(&raw_full[rr.slot()]);
          mbar_arrive_expect_tx(rf, (uint32_t)C::kRaw);
          const uint32_t dst = smem_u32(raw + rr.slot() * C::kRaw);
          tma_load_2d(dst, &tm0, b0, row0, rf);
          tma_load_2d(dst + KC * WS_M * 4, &tm1, b0, row0 / KC, rf);
          if (MODE == MODE_CF) tma_load_2d(dst + (KC + 1) * WS_M * 4, &tm2, b0, row0 / KC, rf);
          rr.next();
        }
      }
    }
  } else if (warp == W::kTheta) {
    // ------------------------------------------------------------ theta producer
    // stacked theta tiles of each K block: hi planes back to back, then lo
    // planes, so the S tiles form one N = S * nb operand per plane
    Ring<C::kBS> brr;
    for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
      const WsItem it = ws_item(a, item);
      const int m0 = it.m0, S = it.S;
      const int32_t* real = a.real_ids + (int64_t)it.r0 * a.cap;
      const bool contig = a.flags && (__ldg(a.flags + it.sr) & 4);
      const bool dn = dense_row(a, it);
      int c = col_first(real, a.cap, it.ks * a.kper, dn);
      for (int k = 0; c < a.cap && k < a.kper; ++k, c = col_next(real, a.cap, c + 1, dn)) {
        mbar_wait(smem_u32(&b_empty[brr.slot()]), brr.empty_par());
        const uint32_t of = smem_u32(&b_full[brr.slot()]);
        uint8_t* bdst = bops + brr.slot() * C::kB;
        if (lane == 0) mbar_arrive_expect_tx(of, (uint32_t)(2 * S * plane_bytes));
        __syncwarp();
        if (contig) {  // the S tiles of this column are one run per plane
          if (lane < 2) {
            const int64_t slab = __ldg(a.slab + (int64_t)__ldg(a.members + m0) * a.cap + c);
            bulk_g2s(smem_u32(bdst + lane * C::kBPlane), a.mma + slab + lane * a.plane,
                     (uint32_t)(S * plane_bytes), of);
          }
        } else {
          for (int q = lane; q < 2 * S; q += 32) {
            const int s = q >> 1, lo = q & 1;
            const int64_t slab = __ldg(a.slab + (int64_t)__ldg(a.members + m0 + s) * a.cap + c);
            bulk_g2s(smem_u32(bdst + lo * C::kBPlane + s * plane_bytes), a.mma + slab + lo * a.plane,
                     (uint32_t)plane_bytes, of);
          }
        }
        brr.next();
      }
    }
  } else if (warp == WS_MMA) {
    // ------------------------------------------------------------ MMA issuer
    Ring<C::kAS> arr;
    Ring<C::kBS> brr;
    int acc_u = 0;
    constexpr uint32_t SBO = (KC / 8) * 128;  // A and B both K-major, no swizzle
    for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
      const WsItem it = ws_item(a, item);
      const int S = it.S;
      const int32_t* real = a.real_ids + (int64_t)it.r0 * a.cap;
      const int as = acc_u & 1;
      mbar_wait(smem_u32(&acc_empty[as]), (uint32_t)(((acc_u >> 1) & 1) ^ 1));
      tc_fence_after();
      const uint32_t d0 = tmem + (uint32_t)(as * WS_NMAX);
      bool first = true;
      const bool dn = dense_row(a, it);
      int c = col_first(real, a.cap, it.ks * a.kper, dn);
      for (int k = 0; c < a.cap && k < a.kper; ++k, c = col_next(real, a.cap, c + 1, dn)) {
        mbar_wait(smem_u32(&b_full[brr.slot()]), brr.full_par());
        mbar_wait(smem_u32(&a_full[arr.slot()]), arr.full_par());
        tc_fence_after();
        if (lane == 0) {
          const uint32_t aH = smem_u32(aops + arr.slot() * 2 * C::kA), aL = aH + C::kA;
          const uint32_t bH = smem_u32(bops + brr.slot() * C::kB), bL = bH + C::kBPlane;
          const uint32_t idesc = idesc_bf16(WS_M, S * a.nb);
#pragma unroll
          for (int ks = 0; ks < KC / 16; ++ks) {
            const uint64_t ah = make_desc(aH + ks * 256, 128, SBO);
            const uint64_t al = make_desc(aL + ks * 256, 128, SBO);
            const uint64_t bh = make_desc(bH + ks * 256, 128, SBO);
            const uint64_t bl = make_desc(bL + ks * 256, 128, SBO);
            mma_bf16_keep_a(d0, ah, bh, idesc, (first && ks == 0) ? 0u : 1u);
            mma_bf16_reuse_a(d0, ah, bl, idesc, 1u);
            mma_bf16(d0, al, bh, idesc, 1u);
          }
          mma_commit(smem_u32(&a_empty[arr.slot()]));
          mma_commit(smem_u32(&b_empty[brr.slot()]));
        }
        __syncwarp();
        first = false;
        arr.next();
        brr.next();
      }
      if (lane == 0) {
        if (first)
          mbar_arrive(smem_u32(&acc_full[as]));  // no K block: nothing to wait for
        else
          mma_commit(smem_u32(&acc_full[as]));
      }
      __syncwarp();
      ++acc_u;
    }
  } else if (warp < W::kEpi0) {
    // ------------------------------------------------------------ converters
    const int t = (tid - WS_CONV0 * 32) & (WS_M - 1);  // sample within the item
    const int kh = (tid - WS_CONV0 * 32) / WS_M;        // which part of each K block
    constexpr int KH = KC * 4 / W::kConv;                // K columns per converter thread
    Ring<C::kRS> rr;
    Ring<C::kAS> arr;
    int g_u = 0;
    for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
      const WsItem it = ws_item(a, item);
      const int b = it.b0 + t;
      const bool live = b < a.B;
      const int32_t* real = a.real_ids + (int64_t)it.r0 * a.cap;
      const int gs = g_u & 1;
      mbar_wait(smem_u32(&g_full[gs]), (uint32_t)((g_u >> 1) & 1));
      const float g = g_s[gs][t];
      const float gr = gr_s[gs][t];
      const bool dead = !live || g == PCB_NEG_INF;
      // forward: g is the integer base G (natural log); child flow: g is in
      // log2 units, gr the common base of the parent blocks
      const float gl2 = dead ? 0.f : g;
      const bool dn = dense_row(a, it);
      int c = col_first(real, a.cap, it.ks * a.kper, dn);
      for (int k = 0; c < a.cap && k < a.kper; ++k, c = col_next(real, a.cap, c + 1, dn)) {
        mbar_wait(smem_u32(&raw_full[rr.slot()]), rr.full_par());
        const float* rs = reinterpret_cast<const float*>(raw + rr.slot() * C::kRaw);
        float x[KH];
        const float* rh = rs + kh * KH * WS_M;
        float d;
        if (MODE == MODE_FWD) {
          // (base_block - G) log2 e: an exact integer difference (-inf for an
          // all -inf block), added to offset log2 e in one FFMA
          d = (rs[KC * WS_M + t] - gl2) * kL2E;
#pragma unroll
          for (int j = 0; j < KH; ++j) x[j] = rh[j * WS_M + t];
        } else {
          // r + (R_block + (Gr - base_block) log2 e - g): small, (near-)exact
          d = fmaf(gr - rs[(KC + 1) * WS_M + t], kL2E, rs[KC * WS_M + t]) - gl2;
#pragma unroll
          for (int j = 0; j < KH; ++j) x[j] = rh[j * WS_M + t] + d;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&raw_empty[rr.slot()]));
        rr.next();
#pragma unroll
        for (int j = 0; j < KH; ++j) {
          if (MODE == MODE_FWD)
            x[j] = dead ? 0.f : ex2(fmaf(x[j], kL2E, d));
          else
            x[j] = dead ? 0.f : ex2(x[j]);  // ex2(-inf) = 0: impossible sums, zero flow
        }
        mbar_wait(smem_u32(&a_empty[arr.slot()]), arr.empty_par());
        uint8_t* sAh = aops + arr.slot() * 2 * C::kA;
        uint8_t* sAl = sAh + C::kA;
#pragma unroll
        for (int q = 0; q < KH / 8; ++q) {
          float v8[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v8[e] = x[q * 8 + e];
          uint4 hi, lo;
          split_pack8(v8, hi, lo);
          const uint32_t off = kmajor_off(t, kh * KH + q * 8, KC);
          *reinterpret_cast<uint4*>(sAh + off) = hi;
          *reinterpret_cast<uint4*>(sAl + off) = lo;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&a_full[arr.slot()]));
        arr.next();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&g_empty[gs]));
      ++g_u;
    }
  } else if (warp == W::kShift) {
    // ------------------------------------------------------------ shift warp
    // per item, ahead of the converters and the epilogue: the per-sample
    // shift g_b (max of the side maxima bmax / R over the item's K blocks;
    // lane = 4 samples), the number of real K blocks, and the output rows
    // shifts of the lane's 4 samples: the K blocks' ids once (warp-uniform),
    // then the 4 x 8 side maxima of each round in flight together
    constexpr int SPL = WS_M / 32;  // samples per lane
    // forward: g = max of the K blocks' bases; child flow: gr = max of the
    // parent blocks' bases, then g = max of R + (gr - base) log2 e
    auto shifts = [&](const WsItem& it, float* g, float* gr, int& nk) {
      const int64_t r0 = it.r0;
      const int32_t* src = a.src_ids + r0 * a.cap;
      const int32_t* real = a.real_ids + r0 * a.cap;
#pragma unroll
      for (int u = 0; u < SPL; ++u) g[u] = gr[u] = PCB_NEG_INF;
      nk = 0;
      if (a.gshift) {  // long K: shifts precomputed by k_group_shift
        if (dense_row(a, it))
          nk = a.cap;
        else
          for (int c = 0; c < a.cap; ++c) nk += __ldg(real + c) != 0;
#pragma unroll
        for (int u = 0; u < SPL; ++u) {
          const int b = it.b0 + lane + 32 * u;
          if (b < a.B) {
            g[u] = __ldg(a.gshift + (int64_t)it.sr * a.gshift_stride + b);
            if (MODE == MODE_CF) gr[u] = __ldg(a.gbase + (int64_t)it.sr * a.gshift_stride + b);
          }
        }
        return;
      }
      // one pass: child flow keeps (gr, g) online -- raising gr by d raises
      // every earlier R + (gr - base) log2 e term, hence g, by d log2 e
      for (int c0 = 0; c0 < a.cap; c0 += 8) {
        int sc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int c = c0 + e;
          sc[e] = (c < a.cap && __ldg(real + c) != 0) ? __ldg(src + c) : -1;
          nk += sc[e] >= 0;
        }
        float v[SPL][8], w[SPL][8];
#pragma unroll
        for (int u = 0; u < SPL; ++u) {
          const int b = it.b0 + lane + 32 * u;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const bool ok = sc[e] >= 0 && b < a.B;
            const int64_t o = (int64_t)(sc[e] - a.sb_base) / KC * a.ldb + b;
            v[u][e] = ok ? __ldg(a.shift + o) : PCB_NEG_INF;
            w[u][e] = (MODE == MODE_CF && ok) ? __ldg(a.vbase_in + o) : PCB_NEG_INF;
          }
        }
#pragma unroll
        for (int u = 0; u < SPL; ++u)
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            if (MODE == MODE_FWD) {
              g[u] = fmaxf(g[u], v[u][e]);
            } else if (w[u][e] != PCB_NEG_INF) {
              if (w[u][e] > gr[u]) {
                if (g[u] != PCB_NEG_INF) g[u] += (w[u][e] - gr[u]) * kL2E;
                gr[u] = w[u][e];
              }
              g[u] = fmaxf(g[u], fmaf(gr[u] - w[u][e], kL2E, v[u][e]));
            }
          }
      }
    };
    int g_u = 0;
    for (int item = blockIdx.x; item < a.n_items; item += gridDim.x, ++g_u) {
      const WsItem it = ws_item(a, item);
      const int gs = g_u & 1;
      mbar_wait(smem_u32(&g_empty[gs]), (uint32_t)(((g_u >> 1) & 1) ^ 1));
      int nk = 0;
      if (a.coop && g_u == 0) {  // shifts already in g_s[0] / gr_s[0]
        if (dense_row(a, it))
          nk = a.cap;
        else
          for (int c = 0; c < a.cap; ++c) nk += __ldg(a.real_ids + (int64_t)it.r0 * a.cap + c) != 0;
      } else {
        float gv[SPL], gb[SPL];
        shifts(it, gv, gb, nk);
#pragma unroll
        for (int u = 0; u < SPL; ++u) {
          g_s[gs][lane + 32 * u] = gv[u];
          gr_s[gs][lane + 32 * u] = gb[u];
        }
      }
      const int N = it.S * a.nb;
      if (lane < N / 16) {
        const int c0 = lane * 16, sm = c0 / a.nb;
        g_orow[gs][lane] = __ldg(a.out_ids + __ldg(a.members + it.m0 + sm)) + (c0 - sm * a.nb);
      }
      if (lane == 0) g_nk[gs] = nk;
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&g_full[gs]));
    }
  } else if (warp >= W::kEpi0) {
    // ------------------------------------------------------------ epilogue
    // warps 10..17: lane quarter q4 = warp % 4 (TMEM lanes 32*q4..), column
    // half h (alternate 16-column chunks)
    const int q4 = warp & 3;
    const int h = (warp - W::kEpi0) >> 2;
    const int t = q4 * 32 + lane;          // sample within the item
    int g_u = 0, acc_u = 0;
    for (int item = blockIdx.x; item < a.n_items; item += gridDim.x, ++g_u) {
      const WsItem it = ws_item(a, item);
      const int b = it.b0 + t;
      const bool live = b < a.B;
      const int N = it.S * a.nb;
      const int as = acc_u & 1;
      const int gs = g_u & 1;
      mbar_wait(smem_u32(&g_full[gs]), (uint32_t)((g_u >> 1) & 1));
      // the slot is released at the end of the item (the shift warp runs
      // at most two items ahead, like the TMEM double buffer)
      const float g = g_s[gs][t];
      const float gr = gr_s[gs][t];
      const int nk = g_nk[gs];
      const bool dead = g == PCB_NEG_INF || nk == 0;
      const int* orow_s = g_orow[gs];
      auto out_row = [&](int c0) -> int64_t { return orow_s[c0 >> 4]; };
      // finished result of 16 columns from their fp32 sums d (TMEM or reduced)
      // finished result of 16 columns from their fp32 sums d (TMEM or
      // reduced); forward: offsets ln D from the base G (stored with the
      // first chunk of every sum block); child flow: l = product offsets
      // already moved onto the common base (offset + base_pb - Gr)
      auto finish = [&](int c0, float* o, const float* d, const float* l, float pb) {
        if (MODE == MODE_FWD) {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            o[(int64_t)i * a.ldb] = (dead || !(d[i] > 0.f)) ? PCB_NEG_INF : lg2(d[i]) * kLN2;
          if (c0 % a.nb == 0)
            a.vbase[(out_row(c0) - a.out_base) / a.nb * a.ldb + b] = dead ? 0.f : g;
        } else {
          const float db = pb - gr;  // exact integer difference (-inf: dead block)
#pragma unroll
          for (int i = 0; i < 16; ++i)  // flow = D * 2^g * exp(l) = 2^(log2 D + fma(l, log2 e, g))
            o[(int64_t)i * a.ldb] =
                (dead || !(d[i] > 0.f)) ? 0.f : ex2(lg2(d[i]) + fmaf(l[i] + db, kL2E, g));
        }
      };
      auto load_l = [&](int c0, float* l, float& pb) {
        const int64_t row = out_row(c0);
        const float* lp = a.aux + row * a.ldb + b;
#pragma unroll
        for (int i = 0; i < 16; ++i) l[i] = lp[(int64_t)i * a.ldb];
        pb = __ldg(a.pbase_in + row / a.nb * a.ldb + b);
      };
      mbar_wait(smem_u32(&acc_full[as]), (uint32_t)((acc_u >> 1) & 1));
      tc_fence_after();
      const uint32_t tbase = tmem + (uint32_t)(as * WS_NMAX) + ((uint32_t)(q4 * 32) << 16);
      if (a.kslices == 1) {
        // child flow: the epilogue also reads the children's log values; the
        // next chunk's are loaded before this chunk's TMEM load
        float l[16], ln[16], pb = 0.f, pbn = 0.f;
        if (MODE == MODE_CF && live && h * 16 < N) load_l(h * 16, ln, pbn);
        for (int c0 = h * 16; c0 < N; c0 += 32) {
          if (MODE == MODE_CF) {
#pragma unroll
            for (int i = 0; i < 16; ++i) l[i] = ln[i];
            pb = pbn;
            if (live && c0 + 32 < N) load_l(c0 + 32, ln, pbn);
          }
          float v[16];
          tmem_ld16(tbase + c0, v);
          if (!live) continue;
          if (!nk) {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = 0.f;
          }
          finish(c0, a.out + out_row(c0) * a.ldb + b, v, l, pb);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&acc_empty[as]));
      } else {
        // split K: add this slice's partial sums into the (zeroed) output rows;
        // the last slice to arrive finishes the item from the reduced sums
        const int nks = min(a.kper, max(0, nk - it.ks * a.kper));
        for (int c0 = h * 16; c0 < N; c0 += 32) {
          float v[16];
          tmem_ld16(tbase + c0, v);
          if (!live) continue;
          if (a.part) {  // this slice's partial sums: plain coalesced stores (zeros
                         // for a slice without real K blocks: the finish reads every slice)
            float* pp = a.part + ((int64_t)blockIdx.x * WS_NMAX + c0) * WS_M + t;
#pragma unroll
            for (int i = 0; i < 16; ++i) pp[(int64_t)i * WS_M] = nks ? v[i] : 0.f;
            continue;
          }
          if (!nks) continue;
          float* o = a.out + out_row(c0) * a.ldb + b;
#ifdef PCB_ABL_NOATOMIC  // timing ablation only: wrong results
#pragma unroll
          for (int i = 0; i < 16; ++i) o[(int64_t)i * a.ldb] = v[i];
#else
#pragma unroll
          for (int i = 0; i < 16; ++i) atomicAdd(o + (int64_t)i * a.ldb, v[i]);
#endif
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&acc_empty[as]));
        // arrival protocol (release / acquire by one thread, cumulative over
        // the epilogue barrier -- no per-thread GPU-scope fence)
        asm volatile("bar.sync 2, %0;" ::"n"(8 * 32) : "memory");
        // Co-resident slices (coop: one item per CTA, all CTAs resident):
        // every slice waits for all partial sums, then finishes its own
        // share of the columns -- the finish is spread over the k slices
        // instead of serialised on the last one.  Otherwise the last slice
        // to arrive finishes the whole item.
        const bool spread = a.coop && a.split_finish;
        if (warp == W::kEpi0 && lane == 0) {
          int32_t* cnt = a.counters + it.sr * a.ntiles + it.tile;
          asm volatile("fence.acq_rel.gpu;" ::: "memory");  // this CTA's partial sums first
          const int old = atomicAdd(cnt, 1);
          bool last = old == a.kslices - 1;
          if (spread) {
            int v = old + 1;
            while (v < a.kslices) {
              __nanosleep(64);
              v = atomicAdd(cnt, 0);
            }
            last = true;
          } else if (last) {
            *cnt = 0;  // self-resetting for the next launch
          }
          asm volatile("fence.acq_rel.gpu;" ::: "memory");  // then every slice's partial sums
          g_last = last;
        }
        asm volatile("bar.sync 2, %0;" ::"n"(8 * 32) : "memory");
        if (g_last) {
          int cq0 = 0, cq1 = N;
          if (spread) {  // this slice's columns (16-column aligned)
            const int per = ((N / 16 + a.kslices - 1) / a.kslices) * 16;
            cq0 = min(N, it.ks * per);
            cq1 = min(N, cq0 + per);
          }
          for (int c0 = cq0 + h * 16; c0 < cq1; c0 += 32) {
            if (!live) continue;
            float* o = a.out + out_row(c0) * a.ldb + b;
            float d[16], l[16], pb = 0.f;
            if (a.part) {  // the k slices' partial sums (one CTA per slice)
#pragma unroll
              for (int i = 0; i < 16; ++i) d[i] = 0.f;
              for (int q = 0; q < a.kslices; ++q) {
                const float* pp =
                    a.part + ((int64_t)(it.tile + a.ntiles * (q + a.kslices * it.sr)) * WS_NMAX + c0) *
                                 WS_M + t;
#pragma unroll
                for (int i = 0; i < 16; ++i) d[i] += __ldcg(pp + (int64_t)i * WS_M);
              }
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) d[i] = __ldcg(o + (int64_t)i * a.ldb);
            }
            if (MODE == MODE_CF) load_l(c0, l, pb);
            finish(c0, o, d, l, pb);
          }
        }
        asm volatile("bar.sync 2, %0;" ::"n"(8 * 32) : "memory");  // g_last reuse
        if (spread && warp == W::kEpi0 && lane == 0) {  // second arrival; the last resets
          int32_t* cnt = a.counters + it.sr * a.ntiles + it.tile;
          if (atomicAdd(cnt, 1) == 2 * a.kslices - 1) atomicExch(cnt, 0);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&g_empty[gs]));
      ++acc_u;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == WS_MMA) tmem_free(tmem, 512);
}

namespace {

template <int MODE, int KC>
int launch_ws(const WsArgs& a, int64_t rows0, int64_t rows1, cudaStream_t s) {
  using C = WsCfg<MODE, KC>;
  static int attr[kMaxDev] = {};
  if (ensure_smem((const void*)k_sum_ws<MODE, KC>, C::kBytes, attr)) return PCB_CUDA;
  CUtensorMap tm0, tm1, tm2;
  if (make_rows_map(&tm0, a.src0, rows0, a.ldb, KC)) return PCB_CUDA;
  // per K block one row: the block base (forward) / the ratio shift R and the
  // block base (child flow)
  if (make_rows_map(&tm1, a.shift, rows1, a.ldb, 1)) return PCB_CUDA;
  if (make_rows_map(&tm2, MODE == MODE_CF ? a.vbase_in : a.shift, rows1, a.ldb, 1))
    return PCB_CUDA;
  const int grid = min(a.n_items, sm_count());
  launch_k((k_sum_ws<MODE, KC>), dim3(grid), dim3(WsWarps<C::kNConv>::kThreads), C::kBytes, s, a, tm0, tm1, tm2);
  return check_launch();
}

// per-(super-row, sample) shift of a long-K group over the super-row's real
// K blocks: forward: the max of the blocks' bases; child flow: the common
// base gr = max of the parent blocks' bases (to gbase) and the shift
// max R + (gr - base) log2 e.  CTA = super-row x 32 samples; its 32 warps
// split the K blocks (lane = sample), combined in smem: a 128-block row is
// one round of loads per warp.
constexpr int GS_WARPS = 32;
template <int MODE>
__global__ void __launch_bounds__(GS_WARPS * 32)
    k_group_shift(int cap, int kc, int B, int ldb, int64_t sb_base,
                  const int32_t* __restrict__ row_off, const int32_t* __restrict__ members,
                  const int32_t* __restrict__ src_ids, const int32_t* __restrict__ real_ids,
                  const float* __restrict__ shift, const float* __restrict__ base,
                  float* __restrict__ gout, float* __restrict__ gbase) {
  pdl_enter();
  __shared__ float part[GS_WARPS][33];
  const int sr = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = blockIdx.y * 32 + lane;
  const int64_t r0 = __ldg(members + __ldg(row_off + sr));
  const int32_t* src = src_ids + r0 * cap;
  const int32_t* real = real_ids + r0 * cap;
  auto reduce = [&](const float* tab, float gr) {
    float g = PCB_NEG_INF;
    if (b < B)
      for (int c0 = warp; c0 < cap; c0 += GS_WARPS * 4) {
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + GS_WARPS * u;
          const bool ok = c < cap && __ldg(real + c) != 0;
          const int64_t o = ok ? (int64_t)(__ldg(src + c) - sb_base) / kc * ldb + b : 0;
          v[u] = ok ? __ldg(tab + o) : PCB_NEG_INF;
          if (ok && MODE == MODE_CF && gr != PCB_NEG_INF)
            v[u] = fmaf(gr - __ldg(base + o), kL2E, v[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) g = fmaxf(g, v[u]);
      }
    part[warp][lane] = g;
    __syncthreads();
#pragma unroll 8
    for (int w = 0; w < GS_WARPS; ++w) g = fmaxf(g, part[w][lane]);
    __syncthreads();
    return g;
  };
  if (MODE == MODE_FWD) {
    const float g = reduce(shift, 0.f);
    if (warp == 0 && b < B) gout[(int64_t)sr * ldb + b] = g;
  } else {
    const float gr = reduce(base, PCB_NEG_INF);
    const float g = reduce(shift, gr);
    if (warp == 0 && b < B) {
      gout[(int64_t)sr * ldb + b] = g;
      gbase[(int64_t)sr * ldb + b] = gr;
    }
  }
}

template <int MODE>
int launch_group_shift(const WsArgs& a, int kc, int64_t count, float* gout, float* gbase,
                       cudaStream_t s) {
  dim3 grid((unsigned)count, (unsigned)((a.B + 31) / 32));
  launch_k((k_group_shift<MODE>), dim3(grid), dim3(GS_WARPS * 32), 0, s, a.cap, kc, a.B, a.ldb, a.sb_base, a.row_off,
                                           a.members, a.src_ids, a.real_ids, a.shift,
                                           a.vbase_in, gout, gbase);
  return check_launch();
}

// In-kernel long-K shifts when every CTA runs exactly one item (the persistent
// grid is min(items, SMs)).  The environment is read per launch so tests can
// drive every shift path: PCB_NO_COOP_SHIFT=1 keeps the separate shift kernel.
bool coop_ok(const WsArgs& a) {
  return getenv("PCB_NO_COOP_SHIFT") == nullptr && a.n_items <= sm_count();
}

// Many items per CTA and a moderate K (RAT-SPN: 32 blocks, ~100 items per
// CTA): the shift warp computes each item's shifts while the previous item
// runs (four rounds of loads), so no precompute launch is needed either.
// PCB_FORCE_GROUP_SHIFT=1 disables it; PCB_SHIFT_WARP_MIN_ITEMS overrides the
// item threshold (default 4 x SMs).
bool shift_warp_ok(const WsArgs& a) {
  if (getenv("PCB_FORCE_GROUP_SHIFT")) return false;
  const char* m = getenv("PCB_SHIFT_WARP_MIN_ITEMS");
  const int64_t min_items = m ? atoll(m) : 4 * (int64_t)sm_count();
  return a.cap <= 64 && a.n_items >= min_items;
}

// K split so a layer with few (super-row, tile) items still covers the SMs:
// >= 2 K blocks per slice; only when the group owns all output rows it zeroes
// The slice count minimises a wave model: waves(items) x (K blocks per item +
// per-item pipeline fill / epilogue overhead, ~3 K blocks), with >= 2 blocks
// per slice.
void plan_split(WsArgs& a, int64_t count, bool split_ok) {
  const int64_t base = count * a.ntiles;
  const int64_t sms = sm_count();
  int best = 1;
  if (split_ok && ws_long_k(a.cap)) {
    int64_t best_cost = -1;
    for (int ks = 1; ks <= a.cap / 2; ++ks) {
      const int64_t per = (a.cap + ks - 1) / ks;
      const int64_t waves = (base * ks + sms - 1) / sms;
      const int64_t cost = waves * (per + 3);
      if (best_cost < 0 || cost < best_cost) best_cost = cost, best = ks;
    }
  }
  a.kper = (a.cap + best - 1) / best;
  a.kslices = (a.cap + a.kper - 1) / a.kper;
  a.n_items = (int)(base * a.kslices);
}

}  // namespace

int64_t ws_part_floats() { return (int64_t)sm_count() * WS_M * WS_NMAX; }

bool ws_supported(int kc, int nb) { return (kc == 16 || kc == 32) && (nb == 16 || nb == 32 || nb == 64); }

namespace {
inline bool tc_k(int64_t k) { return k == 16 || k == 32 || k == 64; }
}  // namespace
bool tc_supported(const Layer& L) { return tc_k(L.k_m) && tc_k(L.k_n); }
bool tc_bwd_supported(const Layer& L) { return tc_k(L.k_m) && tc_k(L.k_n); }

int launch_sum_fwd_ws(const pcb_plan* P, const Layer& L, const FwdGroup& g, const TcRows& tc,
                      cudaStream_t s, int B, int ldb, const float* scratch, const float* pbase,
                      float* values, float* vbase, float* gshift, int32_t* counters,
                      bool split_ok, float* part) {
  ProfScope prof_(KC_SUM_FWD_TC, s);
  if (!tc.count || !B) return PCB_OK;
  WsArgs a{};
  a.cap = (int)g.cap;
  a.nb = (int)L.k_m;
  a.B = B;
  a.ldb = ldb;
  a.ntiles = (B + WS_M - 1) / WS_M;
  a.n_items = (int)tc.count * a.ntiles;
  a.sb_base = 0;
  a.row_off = tc.row_off;
  a.members = tc.members;
  a.out_ids = g.sum_ids;
  a.src_ids = g.prod_ids;
  a.real_ids = g.param_ids;
  a.slab = g.param_slab;
  a.flags = tc.flags;
  a.plane = P->mma_plane;
  a.mma = P->mma;
  a.src0 = scratch;
  a.shift = pbase;
  a.aux = nullptr;
  a.out = values;
  a.vbase = vbase;
  a.out_base = L.sb_base;
  a.counters = counters;
  plan_split(a, tc.count, split_ok);
  if (ws_long_k(a.cap) && !shift_warp_ok(a)) {
    if (coop_ok(a)) {
      a.coop = 1;
      // part != nullptr: the caller guarantees no other spread launch runs
      // concurrently (pcb_capi.cu carve), so the slices may wait for each other
      a.split_finish = part && getenv("PCB_NO_SPLIT_FINISH") == nullptr;
      // partial sums through a slab instead of L2 reductions into the output
      if (a.split_finish && a.kslices > 1 && getenv("PCB_NO_SPLIT_SLAB") == nullptr)
        a.part = part;
    } else {
      if (launch_group_shift<MODE_FWD>(a, (int)L.k_n, g.uniform ? 1 : tc.count, gshift, nullptr, s))
        return PCB_CUDA;
      a.gshift = gshift;
      a.gshift_stride = g.uniform ? 0 : ldb;
    }
  }
  // split K reduces partial sums in place: zero the layer's sum rows first
  if (a.kslices > 1 &&
      cudaMemsetAsync(values + L.sb_base * (int64_t)ldb, 0,
                      sizeof(float) * L.n_sb * L.k_m * (int64_t)ldb, s) != cudaSuccess)
    return PCB_CUDA;
  switch (L.k_n) {
    case 16: return launch_ws<MODE_FWD, 16>(a, L.window, L.n_pb, s);
    case 32: return launch_ws<MODE_FWD, 32>(a, L.window, L.n_pb, s);
    default: return PCB_USAGE;
  }
}

int launch_child_flow_ws(const pcb_plan* P, const Layer& L, const BwdGroup& g, const TcRows& tc,
                         cudaStream_t s, int B, int ldb, const float* ratio, const float* scratch,
                         const float* rmax, const float* vbase, const float* pbase,
                         float* flow_scratch, float* gshift, int32_t* counters, bool split_ok,
                         float* part) {
  ProfScope prof_(KC_CHILD_FLOW, s);
  if (!tc.count || !B) return PCB_OK;
  WsArgs a{};
  a.cap = (int)g.cap;
  a.nb = (int)L.k_n;
  a.B = B;
  a.ldb = ldb;
  a.ntiles = (B + WS_M - 1) / WS_M;
  a.n_items = (int)tc.count * a.ntiles;
  a.sb_base = L.sb_base;
  a.row_off = tc.row_off;
  a.members = tc.members;
  a.out_ids = g.ch_ids;
  a.src_ids = g.par_ids;
  a.real_ids = g.par_param_ids;
  a.slab = g.par_slab;
  a.flags = tc.flags;
  a.plane = P->mma_plane;
  a.mma = P->mma;
  a.src0 = ratio;
  a.shift = rmax;
  a.aux = scratch;
  a.out = flow_scratch;
  a.vbase_in = vbase;
  a.pbase_in = pbase;
  a.counters = counters;
  plan_split(a, tc.count, split_ok);
  if (ws_long_k(a.cap) && !shift_warp_ok(a)) {
    if (coop_ok(a)) {
      a.coop = 1;
      // part != nullptr: the caller guarantees no other spread launch runs
      // concurrently (pcb_capi.cu carve), so the slices may wait for each other
      a.split_finish = part && getenv("PCB_NO_SPLIT_FINISH") == nullptr;
      // partial sums through a slab instead of L2 reductions into the output
      if (a.split_finish && a.kslices > 1 && getenv("PCB_NO_SPLIT_SLAB") == nullptr)
        a.part = part;
    } else {
      const int64_t n = g.uniform ? 1 : tc.count;
      if (launch_group_shift<MODE_CF>(a, (int)L.k_m, n, gshift, gshift + n * ldb, s))
        return PCB_CUDA;
      a.gshift = gshift;
      a.gbase = gshift + n * ldb;
      a.gshift_stride = g.uniform ? 0 : ldb;
    }
  }
  if (a.kslices > 1 &&
      cudaMemsetAsync(flow_scratch, 0, sizeof(float) * L.window * (int64_t)ldb, s) != cudaSuccess)
    return PCB_CUDA;
  switch (L.k_m) {
    case 16: return launch_ws<MODE_CF, 16>(a, L.n_sb * L.k_m, L.n_sb, s);
    case 32: return launch_ws<MODE_CF, 32>(a, L.n_sb * L.k_m, L.n_sb, s);
    default: return PCB_USAGE;
  }
}

}  // namespace pcb
