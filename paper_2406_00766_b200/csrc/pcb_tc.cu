// Tensor-core (tcgen05 + TMEM) sum-layer kernels for sm_100a.
//
// Sum-layer forward (Alg. 1, engine.py:74-102) as a block contraction:
//   D[b, n] = sum_k exp(child[k, b] - gmax[b]) * theta[n, k]
//   values[n, b] = log(D[b, n]) + gmax[b]
// for one "super-row" (sum blocks sharing an identical child-block row,
// stacked on N, <= 256 sums) and a 128-sample tile on M.  gmax is the
// per-sample maximum over all children of the super-row, so one fp32 TMEM
// accumulation replaces the per-block streaming rescale of the reference;
// the two agree except below fp32 underflow (e^-87 relative to the max term).
//
// Precision: operands are split into bf16 hi + lo and contracted as
// hi*hi + hi*lo + lo*hi (three kind::f16 MMAs, fp32 accumulation), i.e.
// ~2^-16 relative operand precision — the 1e-4 parity bar of the north star
// holds with an order of magnitude to spare, at 3x the MMA work of plain bf16
// (the HCLT-256 sum layers are HBM-bound, so the extra MMAs are free there).
#include <math.h>

#include "pcb_internal.cuh"
#include "pcb_tc.cuh"

namespace pcb {

using namespace tc;

// --------------------------------------------------------------- self test
// D[128 x n] = A[128 x k] . B[n x k]^T, bf16 inputs (row-major, K contiguous).
__global__ void __launch_bounds__(128, 1)
    k_tc_selftest(int n, int k, const uint16_t* __restrict__ A, const uint16_t* __restrict__ Bm,
                  float* __restrict__ D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + 128 * k * 2;
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int q = tid; q < 128 * (k / 8); q += 128) {
    int row = q / (k / 8), kq = q % (k / 8);
    uint4 v = *reinterpret_cast<const uint4*>(A + (size_t)row * k + kq * 8);
    *reinterpret_cast<uint4*>(sA + kmajor_off(row, kq * 8, k)) = v;
  }
  for (int q = tid; q < n * (k / 8); q += 128) {
    int row = q / (k / 8), kq = q % (k / 8);
    uint4 v = *reinterpret_cast<const uint4*>(Bm + (size_t)row * k + kq * 8);
    *reinterpret_cast<uint4*>(sB + kmajor_off(row, kq * 8, k)) = v;
  }
  const uint32_t ncols = tmem_cols_for(n);
  if (tid == 0) {
    mbar_init(smem_u32(&mbar), 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(smem_u32(&tmem_base), ncols);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = idesc_bf16(128, n);
    const uint32_t sbo = (k / 8) * 128;
    for (int ks = 0; ks < k / 16; ++ks) {
      uint64_t ad = make_desc(smem_u32(sA) + ks * 256, 128, sbo);
      uint64_t bd = make_desc(smem_u32(sB) + ks * 256, 128, sbo);
      mma_bf16(tmem, ad, bd, idesc, ks > 0);
    }
    mma_commit(smem_u32(&mbar));
  }
  __syncwarp();
  mbar_wait(smem_u32(&mbar), 0);
  tc_fence_after();
  for (int c0 = 0; c0 < n; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
    for (int i = 0; i < 16; ++i) D[(size_t)tid * n + c0 + i] = v[i];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free(tmem, ncols);
}

// --------------------------------------------------------------- sum forward
constexpr int TC_M = 128;
constexpr int TC_NMAX = 256;

template <int KN>
struct FwdSmem {
  static constexpr int kA = TC_M * KN * 2;      // one bf16 A plane
  static constexpr int kB = TC_NMAX * KN * 2;   // one bf16 B plane
  static constexpr int kStage = 2 * kA + 2 * kB;
  static constexpr int kBytes = 2 * kStage;
};

template <int KN>
__global__ void __launch_bounds__(128, 1)
    k_sum_fwd_tc(int cap, int k_m, int B, int ldb, const int32_t* __restrict__ row_off,
                 const int32_t* __restrict__ members, const int32_t* __restrict__ sum_ids,
                 const int32_t* __restrict__ prod_ids, const int32_t* __restrict__ param_ids,
                 const float* __restrict__ theta, const float* __restrict__ scratch,
                 const float* __restrict__ bmax, float* __restrict__ values) {
  using SM = FwdSmem<KN>;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int sr = blockIdx.x;
  const int b = blockIdx.y * TC_M + tid;
  const bool live = b < B;
  const int m0 = row_off[sr];
  const int S = row_off[sr + 1] - m0;
  const int N = S * k_m;
  const int Npad = (N + 15) & ~15;
  const int r0 = members[m0];
  const int32_t* prow = prod_ids + (int64_t)r0 * cap;
  const int32_t* trow = param_ids + (int64_t)r0 * cap;

  // per-sample maximum over every child of the super-row, from the product
  // kernel's per-block maxima (scratch block index = scratch row / k_n)
  float gm = PCB_NEG_INF;
  if (live)
    for (int c = 0; c < cap; ++c) {
      if (trow[c] == 0) continue;
      gm = fmaxf(gm, bmax[(int64_t)(prow[c] / KN) * ldb + b]);
    }
  const bool dead = (gm == PCB_NEG_INF);

  const uint32_t ncols = tmem_cols_for(Npad);
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
  const uint32_t idesc = idesc_bf16(TC_M, Npad);
  constexpr uint32_t SBO = (KN / 8) * 128;

  int it = 0;
  for (int c = 0; c < cap; ++c) {
    if (trow[c] == 0) continue;  // padded child column (uniform across the CTA)
    const int stage = it & 1;
    if (it >= 2) mbar_wait(smem_u32(&mbar[stage]), ((it - 2) >> 1) & 1);
    uint8_t* sAh = smem + stage * SM::kStage;
    uint8_t* sAl = sAh + SM::kA;
    uint8_t* sBh = sAl + SM::kA;
    uint8_t* sBl = sBh + SM::kB;
    // A: exp(child - gmax) for this thread's sample, split hi/lo
    const float* src = scratch + (int64_t)prow[c] * ldb + b;
#pragma unroll
    for (int jq = 0; jq < KN / 8; ++jq) {
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float x0 = PCB_NEG_INF, x1 = PCB_NEG_INF;
        if (live) {
          x0 = src[(int64_t)(jq * 8 + 2 * e) * ldb];
          x1 = src[(int64_t)(jq * 8 + 2 * e + 1) * ldb];
        }
        const float e0 = dead ? 0.f : __expf(x0 - gm);
        const float e1 = dead ? 0.f : __expf(x1 - gm);
        __nv_bfloat16 h0, l0, h1, l1;
        split_bf16(e0, h0, l0);
        split_bf16(e1, h1, l1);
        hi[e] = pack2(h0, h1);
        lo[e] = pack2(l0, l1);
      }
      const uint32_t off = kmajor_off(tid, jq * 8, KN);
      *reinterpret_cast<uint4*>(sAh + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4*>(sAl + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
    // B: theta tiles of the stacked sum blocks, row n = s * k_m + mm
    for (int q = tid; q < Npad * (KN / 8); q += TC_M) {
      const int n = q / (KN / 8), jq = q - n * (KN / 8);
      uint32_t hi[4] = {0, 0, 0, 0}, lo[4] = {0, 0, 0, 0};
      if (n < N) {
        const int s = n / k_m, mm = n - s * k_m;
        const int tile = param_ids[(int64_t)members[m0 + s] * cap + c];
        const float* t = theta + tile + mm * KN + jq * 8;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __nv_bfloat16 h0, l0, h1, l1;
          split_bf16(__ldg(t + 2 * e), h0, l0);
          split_bf16(__ldg(t + 2 * e + 1), h1, l1);
          hi[e] = pack2(h0, h1);
          lo[e] = pack2(l0, l1);
        }
      }
      const uint32_t off = kmajor_off(n, jq * 8, KN);
      *reinterpret_cast<uint4*>(sBh + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4*>(sBl + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t aH = smem_u32(sAh), aL = smem_u32(sAl);
      const uint32_t bH = smem_u32(sBh), bL = smem_u32(sBl);
#pragma unroll
      for (int ks = 0; ks < KN / 16; ++ks) {
        const uint32_t o = ks * 256;
        mma_bf16(tmem, make_desc(aH + o, 128, SBO), make_desc(bH + o, 128, SBO), idesc,
                 (it > 0 || ks > 0) ? 1u : 0u);
        mma_bf16(tmem, make_desc(aH + o, 128, SBO), make_desc(bL + o, 128, SBO), idesc, 1u);
        mma_bf16(tmem, make_desc(aL + o, 128, SBO), make_desc(bH + o, 128, SBO), idesc, 1u);
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
  for (int c0 = 0; c0 < Npad; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
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

// --------------------------------------------------------------- param flows
// Alg. 3 (engine.py:105-126) as a contraction over the batch:
//   cum[m, n] = sum_b exp(lnf[m, b] - c_b) * exp(child[n, b] + c_b)
//   f_params[flow + m*k_n + j] += theta * cum
// One CTA = one 128-sum M tile of a super-row x up to 256 product columns
// (N); K = samples streamed in chunks of 32 through two smem stages.  c_b is
// the per-sample max of lnf over the M tile (any shift is exact in real
// arithmetic; the max keeps both operands in range).
constexpr int PF_KC = 32;  // samples per stage

struct PfSmem {
  static constexpr int kA = TC_M * PF_KC * 2;
  static constexpr int kB = TC_NMAX * PF_KC * 2;
  static constexpr int kStage = 2 * kA + 2 * kB;
  static constexpr int kBytes = 2 * kStage;
};

__device__ __forceinline__ float lnf_of(float f, float l) {
  return (l == PCB_NEG_INF) ? PCB_NEG_INF : (__logf(f) - l);
}

template <int KN>
__global__ void __launch_bounds__(128, 1)
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
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int sr = blockIdx.x;
  const int mt = blockIdx.y;        // M tile of the super-row
  const int cg = blockIdx.z;        // column group
  const int m0 = row_off[sr];
  const int S = row_off[sr + 1] - m0;
  const int Nsum = S * k_m;
  if (mt * TC_M >= Nsum) return;
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
  const int Npad = ncol * KN;  // multiple of 16
  // my A row: sum index within the super-row
  const int ms = mt * TC_M + tid;
  const bool row_live = ms < Nsum;
  int sum_slot = 0;
  if (row_live) sum_slot = sum_ids[members[m0 + ms / k_m]] + (ms % k_m);

  const uint32_t ncols_t = tmem_cols_for(Npad);
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

  int it = 0;
  for (int b0 = 0; b0 < B; b0 += PF_KC, ++it) {
    const int stage = it & 1;
    // A operand inputs: lnf for my sum row over the 32 samples of the chunk
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
#pragma unroll
    for (int q = 0; q < PF_KC; ++q)
      if (b0 + q >= B) ln[q] = PCB_NEG_INF;
    if (it >= 2) mbar_wait(smem_u32(&mbar[stage]), ((it - 2) >> 1) & 1);
    __syncthreads();  // previous chunk's readers of cb are done
    // per-sample shift: max of the ratio-max rows of the tile's sum blocks
    if (tid < PF_KC) {
      float v = PCB_NEG_INF;
      if (b0 + tid < B) {
        const int s_lo = (mt * TC_M) / k_m;
        const int s_hi = (min(mt * TC_M + TC_M, Nsum) - 1) / k_m;
        for (int s = s_lo; s <= s_hi; ++s) {
          const int64_t blk = (sum_ids[members[m0 + s]] - sb_base) / k_m;
          v = fmaxf(v, rmax[blk * ldb + b0 + tid]);
        }
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
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int q0 = kq * 8 + 2 * e;
        const float c0 = cb[q0], c1 = cb[q0 + 1];
        const float s0 = (c0 == PCB_NEG_INF || ln[q0] == PCB_NEG_INF) ? 0.f : __expf(ln[q0] - c0);
        const float s1 = (c1 == PCB_NEG_INF || ln[q0 + 1] == PCB_NEG_INF) ? 0.f : __expf(ln[q0 + 1] - c1);
        __nv_bfloat16 h0, l0, h1, l1;
        split_bf16(s0, h0, l0);
        split_bf16(s1, h1, l1);
        hi[e] = pack2(h0, h1);
        lo[e] = pack2(l0, l1);
      }
      const uint32_t off = kmajor_off(tid, kq * 8, PF_KC);
      *reinterpret_cast<uint4*>(sAh + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4*>(sAl + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
    // B operand: exp(child + c_b) for every product of the column group
    const int32_t* prow = prod_ids + (int64_t)r0 * cap;
    for (int q = tid; q < Npad * (PF_KC / 8); q += TC_M) {
      const int n = q / (PF_KC / 8), kq = q - n * (PF_KC / 8);
      const int c = cols[n / KN], j = n % KN;
      const float* src = scratch + (int64_t)(prow[c] + j) * ldb + b0 + kq * 8;
      const float4 x0 = *reinterpret_cast<const float4*>(src);
      const float4 x1 = *reinterpret_cast<const float4*>(src + 4);
      const float xs[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int q0 = kq * 8 + 2 * e;
        const float c0 = cb[q0], c1 = cb[q0 + 1];
        const float e0 = (c0 == PCB_NEG_INF) ? 0.f : fminf(__expf(xs[2 * e] + c0), 1e37f);
        const float e1 = (c1 == PCB_NEG_INF) ? 0.f : fminf(__expf(xs[2 * e + 1] + c1), 1e37f);
        __nv_bfloat16 h0, l0, h1, l1;
        split_bf16(e0, h0, l0);
        split_bf16(e1, h1, l1);
        hi[e] = pack2(h0, h1);
        lo[e] = pack2(l0, l1);
      }
      const uint32_t off = kmajor_off(n, kq * 8, PF_KC);
      *reinterpret_cast<uint4*>(sBh + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4*>(sBl + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t aH = smem_u32(sAh), aL = smem_u32(sAl);
      const uint32_t bH = smem_u32(sBh), bL = smem_u32(sBl);
#pragma unroll
      for (int ks = 0; ks < PF_KC / 16; ++ks) {
        const uint32_t o = ks * 256;
        mma_bf16(tmem, make_desc(aH + o, 128, SBO), make_desc(bH + o, 128, SBO), idesc,
                 (it > 0 || ks > 0) ? 1u : 0u);
        mma_bf16(tmem, make_desc(aH + o, 128, SBO), make_desc(bL + o, 128, SBO), idesc, 1u);
        mma_bf16(tmem, make_desc(aL + o, 128, SBO), make_desc(bH + o, 128, SBO), idesc, 1u);
      }
      mma_commit(smem_u32(&mbar[stage]));
    }
    __syncwarp();
  }
  mbar_wait(smem_u32(&mbar[(it - 1) & 1]), ((it - 1) >> 1) & 1);
  tc_fence_after();
  // epilogue: lane = sum row; f_params[flow + mm*k_n + j] += theta * cum
  int s = 0, mm = 0;
  if (row_live) {
    s = ms / k_m;
    mm = ms - s * k_m;
  }
  const int64_t rowbase = (int64_t)members[m0 + (row_live ? s : 0)] * cap;
  for (int c0 = 0; c0 < Npad; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
    if (!row_live) continue;
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

// --------------------------------------------------------------- child flows
// Alg. 4 (engine.py:129-165) as a transposed contraction:
//   D[b, n] = sum_{k in parent sums} exp(lnf[k, b] - g_b) * theta[k, n]
//   flow_scratch[n, b] = D * exp(g_b + child[n, b])
// One CTA = one bwd super-row (product blocks with identical parent rows,
// stacked on N <= 256) x 128 samples; K = parent sums, one parent block per
// stage.  g_b = per-sample max of lnf over every parent sum.
template <int KM>
struct CfSmem {
  static constexpr int kA = TC_M * KM * 2;
  static constexpr int kB = TC_NMAX * KM * 2;
  static constexpr int kStage = 2 * kA + 2 * kB;
  static constexpr int kBytes = 2 * kStage;
};

template <int KM>
__global__ void __launch_bounds__(128, 1)
    k_child_flow_tc(int cap, int k_n, int B, int ldb, const int32_t* __restrict__ row_off,
                    const int32_t* __restrict__ members, const int32_t* __restrict__ ch_ids,
                    const int32_t* __restrict__ par_ids, const int32_t* __restrict__ ppids,
                    const float* __restrict__ theta, const float* __restrict__ values,
                    const float* __restrict__ flows, const float* __restrict__ scratch,
                    const float* __restrict__ rmax, int64_t sb_base,
                    float* __restrict__ flow_scratch) {
  using SM = CfSmem<KM>;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int sr = blockIdx.x;
  const int b = blockIdx.y * TC_M + tid;
  const bool live = b < B;
  const int m0 = row_off[sr];
  const int S = row_off[sr + 1] - m0;
  const int N = S * k_n;
  const int Npad = (N + 15) & ~15;
  const int r0 = members[m0];
  const int32_t* parow = par_ids + (int64_t)r0 * cap;
  const int32_t* pprow = ppids + (int64_t)r0 * cap;

  // per-sample max of lnf over every parent sum, from the ratio-max pass
  float gm = PCB_NEG_INF;
  if (live)
    for (int p = 0; p < cap; ++p) {
      if (pprow[p] == 0) continue;
      gm = fmaxf(gm, rmax[((int64_t)parow[p] - sb_base) / KM * ldb + b]);
    }
  const bool dead = (gm == PCB_NEG_INF);

  const uint32_t ncols = tmem_cols_for(Npad);
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
  const uint32_t idesc = idesc_bf16(TC_M, Npad);
  constexpr uint32_t SBO = (KM / 8) * 128;

  int it = 0;
  for (int p = 0; p < cap; ++p) {
    if (pprow[p] == 0) continue;
    const int stage = it & 1;
    if (it >= 2) mbar_wait(smem_u32(&mbar[stage]), ((it - 2) >> 1) & 1);
    uint8_t* sAh = smem + stage * SM::kStage;
    uint8_t* sAl = sAh + SM::kA;
    uint8_t* sBh = sAl + SM::kA;
    uint8_t* sBl = sBh + SM::kB;
    const int64_t base = (int64_t)parow[p] * ldb + b;
#pragma unroll
    for (int kq = 0; kq < KM / 8; ++kq) {
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float s0 = 0.f, s1 = 0.f;
        if (live && !dead) {
          const int64_t o0 = base + (int64_t)(kq * 8 + 2 * e) * ldb;
          const float a0 = lnf_of(flows[o0], values[o0]);
          const float a1 = lnf_of(flows[o0 + ldb], values[o0 + ldb]);
          s0 = (a0 == PCB_NEG_INF) ? 0.f : __expf(a0 - gm);
          s1 = (a1 == PCB_NEG_INF) ? 0.f : __expf(a1 - gm);
        }
        __nv_bfloat16 h0, l0, h1, l1;
        split_bf16(s0, h0, l0);
        split_bf16(s1, h1, l1);
        hi[e] = pack2(h0, h1);
        lo[e] = pack2(l0, l1);
      }
      const uint32_t off = kmajor_off(tid, kq * 8, KM);
      *reinterpret_cast<uint4*>(sAh + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4*>(sAl + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
    // B: theta transposed, row n = s * k_n + j, column k = parent sum mm
    for (int q = tid; q < Npad * (KM / 8); q += TC_M) {
      const int kq = q / Npad, n = q - kq * Npad;  // consecutive threads -> consecutive j
      uint32_t hi[4] = {0, 0, 0, 0}, lo[4] = {0, 0, 0, 0};
      if (n < N) {
        const int s = n / k_n, j = n - s * k_n;
        const int tile = ppids[(int64_t)members[m0 + s] * cap + p];
        const float* t = theta + tile + (kq * 8) * k_n + j;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __nv_bfloat16 h0, l0, h1, l1;
          split_bf16(__ldg(t + (2 * e) * k_n), h0, l0);
          split_bf16(__ldg(t + (2 * e + 1) * k_n), h1, l1);
          hi[e] = pack2(h0, h1);
          lo[e] = pack2(l0, l1);
        }
      }
      const uint32_t off = kmajor_off(n, kq * 8, KM);
      *reinterpret_cast<uint4*>(sBh + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4*>(sBl + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t aH = smem_u32(sAh), aL = smem_u32(sAl);
      const uint32_t bH = smem_u32(sBh), bL = smem_u32(sBl);
#pragma unroll
      for (int ks = 0; ks < KM / 16; ++ks) {
        const uint32_t o = ks * 256;
        mma_bf16(tmem, make_desc(aH + o, 128, SBO), make_desc(bH + o, 128, SBO), idesc,
                 (it > 0 || ks > 0) ? 1u : 0u);
        mma_bf16(tmem, make_desc(aH + o, 128, SBO), make_desc(bL + o, 128, SBO), idesc, 1u);
        mma_bf16(tmem, make_desc(aL + o, 128, SBO), make_desc(bH + o, 128, SBO), idesc, 1u);
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
  for (int c0 = 0; c0 < Npad; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
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

bool tc_supported(const Layer& L) {
  return (L.k_n == 16 || L.k_n == 32 || L.k_n == 64) && L.k_m >= 1 && L.k_m <= TC_NMAX;
}

bool tc_bwd_supported(const Layer& L) {
  return (L.k_n == 16 || L.k_n == 32 || L.k_n == 64) &&
         (L.k_m == 16 || L.k_m == 32 || L.k_m == 64);
}

template <int KN>
static int launch_pf_kn(const Layer& L, const FwdGroup& g, const TcRows& tc, cudaStream_t s,
                        int B, int ldb, const float* theta, const float* values,
                        const float* flows, const float* scratch, const float* rmax,
                        float* f_params) {
  static bool attr_set = false;
  const int bytes = PfSmem::kBytes;
  if (!attr_set) {
    if (cudaFuncSetAttribute(k_param_flow_tc<KN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             bytes) != cudaSuccess)
      return PCB_CUDA;
    attr_set = true;
  }
  const int max_stack = (int)(TC_NMAX / L.k_m) > 0 ? (int)(TC_NMAX / L.k_m) : 1;
  const int mtiles = (max_stack * (int)L.k_m + TC_M - 1) / TC_M;
  const int cgroups = (int)((g.cap * KN + TC_NMAX - 1) / TC_NMAX);
  dim3 grid((unsigned)tc.count, (unsigned)mtiles, (unsigned)cgroups);
  k_param_flow_tc<KN><<<grid, TC_M, bytes, s>>>(
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
    case 16: return launch_pf_kn<16>(L, g, tc, s, B, ldb, theta, values, flows, scratch, rmax, f_params);
    case 32: return launch_pf_kn<32>(L, g, tc, s, B, ldb, theta, values, flows, scratch, rmax, f_params);
    case 64: return launch_pf_kn<64>(L, g, tc, s, B, ldb, theta, values, flows, scratch, rmax, f_params);
    default: return PCB_USAGE;
  }
}

template <int KM>
static int launch_cf_km(const Layer& L, const BwdGroup& g, const TcRows& tc, cudaStream_t s,
                        int B, int ldb, const float* theta, const float* values,
                        const float* flows, const float* scratch, const float* rmax,
                        float* flow_scratch) {
  static bool attr_set = false;
  const int bytes = CfSmem<KM>::kBytes;
  if (!attr_set) {
    if (cudaFuncSetAttribute(k_child_flow_tc<KM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             bytes) != cudaSuccess)
      return PCB_CUDA;
    attr_set = true;
  }
  dim3 grid((unsigned)tc.count, (unsigned)((B + TC_M - 1) / TC_M));
  k_child_flow_tc<KM><<<grid, TC_M, bytes, s>>>((int)g.cap, (int)L.k_n, B, ldb, tc.row_off,
                                                 tc.members, g.ch_ids, g.par_ids,
                                                 g.par_param_ids, theta, values, flows, scratch,
                                                 rmax, L.sb_base, flow_scratch);
  return check_launch();
}

int launch_child_flow_tc(const Layer& L, const BwdGroup& g, const TcRows& tc, cudaStream_t s,
                         int B, int ldb, const float* theta, const float* values,
                         const float* flows, const float* scratch, const float* rmax,
                         float* flow_scratch) {
  ProfScope prof_(KC_CHILD_FLOW, s);
  if (!tc.count || !B) return PCB_OK;
  switch (L.k_m) {
    case 16: return launch_cf_km<16>(L, g, tc, s, B, ldb, theta, values, flows, scratch, rmax, flow_scratch);
    case 32: return launch_cf_km<32>(L, g, tc, s, B, ldb, theta, values, flows, scratch, rmax, flow_scratch);
    case 64: return launch_cf_km<64>(L, g, tc, s, B, ldb, theta, values, flows, scratch, rmax, flow_scratch);
    default: return PCB_USAGE;
  }
}

template <int KN>
static int launch_fwd_kn(const Layer& L, const FwdGroup& g, const TcRows& tc, cudaStream_t s,
                         int B, int ldb, const float* theta, const float* scratch,
                         const float* bmax, float* values) {
  static bool attr_set = false;
  const int bytes = FwdSmem<KN>::kBytes;
  if (!attr_set) {
    if (cudaFuncSetAttribute(k_sum_fwd_tc<KN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             bytes) != cudaSuccess)
      return PCB_CUDA;
    attr_set = true;
  }
  dim3 grid((unsigned)tc.count, (unsigned)((B + TC_M - 1) / TC_M));
  k_sum_fwd_tc<KN><<<grid, TC_M, bytes, s>>>((int)g.cap, (int)L.k_m, B, ldb, tc.row_off,
                                              tc.members, g.sum_ids, g.prod_ids, g.param_ids,
                                              theta, scratch, bmax, values);
  return check_launch();
}

int launch_sum_fwd_tc(const Layer& L, const FwdGroup& g, const TcRows& tc, cudaStream_t s,
                      int B, int ldb, const float* theta, const float* scratch,
                      const float* bmax, float* values) {
  ProfScope prof_(KC_SUM_FWD_TC, s);
  if (!tc.count || !B) return PCB_OK;
  switch (L.k_n) {
    case 16: return launch_fwd_kn<16>(L, g, tc, s, B, ldb, theta, scratch, bmax, values);
    case 32: return launch_fwd_kn<32>(L, g, tc, s, B, ldb, theta, scratch, bmax, values);
    case 64: return launch_fwd_kn<64>(L, g, tc, s, B, ldb, theta, scratch, bmax, values);
    default: return PCB_USAGE;
  }
}

}  // namespace pcb

extern "C" int pcb_tc_selftest(void* stream, int n, int k, const uint16_t* d_a,
                               const uint16_t* d_b, float* d_d) {
  if (n < 16 || n > 256 || (n % 16) || k < 16 || k > 256 || (k % 16)) return PCB_USAGE;
  const int bytes = 128 * k * 2 + n * k * 2;
  if (cudaFuncSetAttribute(pcb::k_tc_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           bytes) != cudaSuccess)
    return PCB_CUDA;
  pcb::k_tc_selftest<<<1, 128, bytes, reinterpret_cast<cudaStream_t>(stream)>>>(n, k, d_a, d_b,
                                                                                 d_d);
  return pcb::check_launch();
}
