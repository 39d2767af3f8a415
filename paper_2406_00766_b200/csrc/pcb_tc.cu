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
                 float* __restrict__ values) {
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

  // per-sample maximum over every child of the super-row
  float gm = PCB_NEG_INF;
  if (live)
    for (int c = 0; c < cap; ++c) {
      if (trow[c] == 0) continue;
      const float* src = scratch + (int64_t)prow[c] * ldb + b;
#pragma unroll 8
      for (int j = 0; j < KN; ++j) gm = fmaxf(gm, src[(int64_t)j * ldb]);
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

bool tc_supported(const Layer& L) {
  return (L.k_n == 16 || L.k_n == 32 || L.k_n == 64) && L.k_m >= 1 && L.k_m <= TC_NMAX;
}

template <int KN>
static int launch_fwd_kn(const Layer& L, const FwdGroup& g, const TcRows& tc, cudaStream_t s,
                         int B, int ldb, const float* theta, const float* scratch,
                         float* values) {
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
                                              theta, scratch, values);
  return check_launch();
}

int launch_sum_fwd_tc(const Layer& L, const FwdGroup& g, const TcRows& tc, cudaStream_t s,
                      int B, int ldb, const float* theta, const float* scratch, float* values) {
  if (!tc.count || !B) return PCB_OK;
  switch (L.k_n) {
    case 16: return launch_fwd_kn<16>(L, g, tc, s, B, ldb, theta, scratch, values);
    case 32: return launch_fwd_kn<32>(L, g, tc, s, B, ldb, theta, scratch, values);
    case 64: return launch_fwd_kn<64>(L, g, tc, s, B, ldb, theta, scratch, values);
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
