// Tensor-core support for sm_100a: UMMA descriptor self-tests and the
// theta -> bf16 hi/lo MMA-tile conversion used by the sum-layer kernels
// (pcb_tc_sum.cu).
#include <math.h>

#include "pcb_internal.cuh"
#include "pcb_tc.cuh"

namespace pcb {

using namespace tc;

// --------------------------------------------------------------- self tests
// D[128 x n] = A[128 x k] . B[n x k]^T, bf16 inputs (row-major, K contiguous),
// both operands K-major in the no-swizzle core-matrix layout.
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

// MN-major B variant: B is [k x n] row-major (N contiguous), stored in the
// "tile layout" of the pre-split theta tables (core matrices of 8 k-rows x
// 8 n-elements, k-major order of cores).  variant 0: LBO = K-adjacent core
// stride, SBO = MN-adjacent; variant 1: swapped.
__global__ void __launch_bounds__(128, 1)
    k_tc_selftest_mn(int n, int k, int variant, const uint16_t* __restrict__ A,
                     const uint16_t* __restrict__ Bkn, float* __restrict__ D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint16_t* sB = reinterpret_cast<uint16_t*>(smem + 128 * k * 2);
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int q = tid; q < 128 * (k / 8); q += 128) {
    int row = q / (k / 8), kq = q % (k / 8);
    uint4 v = *reinterpret_cast<const uint4*>(A + (size_t)row * k + kq * 8);
    *reinterpret_cast<uint4*>(sA + kmajor_off(row, kq * 8, k)) = v;
  }
  for (int q = tid; q < k * n; q += 128) {
    int kk = q / n, nn = q % n;
    sB[tile_off(kk, nn, n)] = Bkn[q];
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
    const uint32_t idesc = idesc_bf16_bmn(128, n);
    const uint32_t kstride = (n / 8) * 128;  // bytes between K-adjacent cores
    const uint32_t lbo = variant == 0 ? kstride : 128;
    const uint32_t sbo = variant == 0 ? 128 : kstride;
    for (int ks = 0; ks < k / 16; ++ks) {
      uint64_t ad = make_desc(smem_u32(sA) + ks * 256, 128, (k / 8) * 128);
      uint64_t bd = make_desc(smem_u32(sB) + ks * 2 * kstride, lbo, sbo);
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

// ------------------------------------------------- theta -> bf16 MMA tiles
// Every tensor-core tile (k_m x k_n, row-major in theta) is re-laid as two
// bf16 planes (hi, lo with theta ~= hi + lo) in core-matrix order
// (tile_off): the same bytes are a K-major B operand for the sum forward
// (N = sums, K = products) and an MN-major B operand for the child flows
// (N = products, K = sums).  Refreshed after every theta update.
__global__ void k_theta_to_mma(int64_t n_tiles, const int32_t* __restrict__ t_theta,
                               const int32_t* __restrict__ t_slab, const int32_t* __restrict__ t_km,
                               const int32_t* __restrict__ t_kn, const float* __restrict__ theta,
                               __nv_bfloat16* __restrict__ mma) {
  for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const int km = t_km[t], kn = t_kn[t];
    const int sz = km * kn;
    const float* src = theta + t_theta[t];
    __nv_bfloat16* hi = mma + (int64_t)t_slab[t];
    __nv_bfloat16* lo = hi + sz;
    for (int q = threadIdx.x; q < sz; q += blockDim.x) {
      const int m = q / kn, j = q - m * kn;
      const int o = tile_off(m, j, kn);
      __nv_bfloat16 h, l;
      split_bf16(src[q], h, l);
      hi[o] = h;
      lo[o] = l;
    }
  }
}

int launch_theta_to_mma(const pcb_plan* p, cudaStream_t s, const float* theta) {
  ProfScope prof_(KC_EM, s);
  if (!p->n_mma_tiles || !p->mma) return PCB_OK;
  k_theta_to_mma<<<grid_for(p->n_mma_tiles, 1, 148 * 8), 256, 0, s>>>(
      p->n_mma_tiles, p->mma_theta, p->mma_slab, p->mma_km, p->mma_kn, theta, p->mma);
  return check_launch();
}

}  // namespace pcb

extern "C" int pcb_tc_selftest_mn(void* stream, int n, int k, int variant, const uint16_t* d_a,
                                  const uint16_t* d_b, float* d_d) {
  if (n < 16 || n > 256 || (n % 16) || k < 16 || k > 256 || (k % 16)) return PCB_USAGE;
  const int bytes = 128 * k * 2 + n * k * 2;
  if (cudaFuncSetAttribute(pcb::k_tc_selftest_mn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           bytes) != cudaSuccess)
    return PCB_CUDA;
  pcb::k_tc_selftest_mn<<<1, 128, bytes, reinterpret_cast<cudaStream_t>(stream)>>>(
      n, k, variant, d_a, d_b, d_d);
  return pcb::check_launch();
}

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
