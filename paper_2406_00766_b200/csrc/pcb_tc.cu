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
  pdl_enter();
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
  pdl_enter();
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
// Every tensor-core tile (k_m x k_n, row-major in theta) is re-laid as four
// bf16 planes in core-matrix order (tile_off), theta ~= hi + lo, in four
// regions of `plane` elements (runtime/plan.py mma_tiles):
//   slab_f             hi, sum-major      K-major B of the sum forward (N =
//   plane + slab_f     lo, sum-major      sums, K = products); also the MN-major
//                                         B of the per-launch child-flow kernel
//   2 plane + slab_c   hi, product-major  K-major B of the child flows (N =
//   3 plane + slab_c   lo, product-major  products, K = sums)
// Hi planes of consecutive tiles stack along N with a uniform core stride,
// and slab_f / slab_c follow the stacking orders, so a super-row's stacked
// tiles of one column are one contiguous run per plane.  One CTA per tile:
// the tile is staged in shared memory, then every thread packs one 8-wide
// core row per plane pair (16-byte stores).  Refreshed after every theta update.
constexpr int TM_MAX = 64;
constexpr int TM_THREADS = 256;
constexpr int TM_V4 = TM_MAX * TM_MAX / 4 / TM_THREADS;  // float4 loads per thread (max)
__global__ void __launch_bounds__(TM_THREADS)
    k_theta_to_mma(int64_t n_tiles, const int32_t* __restrict__ t_theta,
                   const int32_t* __restrict__ t_slab_f, const int32_t* __restrict__ t_slab_c,
                   const int32_t* __restrict__ t_km, const int32_t* __restrict__ t_kn,
                   const float* __restrict__ theta, __nv_bfloat16* __restrict__ mma,
                   int64_t plane) {
  pdl_enter();
  __shared__ float tile[TM_MAX * (TM_MAX + 1)];
  // the next tile's elements are loaded (float4, row-major) while this one is packed
  float4 nx[TM_V4];
  auto load = [&](int64_t t) {
    const int sz = __ldg(t_km + t) * __ldg(t_kn + t);
    const int64_t start = __ldg(t_theta + t);
    const float* src = theta + start;
    if ((start & 3) == 0) {  // tiles after odd-sized input pmfs may be unaligned
#pragma unroll
      for (int u = 0; u < TM_V4; ++u) {
        const int q = (threadIdx.x + u * TM_THREADS) * 4;
        if (q < sz) nx[u] = __ldg(reinterpret_cast<const float4*>(src + q));
      }
    } else {
#pragma unroll
      for (int u = 0; u < TM_V4; ++u) {
        const int q = (threadIdx.x + u * TM_THREADS) * 4;
        if (q < sz)
          nx[u] = make_float4(__ldg(src + q), __ldg(src + q + 1), __ldg(src + q + 2),
                              __ldg(src + q + 3));
      }
    }
  };
  int64_t t = blockIdx.x;
  if (t < n_tiles) load(t);
  for (; t < n_tiles; t += gridDim.x) {
    const int km = __ldg(t_km + t), kn = __ldg(t_kn + t);
    const int sz = km * kn, ld = kn + 1;
#pragma unroll
    for (int u = 0; u < TM_V4; ++u) {
      const int q = (threadIdx.x + u * TM_THREADS) * 4;
      if (q < sz) {
        const int m = q / kn, j = q - m * kn;
        float* d = tile + m * ld + j;
        d[0] = nx[u].x, d[1] = nx[u].y, d[2] = nx[u].z, d[3] = nx[u].w;
      }
    }
    __syncthreads();
    if (t + gridDim.x < n_tiles) load(t + gridDim.x);
    __nv_bfloat16* fh = mma + __ldg(t_slab_f + t);
    __nv_bfloat16* ch = mma + 2 * plane + __ldg(t_slab_c + t);
    const int n8 = sz / 8;
    for (int q = threadIdx.x; q < 2 * n8; q += TM_THREADS) {
      float v[8];
      uint32_t off;
      int pl;
      if (q < n8) {  // sum-major: core row (m, j..j+7)
        const int m = q / (kn / 8), j = (q - m * (kn / 8)) * 8;
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = tile[m * ld + j + e];
        off = (uint32_t)tile_off(m, j, kn) * 2u;
        pl = 0;
      } else {       // product-major: core row (j, m..m+7)
        const int r = q - n8;
        const int j = r / (km / 8), m = (r - j * (km / 8)) * 8;
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = tile[(m + e) * ld + j];
        off = (uint32_t)tile_off(j, m, km) * 2u;
        pl = 2;
      }
      uint4 hi, lo;
      split_pack8(v, hi, lo);
      uint8_t* dst = reinterpret_cast<uint8_t*>(pl == 0 ? fh : ch) + off;
      *reinterpret_cast<uint4*>(dst) = hi;
      *reinterpret_cast<uint4*>(dst + plane * 2) = lo;
    }
    __syncthreads();
  }
}

// ------------------------------------------------- EM over tile blocks
// One CTA per tile block (em.py:58-94 for k_m groups that exactly tile a set
// of k_m x k_n tensor-core tiles, group i = row i of every tile): pass 1 sums
// F + k per row over the block's tiles (threads = row x 4-column quads,
// float4 loads, quad-group shuffles); pass 2 renormalises, blends and stores
// theta tile by tile and, for the plan's own table, packs the updated tile
// into its four bf16 MMA planes (k_theta_to_mma layout) from shared memory.
// 4 consecutive floats: one vector load when 16-byte aligned (tiles after
// odd-sized input pmfs may not be)
__device__ __forceinline__ float4 ld4(const float* p) {
  if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) return *reinterpret_cast<const float4*>(p);
  return make_float4(p[0], p[1], p[2], p[3]);
}

constexpr int EM_THREADS = 256;
constexpr int EM_NP = 4;  // row passes per thread (k_m x k_n <= 64 x 64)
// register path: blocks of <= EM_RT tiles of exactly EM_THREADS float4s
// (32 x 32): every thread loads its quad of every tile's flows and theta at
// once (2 x EM_RT vector loads in flight), and all tiles are staged in shared
// memory for one plane-packing pass
constexpr int EM_RT = 8;
constexpr int EM_SMEM = (8 * 32 * 33 > TM_MAX * (TM_MAX + 1)) ? 8 * 32 * 33 : TM_MAX * (TM_MAX + 1);
// tile blocks of k_em_tiles32: 32 x 32 tiles, more than one register round
__host__ __device__ __forceinline__ bool split32_blk(int km, int kn, int nt) {
  return km == 32 && kn == 32 && nt > EM_RT;
}
__global__ void __launch_bounds__(EM_THREADS)
    k_em_tiles(int64_t blk0, int64_t n_blk, const int32_t* __restrict__ bkm,
               const int32_t* __restrict__ bkn,
               const int32_t* __restrict__ toff, const int32_t* __restrict__ tstart,
               const int32_t* __restrict__ tslab_f, const int32_t* __restrict__ tslab_c,
               const float* __restrict__ F, float* __restrict__ theta,
               __nv_bfloat16* __restrict__ mma, int64_t plane_n, float kappa, float step,
               int planes, int32_t* status, int skip32) {
  pdl_enter();
  __shared__ float tile[EM_SMEM];
  const int tid = threadIdx.x;
  int informative = 0, bad = 0;
  for (int64_t b = blk0 + blockIdx.x; b < n_blk; b += gridDim.x) {
    const int km = __ldg(bkm + b), kn = __ldg(bkn + b);
    const int t0 = __ldg(toff + b), t1 = __ldg(toff + b + 1);
    if (skip32 && split32_blk(km, kn, t1 - t0)) continue;  // k_em_tiles32
    if (km == 32 && kn == 32) {
      // 32 x 32 tiles, any number per block (HMM-4096: 128): the row totals
      // with EM_RT tiles' flows in flight per round, then blend / store /
      // pack EM_RT tiles per round (their flows and theta loaded together;
      // one barrier pair per round instead of per tile)
      const int r = tid >> 3, c4 = (tid & 7) * 4;  // row, column quad (k_n = 32)
      const int nt = t1 - t0;
      float4 fv[EM_RT], ov[EM_RT];
      float acc = 0.f;
      for (int c0 = 0; c0 < nt; c0 += EM_RT) {
#pragma unroll
        for (int u = 0; u < EM_RT; ++u) {
          if (c0 + u < nt) {
            const int64_t o = __ldg(tstart + t0 + c0 + u) + r * 32 + c4;
            fv[u] = ld4(F + o);
            if (nt <= EM_RT) ov[u] = ld4(theta + o);
          }
        }
#pragma unroll
        for (int u = 0; u < EM_RT; ++u)
          if (c0 + u < nt)
            acc += (fv[u].x + kappa) + (fv[u].y + kappa) + (fv[u].z + kappa) + (fv[u].w + kappa);
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      const float inv = acc > 0.f ? 1.f / acc : 0.f;
      if (acc > 0.f && (tid & 7) == 0) ++informative;
      for (int c0 = 0; c0 < nt; c0 += EM_RT) {
        const int nc = min(EM_RT, nt - c0);
        if (nt > EM_RT) {
#pragma unroll
          for (int u = 0; u < EM_RT; ++u) {
            if (u < nc) {
              const int64_t o = __ldg(tstart + t0 + c0 + u) + r * 32 + c4;
              fv[u] = ld4(F + o);
              ov[u] = ld4(theta + o);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < EM_RT; ++u) {
          if (u >= nc) continue;
          float4 o = ov[u];
          if (inv > 0.f) {
            const float4 f = fv[u];
            const float n[4] = {(f.x + kappa) * inv, (f.y + kappa) * inv, (f.z + kappa) * inv,
                                (f.w + kappa) * inv};
            float* op = &o.x;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              op[e] = (step >= 1.f) ? n[e] : ((1.f - step) * op[e] + step * n[e]);
              if (!isfinite(op[e])) ++bad;
            }
            float* tp = theta + __ldg(tstart + t0 + c0 + u) + r * 32 + c4;
            if ((reinterpret_cast<uintptr_t>(tp) & 15) == 0) {
              *reinterpret_cast<float4*>(tp) = o;
            } else {
              tp[0] = o.x, tp[1] = o.y, tp[2] = o.z, tp[3] = o.w;
            }
          }
          if (planes) {
            float* d = tile + u * (32 * 33) + r * 33 + c4;
            d[0] = o.x, d[1] = o.y, d[2] = o.z, d[3] = o.w;
          }
        }
        if (!planes) continue;
        __syncthreads();
        const int n8 = 32 * 32 / 8;
        for (int q = tid; q < nc * 2 * n8; q += EM_THREADS) {
          const int u = q / (2 * n8), qq = q - u * 2 * n8;
          const float* tl = tile + u * (32 * 33);
          float v[8];
          uint32_t off;
          int pl;
          if (qq < n8) {  // sum-major core row (m, j..j+7)
            const int m = qq >> 2, j = (qq & 3) * 8;
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = tl[m * 33 + j + e];
            off = (uint32_t)tile_off(m, j, 32) * 2u;
            pl = 0;
          } else {  // product-major core row (j, m..m+7)
            const int rr = qq - n8;
            const int j = rr >> 2, m = (rr & 3) * 8;
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = tl[(m + e) * 33 + j];
            off = (uint32_t)tile_off(j, m, 32) * 2u;
            pl = 2;
          }
          uint4 hi, lo;
          split_pack8(v, hi, lo);
          uint8_t* dst = reinterpret_cast<uint8_t*>(
                             pl == 0 ? mma + __ldg(tslab_f + t0 + c0 + u)
                                     : mma + 2 * plane_n + __ldg(tslab_c + t0 + c0 + u)) +
                         off;
          *reinterpret_cast<uint4*>(dst) = hi;
          *reinterpret_cast<uint4*>(dst + plane_n * 2) = lo;
        }
        __syncthreads();
      }
      continue;
    }

    const int tpr = kn / 4, rp = EM_THREADS / tpr;  // threads per row, rows per pass
    const int c4 = (tid % tpr) * 4, r_in = tid / tpr;
    float acc[EM_NP];
#pragma unroll
    for (int p = 0; p < EM_NP; ++p) acc[p] = 0.f;
    const bool one_pass = rp >= km;  // every thread owns one row quad of each tile
    if (one_pass) {
      // 4 tiles' flows in flight per round
      for (int t = t0; t < t1; t += 4) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          v[u] = (t + u < t1 && r_in < km) ? ld4(F + __ldg(tstart + t + u) + r_in * kn + c4)
                                           : make_float4(-kappa, -kappa, -kappa, -kappa);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          acc[0] += (v[u].x + kappa) + (v[u].y + kappa) + (v[u].z + kappa) + (v[u].w + kappa);
      }
    } else {
      for (int t = t0; t < t1; ++t) {
        const float* f = F + __ldg(tstart + t);
#pragma unroll
        for (int p = 0; p < EM_NP; ++p) {
          const int row = p * rp + r_in;
          if (row < km) {
            const float4 v = ld4(f + row * kn + c4);
            acc[p] += (v.x + kappa) + (v.y + kappa) + (v.z + kappa) + (v.w + kappa);
          }
        }
      }
    }
    // row totals: reduce over the tpr (power of two) threads of each row
#pragma unroll
    for (int p = 0; p < EM_NP; ++p)
      for (int o = tpr / 2; o > 0; o >>= 1) acc[p] += __shfl_xor_sync(0xffffffffu, acc[p], o);
    float inv[EM_NP];
#pragma unroll
    for (int p = 0; p < EM_NP; ++p) {
      const int row = p * rp + r_in;
      const bool live = row < km && acc[p] > 0.f;
      inv[p] = live ? 1.f / acc[p] : 0.f;
      if (live && tid % tpr == 0) ++informative;
    }
    const int ld = kn + 1;
    // one-pass blocks: the next tile's flows and theta are loaded before this
    // tile's plane packing (two barriers) runs
    float4 fn = make_float4(0.f, 0.f, 0.f, 0.f), on = fn;
    if (one_pass && r_in < km) {
      const int64_t ts = __ldg(tstart + t0);
      fn = ld4(F + ts + r_in * kn + c4);
      on = ld4(theta + ts + r_in * kn + c4);
    }
    for (int t = t0; t < t1; ++t) {
      const int64_t ts = __ldg(tstart + t);
      const float* f = F + ts;
      float* th = theta + ts;
      const float4 fc = fn, oc = on;
      if (one_pass && t + 1 < t1 && r_in < km) {
        const int64_t tn = __ldg(tstart + t + 1);
        fn = ld4(F + tn + r_in * kn + c4);
        on = ld4(theta + tn + r_in * kn + c4);
      }
#pragma unroll
      for (int p = 0; p < EM_NP; ++p) {
        const int row = p * rp + r_in;
        if (row >= km || (one_pass && p > 0)) continue;
        const float4 fv = one_pass ? fc : ld4(f + row * kn + c4);
        float4 o = one_pass ? oc : ld4(th + row * kn + c4);
        if (inv[p] > 0.f) {
          const float w = inv[p];
          const float n[4] = {(fv.x + kappa) * w, (fv.y + kappa) * w, (fv.z + kappa) * w,
                              (fv.w + kappa) * w};
          float* op = &o.x;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            op[e] = (step >= 1.f) ? n[e] : ((1.f - step) * op[e] + step * n[e]);
            if (!isfinite(op[e])) ++bad;
          }
          float* tp = th + row * kn + c4;
          if ((reinterpret_cast<uintptr_t>(tp) & 15) == 0) {
            *reinterpret_cast<float4*>(tp) = o;
          } else {
            tp[0] = o.x, tp[1] = o.y, tp[2] = o.z, tp[3] = o.w;
          }
        }
        if (planes) {
          float* d = tile + row * ld + c4;
          d[0] = o.x, d[1] = o.y, d[2] = o.z, d[3] = o.w;
        }
      }
      if (!planes) continue;
      __syncthreads();
      __nv_bfloat16* fh = mma + __ldg(tslab_f + t);
      __nv_bfloat16* ch = mma + 2 * plane_n + __ldg(tslab_c + t);
      const int sz = km * kn, n8 = sz / 8;
      for (int q = tid; q < 2 * n8; q += EM_THREADS) {
        float v[8];
        uint32_t off;
        int pl;
        if (q < n8) {  // sum-major core row (m, j..j+7)
          const int m = q / (kn / 8), j = (q - m * (kn / 8)) * 8;
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = tile[m * ld + j + e];
          off = (uint32_t)tile_off(m, j, kn) * 2u;
          pl = 0;
        } else {       // product-major core row (j, m..m+7)
          const int r = q - n8;
          const int j = r / (km / 8), m = (r - j * (km / 8)) * 8;
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = tile[(m + e) * ld + j];
          off = (uint32_t)tile_off(j, m, km) * 2u;
          pl = 2;
        }
        uint4 hi, lo;
        split_pack8(v, hi, lo);
        uint8_t* dst = reinterpret_cast<uint8_t*>(pl == 0 ? fh : ch) + off;
        *reinterpret_cast<uint4*>(dst) = hi;
        *reinterpret_cast<uint4*>(dst + plane_n * 2) = lo;
      }
      __syncthreads();
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    informative += __shfl_xor_sync(0xffffffffu, informative, o);
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((tid & 31) == 0) {
    if (informative) atomicAdd(status, informative);
    if (bad) atomicAdd(status + 1, bad);
  }
}

// Blocks of more than EM_RT 32 x 32 tiles (HMM-4096: 128 per block, only
// 128 blocks): four 256-thread tile groups per CTA split the block's tiles
// (rounds of E32_RT tiles, interleaved), combine their row partials in
// shared memory in a fixed order, then blend / store / pack their own tiles
// under per-group named barriers -- four times the loads in flight of one
// group per block.
constexpr int E32_G = 4, E32_RT = 4;
constexpr int E32_SMEM = E32_G * E32_RT * 32 * 33 * 4;
__global__ void __launch_bounds__(E32_G * 256, 1)
    k_em_tiles32(int64_t blk0, int64_t n_blk, const int32_t* __restrict__ bkm,
                 const int32_t* __restrict__ bkn, const int32_t* __restrict__ toff,
                 const int32_t* __restrict__ tstart, const int32_t* __restrict__ tslab_f,
                 const int32_t* __restrict__ tslab_c, const float* __restrict__ F,
                 float* __restrict__ theta, __nv_bfloat16* __restrict__ mma, int64_t plane_n,
                 float kappa, float step, int planes, int32_t* status) {
  pdl_enter();
  extern __shared__ __align__(16) float e32_tiles[];
  __shared__ float part[E32_G][32];
  const int tid = threadIdx.x, g = tid >> 8, lt = tid & 255;
  const int r = lt >> 3, c4 = (lt & 7) * 4;  // row, column quad
  float* tile = e32_tiles + g * (E32_RT * 32 * 33);
  int informative = 0, bad = 0;
  for (int64_t b = blk0 + blockIdx.x; b < n_blk; b += gridDim.x) {
    const int km = __ldg(bkm + b), kn = __ldg(bkn + b);
    const int t0 = __ldg(toff + b), t1 = __ldg(toff + b + 1);
    if (!split32_blk(km, kn, t1 - t0)) continue;
    const int nt = t1 - t0;
    float4 fv[E32_RT], ov[E32_RT];
    float acc = 0.f;
    for (int c0 = g * E32_RT; c0 < nt; c0 += E32_G * E32_RT) {
#pragma unroll
      for (int u = 0; u < E32_RT; ++u)
        if (c0 + u < nt) fv[u] = ld4(F + __ldg(tstart + t0 + c0 + u) + r * 32 + c4);
#pragma unroll
      for (int u = 0; u < E32_RT; ++u)
        if (c0 + u < nt)
          acc += (fv[u].x + kappa) + (fv[u].y + kappa) + (fv[u].z + kappa) + (fv[u].w + kappa);
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((lt & 7) == 0) part[g][r] = acc;
    __syncthreads();
    float tot = 0.f;
#pragma unroll
    for (int q = 0; q < E32_G; ++q) tot += part[q][r];
    const float inv = tot > 0.f ? 1.f / tot : 0.f;
    if (tot > 0.f && g == 0 && (lt & 7) == 0) ++informative;
    for (int c0 = g * E32_RT; c0 < nt; c0 += E32_G * E32_RT) {
      const int nc = min(E32_RT, nt - c0);
#pragma unroll
      for (int u = 0; u < E32_RT; ++u) {
        if (u < nc) {
          const int64_t o = __ldg(tstart + t0 + c0 + u) + r * 32 + c4;
          fv[u] = ld4(F + o);
          ov[u] = ld4(theta + o);
        }
      }
#pragma unroll
      for (int u = 0; u < E32_RT; ++u) {
        if (u >= nc) continue;
        float4 o = ov[u];
        if (inv > 0.f) {
          const float4 f = fv[u];
          const float n[4] = {(f.x + kappa) * inv, (f.y + kappa) * inv, (f.z + kappa) * inv,
                              (f.w + kappa) * inv};
          float* op = &o.x;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            op[e] = (step >= 1.f) ? n[e] : ((1.f - step) * op[e] + step * n[e]);
            if (!isfinite(op[e])) ++bad;
          }
          float* tp = theta + __ldg(tstart + t0 + c0 + u) + r * 32 + c4;
          if ((reinterpret_cast<uintptr_t>(tp) & 15) == 0) {
            *reinterpret_cast<float4*>(tp) = o;
          } else {
            tp[0] = o.x, tp[1] = o.y, tp[2] = o.z, tp[3] = o.w;
          }
        }
        if (planes) {
          float* d = tile + u * (32 * 33) + r * 33 + c4;
          d[0] = o.x, d[1] = o.y, d[2] = o.z, d[3] = o.w;
        }
      }
      if (!planes) continue;
      asm volatile("bar.sync %0, 256;" ::"r"(1 + g) : "memory");
      const int n8 = 32 * 32 / 8;
      for (int q = lt; q < nc * 2 * n8; q += 256) {
        const int u = q / (2 * n8), qq = q - u * 2 * n8;
        const float* tl = tile + u * (32 * 33);
        float v[8];
        uint32_t off;
        int pl;
        if (qq < n8) {  // sum-major core row (m, j..j+7)
          const int m = qq >> 2, j = (qq & 3) * 8;
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = tl[m * 33 + j + e];
          off = (uint32_t)tile_off(m, j, 32) * 2u;
          pl = 0;
        } else {  // product-major core row (j, m..m+7)
          const int rr = qq - n8;
          const int j = rr >> 2, m = (rr & 3) * 8;
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = tl[(m + e) * 33 + j];
          off = (uint32_t)tile_off(j, m, 32) * 2u;
          pl = 2;
        }
        uint4 hi, lo;
        split_pack8(v, hi, lo);
        uint8_t* dst = reinterpret_cast<uint8_t*>(
                           pl == 0 ? mma + __ldg(tslab_f + t0 + c0 + u)
                                   : mma + 2 * plane_n + __ldg(tslab_c + t0 + c0 + u)) +
                       off;
        *reinterpret_cast<uint4*>(dst) = hi;
        *reinterpret_cast<uint4*>(dst + plane_n * 2) = lo;
      }
      asm volatile("bar.sync %0, 256;" ::"r"(1 + g) : "memory");
    }
    __syncthreads();  // part[] reused by the next block
  }
  for (int o = 16; o > 0; o >>= 1) {
    informative += __shfl_xor_sync(0xffffffffu, informative, o);
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((tid & 31) == 0) {
    if (informative) atomicAdd(status, informative);
    if (bad) atomicAdd(status + 1, bad);
  }
}

int launch_em_tiles(const pcb_plan* p, cudaStream_t s, const float* f_params, float* theta,
                    float pseudocount, float step, int32_t* status, bool planes, int64_t blk0,
                    int64_t blk1) {
  ProfScope prof_(KC_EM, s);
  if (blk1 < 0) blk1 = p->n_em_blk;
  if (blk1 <= blk0) return PCB_OK;
  // read per launch (tests toggle it)
  const bool split32 = p->em_split32 && getenv("PCB_NO_EM_SPLIT32") == nullptr;
  launch_k(k_em_tiles, dim3(grid_for(blk1 - blk0, 1, 148 * 8)), dim3(EM_THREADS), 0, s, 
      blk0, blk1, p->em_km, p->em_kn, p->em_tile_off, p->em_tile_start, p->em_tile_slab_f,
      p->em_tile_slab_c, f_params, theta, p->mma, p->mma_plane, pseudocount, step,
      planes ? 1 : 0, status, split32 ? 1 : 0);
  if (check_launch()) return PCB_CUDA;
  if (!split32) return PCB_OK;
  static int attr[kMaxDev] = {};
  if (ensure_smem((const void*)k_em_tiles32, E32_SMEM, attr)) return PCB_CUDA;
  launch_k(k_em_tiles32, dim3(grid_for(blk1 - blk0, 1, 148)), dim3(E32_G * 256), (size_t)E32_SMEM,
           s, blk0, blk1, p->em_km, p->em_kn, p->em_tile_off, p->em_tile_start,
           p->em_tile_slab_f, p->em_tile_slab_c, f_params, theta, p->mma, p->mma_plane,
           pseudocount, step, planes ? 1 : 0, status);
  return check_launch();
}

bool em_split32_block(int km, int kn, int ntiles) { return split32_blk(km, kn, ntiles); }

int launch_theta_to_mma(const pcb_plan* p, cudaStream_t s, const float* theta) {
  ProfScope prof_(KC_EM, s);
  if (!p->n_mma_tiles || !p->mma) return PCB_OK;
  launch_k(k_theta_to_mma, dim3(grid_for(p->n_mma_tiles, 1, 148 * 8)), dim3(TM_THREADS), 0, s, 
      p->n_mma_tiles, p->mma_theta, p->mma_slab_f, p->mma_slab_c, p->mma_km, p->mma_kn, theta,
      p->mma, p->mma_plane);
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
  pcb::launch_k(pcb::k_tc_selftest_mn, dim3(1), dim3(128), bytes, reinterpret_cast<cudaStream_t>(stream), 
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
  pcb::launch_k(pcb::k_tc_selftest, dim3(1), dim3(128), bytes, reinterpret_cast<cudaStream_t>(stream), n, k, d_a, d_b,
                                                                                 d_d);
  return pcb::check_launch();
}
