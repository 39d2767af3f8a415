// Warp-specialised, persistent tcgen05 parameter-flow kernel for sm_100a
// (Alg. 3, engine.py:105-126):
//
//   cum[m, j] = sum_b e^{lnf[m,b] - c_b} e^{child[j,b] + c_b}
//   f_params[flow(m, j)] += theta[m, j] * cum[m, j]
//
// a contraction over the batch.  A work item is one (super-row, column
// group, 128-sum M tile, batch slice): M = the tile's sums, N = up to 256
// child columns, K = samples streamed 32 at a time.  The shift c_b is the
// per-sample max over the tile's sum blocks of the ratio shift R (k_ratio,
// log2 units) and cancels between the two operands:
//   A[m, b] = 2^{r[m,b] + R_blk(m)[b] - c_b},   E[j, b] = 2^{child[j,b] log2e + c_b}
// (r = the shifted log2 ratio rows of k_ratio; child = the product
// offsets moved onto the sums' base: offset + (base_pb - base_sum), an
// exact integer difference — the sums of a super-row share one child row,
// hence one base).  Both operands are split
// into bf16 hi + lo and contracted as hi*hi + hi*lo + lo*hi (fp32 TMEM).
//
// Warp roles (18 warps):
//   warp 0       producer: per 32-sample chunk, 2-D TMA boxes (128-byte
//                swizzled) of the tile's r rows, its R rows and the child
//                log-value rows into the raw ring;
//   warp 1       MMA issuer (double-buffered TMEM accumulators, 2 x 256 cols);
//   warps 2-9    converters: the chunk's shifts c_b, then raw -> exponentials
//                -> packed bf16 planes in the K-major core-matrix layout;
//   warps 10-17  epilogue: TMEM -> theta (.) cum -> f_params (plain stores when
//                the group's flow tiles have a single writer and the batch
//                is not sliced; else vector red.add).
#include <math.h>
#include <stdlib.h>

#include "pcb_internal.cuh"
#include "pcb_tc.cuh"
#include "pcb_ws.cuh"

namespace pcb {

using namespace tc;
using namespace ws;

namespace {

constexpr int PF_M = 128;          // sums per tile
constexpr int PF_N = 256;          // child columns per item
#ifndef PCB_PF_KS
#define PCB_PF_KS 32
#endif
constexpr int PF_KS = PCB_PF_KS;   // samples per chunk (one 128-byte swizzled box row)
constexpr int PF_CH = PF_KS / 4;   // 16-byte chunks per box row
constexpr int PF_SWZ = PF_KS * 4;  // TMA swizzle span in bytes (64 or 128)
#ifndef PCB_PF_NCONV
#define PCB_PF_NCONV 10  // 10 converter warps: RAT-SPN parameter flows 14.7 -> 13.9 ms, HCLT 2.34 -> 2.32
#endif
// warps: producer, MMA, converters, 4 epilogue
constexpr int PF_CONV0 = 2, PF_NCONV = PCB_PF_NCONV, PF_EPI0 = PF_CONV0 + PF_NCONV;
// 8 epilogue warps: two per TMEM lane quarter, alternate 16-column chunks
// (the fused-EM path too: the pair meets at a named barrier for the row
// totals and each staged 32 x 32 product-major tile)
constexpr int PF_NEPI = 8;
constexpr int PF_THREADS = (PF_EPI0 + PF_NEPI) * 32;
constexpr int PF_MAXMEM = PF_M / 16;  // sum blocks per tile (k_m >= 16)

struct PfArgs {
  int cap, k_m, lkm, B, ldb;  // lkm = log2(k_m)
  int store;  // 1: each flow entry has exactly one writer in the pass (plain stores)
  int n_items, mtiles, kslices, cgroups, nchunks;
  int64_t sb_base;
  const int32_t *row_off, *members, *sum_ids, *prod_ids, *param_ids, *flow_ids;
  const int32_t* flags;  // per super-row: bit 0 contiguous sum rows, bit 1 contiguous children
  const float* theta;
  float* f_params;
  // fused EM (em != 0): each epilogue thread holds its sum row's whole group;
  // theta and the four bf16 planes of its tiles are rewritten, f_params not
  int em;
  float kappa, step;
  int32_t* status;
  __nv_bfloat16* mma;
  int64_t plane;
  const int32_t *slab_f, *slab_c;
  float* theta_out;
  // pre-converted operands (PRE kernels): per (128-sum tile, chunk) the A
  // hi + lo plane images, per (256-child column group, chunk) the B images
  const uint8_t *prep_a, *prep_e;
};

// RS raw stages and 4 - RS operand stages (32-sample chunks): 2 / 2 for
// HBM-streaming layers, 3 / 1 for dense layers whose operands sit in L2
template <int KN, int RS>
struct PfCfg {
  static constexpr int kA = PF_M * PF_KS * 4;          // raw r rows of the tile
  static constexpr int kE = PF_N * PF_KS * 4;          // raw child rows
  static constexpr int kRP = 128;                      // R row pitch (TMA destinations are 128-B aligned)
  static constexpr int kR = PF_MAXMEM * kRP;            // raw R rows (one per sum block)
  static constexpr int kCPG = PF_N / KN;                // child columns per item
  static constexpr int kBs = kRP;                       // the sums' base row
  static constexpr int kPb = kCPG * kRP;                // the child blocks' base rows
  static constexpr int kRaw = (kA + kE + kR + kBs + kPb + 1023) / 1024 * 1024;  // swizzle-atom aligned
  static constexpr int kOpA = PF_M * PF_KS * 2;        // one bf16 A plane
  static constexpr int kOpB = PF_N * PF_KS * 2;        // one bf16 B plane
  static constexpr int kOp = 2 * kOpA + 2 * kOpB;
  static constexpr int kRS = (PF_KS == 16) ? 5 : RS, kOS = (PF_KS == 16) ? 3 : 4 - RS;
  static constexpr int kBytes = kRS * kRaw + kOS * kOp;
  // PRE: no raw ring, the whole buffer is operand stages
  static constexpr int kOSP = kBytes / kOp;
  static constexpr int kOSmax = kOSP > kOS ? kOSP : kOS;
  static_assert(kRaw % 1024 == 0 && kA % 1024 == 0, "swizzled boxes need aligned bases");
};

struct PfItem {
  int sr, cg, mt, ks;
  int m0, S, r0;       // super-row members
  int s_lo, nmem;      // member blocks of the tile
  int rows;            // live sum rows of the tile
  int kc0, kc1;        // chunk range
};

__device__ __forceinline__ PfItem pf_item(const PfArgs& a, int item) {
  PfItem it;
  it.mt = item % a.mtiles;
  int q = item / a.mtiles;
  it.ks = q % a.kslices;
  q /= a.kslices;
  it.cg = q % a.cgroups;
  it.sr = q / a.cgroups;
  it.m0 = a.row_off[it.sr];
  it.S = a.row_off[it.sr + 1] - it.m0;
  it.r0 = a.members[it.m0];
  const int nsum = it.S * a.k_m;
  it.rows = min(PF_M, nsum - it.mt * PF_M);
  it.s_lo = it.mt * PF_M / a.k_m;
  it.nmem = it.rows > 0 ? (it.rows + a.k_m - 1) / a.k_m : 0;
  const int per = (a.nchunks + a.kslices - 1) / a.kslices;
  it.kc0 = it.ks * per;
  it.kc1 = min(a.nchunks, it.kc0 + per);
  return it;
}

// every column of the item's row is real (flags bit 3): no scan
__device__ __forceinline__ bool pf_dense_row(const PfArgs& a, const PfItem& it) {
  return (__ldg(a.flags + it.sr) & 8) != 0;
}

// the item's real child columns (at most kCPG): writes cols[], returns count
__device__ __forceinline__ int pf_cols(const PfArgs& a, const PfItem& it, int cpg, int* cols) {
  if (pf_dense_row(a, it)) {
    const int n = max(0, min(cpg, a.cap - it.cg * cpg));
    for (int i = 0; i < n; ++i) cols[i] = it.cg * cpg + i;
    return n;
  }
  const int32_t* trow = a.param_ids + (int64_t)it.r0 * a.cap;
  int seen = 0, n = 0;
  for (int c = 0; c < a.cap && n < cpg; ++c) {
    if (__ldg(trow + c) == 0) continue;
    if (seen >= it.cg * cpg) cols[n++] = c;
    ++seen;
  }
  return n;
}

// number of real child columns of the item
__device__ __forceinline__ int pf_ncols(const PfArgs& a, const PfItem& it, int cpg) {
  if (pf_dense_row(a, it)) return max(0, min(cpg, a.cap - it.cg * cpg));
  const int32_t* trow = a.param_ids + (int64_t)it.r0 * a.cap;
  int seen = 0;
  for (int c = 0; c < a.cap; ++c) seen += __ldg(trow + c) != 0;
  return max(0, min(cpg, seen - it.cg * cpg));
}

__device__ __forceinline__ bool pf_active(const PfItem& it) { return it.rows > 0 && it.kc0 < it.kc1; }

// physical 16-byte chunk of logical chunk c of box row `row` under the TMA
// swizzle (128 B: chunk ^ row % 8; 64 B: chunk ^ (row / 2) % 4): 8
// consecutive rows read conflict-free float4s
__device__ __forceinline__ int swz_chunk(int row, int c) {
  return PF_KS == 32 ? (c ^ (row & 7)) : (c ^ ((row >> 1) & 3));
}

}  // namespace

// PRE: the operands were converted once per layer (k_pf_prep, dense uniform
// groups): the producer bulk-copies the bf16 plane images of the item's
// 128-sum tile and 256-child column group straight into the operand ring;
// the converter warps idle.
template <int KN, int RS, bool PRE>
__global__ void __launch_bounds__(PF_THREADS, 1)
    k_param_flow_ws(const PfArgs a, const __grid_constant__ CUtensorMap tm_r,
                    const __grid_constant__ CUtensorMap tm_R, const __grid_constant__ CUtensorMap tm_e,
                    const __grid_constant__ CUtensorMap tm_r128,
                    const __grid_constant__ CUtensorMap tm_Rt,
                    const __grid_constant__ CUtensorMap tm_e256,
                    const __grid_constant__ CUtensorMap tm_vb,
                    const __grid_constant__ CUtensorMap tm_pb,
                    const __grid_constant__ CUtensorMap tm_pbn) {
  pdl_enter();
  using C = PfCfg<KN, RS>;
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int OS = PRE ? C::kOSP : C::kOS;  // operand stages
  __shared__ uint64_t raw_full[C::kRS], raw_empty[C::kRS], op_full[C::kOSmax],
      op_empty[C::kOSmax];
  __shared__ uint64_t acc_full[2], acc_empty[2];
  __shared__ __align__(16) float cs[C::kRS][PF_KS];
  __shared__ int cols_p[C::kCPG];
  // PRE: the converter warps have nothing to convert and join the epilogue
  constexpr int NEW = PRE ? (PF_NEPI + PF_NCONV) / 4 * 4 : PF_NEPI;  // epilogue warps (x4)
  constexpr int CSTEP = 16 * (NEW / 4);                      // column stride per warp
  __shared__ int cols_w[NEW][C::kCPG];  // epilogue warps' column lists
  __shared__ float em_wt[4][32 * 33];  // fused EM: a warp pair's updated 32 x 32 tile
  __shared__ float em_tot[4][2][32];   // fused EM: the pair's partial row totals
  __shared__ uint32_t tmem_base;
  uint8_t* raw = smem;
  uint8_t* ops = PRE ? smem : smem + C::kRS * C::kRaw;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < C::kRS; ++i) {
      mbar_init(smem_u32(&raw_full[i]), 1);
      mbar_init(smem_u32(&raw_empty[i]), PF_NCONV);
    }
    for (int i = 0; i < OS; ++i) {
      mbar_init(smem_u32(&op_full[i]), PRE ? 1 : PF_NCONV);  // PRE: the producer's tx
      mbar_init(smem_u32(&op_empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&acc_full[i]), 1);
      mbar_init(smem_u32(&acc_empty[i]), NEW);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(smem_u32(&tmem_base), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;

  if (PRE && warp == 0) {
    // ------------------------------------------------------------ producer (PRE)
    if (lane == 0) {
      Ring<OS> orr;
      for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
        const PfItem it = pf_item(a, item);
        if (!pf_active(it)) continue;
        const int ncol = pf_cols(a, it, C::kCPG, cols_p);
        if (!ncol) continue;
        const int ta = (__ldg(a.sum_ids + __ldg(a.members + it.m0 + it.s_lo)) - (int)a.sb_base) /
                       PF_M;
        const uint8_t* ia = a.prep_a + ((int64_t)ta * a.nchunks) * (2 * C::kOpA);
        const uint8_t* ie = a.prep_e + ((int64_t)it.cg * a.nchunks) * (2 * C::kOpB);
        for (int kc = it.kc0; kc < it.kc1; ++kc) {
          mbar_wait(smem_u32(&op_empty[orr.slot()]), orr.empty_par());
          const uint32_t of = smem_u32(&op_full[orr.slot()]);
          mbar_arrive_expect_tx(of, (uint32_t)(2 * C::kOpA + 2 * C::kOpB));
          const uint32_t st = smem_u32(ops + orr.slot() * C::kOp);
          bulk_g2s(st, ia + (int64_t)kc * (2 * C::kOpA), (uint32_t)(2 * C::kOpA), of);
          bulk_g2s(st + 2 * C::kOpA, ie + (int64_t)kc * (2 * C::kOpB), (uint32_t)(2 * C::kOpB), of);
          orr.next();
        }
      }
    }
  } else if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      prefetch_tmap(&tm_r);
      prefetch_tmap(&tm_R);
      prefetch_tmap(&tm_e);
      Ring<C::kRS> rr;
      for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
        const PfItem it = pf_item(a, item);
        if (!pf_active(it)) continue;
        const int ncol = pf_cols(a, it, C::kCPG, cols_p);
        if (!ncol) continue;
        const int32_t* prow = a.prod_ids + (int64_t)it.r0 * a.cap;
        // contiguous sum rows / children: one box each (the boxes may cover
        // rows past the tile, which the converters ignore)
        const int fl = __ldg(a.flags + it.sr);
        // R rows are 32-sample (128-byte) boxes whatever the chunk width
        const int a_rows = (fl & 1) ? PF_M : it.nmem * a.k_m;
        const int r_rows = (fl & 1) ? PF_M / a.k_m : it.nmem;
        const int e_rows = (fl & 2) ? PF_N : ncol * KN;
        const int pb_rows = (fl & 2) ? C::kCPG : ncol;
        const uint32_t bytes = (uint32_t)(a_rows + e_rows) * PF_KS * 4 +
                               (uint32_t)(r_rows + 1 + pb_rows) * C::kRP;
        // the tile's sums share one base: that of its first sum block
        const int vb_row =
            (__ldg(a.sum_ids + __ldg(a.members + it.m0 + it.s_lo)) - (int)a.sb_base) / a.k_m;
        for (int kc = it.kc0; kc < it.kc1; ++kc) {
          const int b0 = kc * PF_KS;
          mbar_wait(smem_u32(&raw_empty[rr.slot()]), rr.empty_par());
          const uint32_t rf = smem_u32(&raw_full[rr.slot()]);
          mbar_arrive_expect_tx(rf, bytes);
          const uint32_t st = smem_u32(raw + rr.slot() * C::kRaw);
          if (fl & 1) {
            const int row = __ldg(a.sum_ids + __ldg(a.members + it.m0 + it.s_lo)) - (int)a.sb_base;
            tma_load_2d(st, &tm_r128, b0, row, rf);
            tma_load_2d(st + C::kA + C::kE, &tm_Rt, b0, row / a.k_m, rf);
          } else {
            for (int s = 0; s < it.nmem; ++s) {
              const int row = __ldg(a.sum_ids + __ldg(a.members + it.m0 + it.s_lo + s)) - (int)a.sb_base;
              tma_load_2d(st + s * a.k_m * PF_KS * 4, &tm_r, b0, row, rf);
              tma_load_2d(st + C::kA + C::kE + s * C::kRP, &tm_R, b0, row / a.k_m, rf);
            }
          }
          const uint32_t sb = st + C::kA + C::kE + C::kR;
          tma_load_2d(sb, &tm_vb, b0, vb_row, rf);
          if (fl & 2) {
            tma_load_2d(st + C::kA, &tm_e256, b0, __ldg(prow + cols_p[0]), rf);
            tma_load_2d(sb + C::kBs, &tm_pbn, b0, __ldg(prow + cols_p[0]) / KN, rf);
          } else {
            for (int ci = 0; ci < ncol; ++ci) {
              tma_load_2d(st + C::kA + ci * KN * PF_KS * 4, &tm_e, b0, __ldg(prow + cols_p[ci]), rf);
              tma_load_2d(sb + C::kBs + ci * C::kRP, &tm_pb, b0, __ldg(prow + cols_p[ci]) / KN, rf);
            }
          }
          rr.next();
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    Ring<OS> orr;
    int acc_u = 0;
    constexpr uint32_t SBO = (PF_KS / 8) * 128;
    for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
      const PfItem it = pf_item(a, item);
      if (!pf_active(it)) continue;
      const int ncol = pf_ncols(a, it, C::kCPG);
      if (!ncol) continue;
      const uint32_t idesc = idesc_bf16(PF_M, ncol * KN);
      const int as = acc_u & 1;
      mbar_wait(smem_u32(&acc_empty[as]), (uint32_t)(((acc_u >> 1) & 1) ^ 1));
      tc_fence_after();
      const uint32_t d = tmem + (uint32_t)(as * PF_N);
      for (int kc = it.kc0; kc < it.kc1; ++kc) {
        mbar_wait(smem_u32(&op_full[orr.slot()]), orr.full_par());
        tc_fence_after();
        if (lane == 0) {
          const uint32_t aH = smem_u32(ops + orr.slot() * C::kOp), aL = aH + C::kOpA;
          const uint32_t bH = aL + C::kOpA, bL = bH + C::kOpB;
#pragma unroll
          for (int k = 0; k < PF_KS / 16; ++k) {
            const uint64_t ah = make_desc(aH + k * 256, 128, SBO);
            const uint64_t al = make_desc(aL + k * 256, 128, SBO);
            const uint64_t bh = make_desc(bH + k * 256, 128, SBO);
            const uint64_t bl = make_desc(bL + k * 256, 128, SBO);
            mma_bf16_keep_a(d, ah, bh, idesc, (kc > it.kc0 || k > 0) ? 1u : 0u);
            mma_bf16_reuse_a(d, ah, bl, idesc, 1u);
            mma_bf16(d, al, bh, idesc, 1u);
          }
          mma_commit(smem_u32(&op_empty[orr.slot()]));
        }
        __syncwarp();
        orr.next();
      }
      if (lane == 0) mma_commit(smem_u32(&acc_full[as]));
      __syncwarp();
      ++acc_u;
    }
  } else if (!PRE && warp < PF_EPI0) {
    // ------------------------------------------------------------ converters
    if constexpr (!PRE) {
    const int t = tid - PF_CONV0 * 32;  // 0..PF_NCONV*32-1
    Ring<C::kRS> rr;
    Ring<C::kOS> orr;
    for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
      const PfItem it = pf_item(a, item);
      if (!pf_active(it)) continue;
      const int ncol = pf_ncols(a, it, C::kCPG);
      if (!ncol) continue;
      const int npad = ncol * KN;
      for (int kc = it.kc0; kc < it.kc1; ++kc) {
        const int b0 = kc * PF_KS;
        mbar_wait(smem_u32(&raw_full[rr.slot()]), rr.full_par());
        const float* rA = reinterpret_cast<const float*>(raw + rr.slot() * C::kRaw);
        const float* rE = rA + C::kA / 4;
        const float* rR = rE + C::kE / 4;
        const float* rB = rR + C::kR / 4;             // the sums' base (32 samples)
        const float* rP = rB + C::kBs / 4;            // child block bases, kRP pitch
        float* c_s = cs[rr.slot()];
        if (t < PF_KS) {  // the chunk's per-sample shift: max of R over the tile's blocks
          float v = PCB_NEG_INF;
          if (b0 + t < a.B)
            for (int s = 0; s < it.nmem; ++s) v = fmaxf(v, rR[s * (C::kRP / 4) + t]);
          c_s[t] = v;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(PF_NCONV * 32) : "memory");
        mbar_wait(smem_u32(&op_empty[orr.slot()]), orr.empty_par());
        uint8_t* oAh = ops + orr.slot() * C::kOp;
        uint8_t* oAl = oAh + C::kOpA;
        uint8_t* oBh = oAl + C::kOpA;
        uint8_t* oBl = oBh + C::kOpB;
        // raw boxes are swizzled (swz_chunk)
        const float4* rA4 = reinterpret_cast<const float4*>(rA);
        const float4* rE4 = reinterpret_cast<const float4*>(rE);
        const float4* rR4 = reinterpret_cast<const float4*>(rR);
        const float4* c4 = reinterpret_cast<const float4*>(c_s);
        // A: 128 rows x 4 octets; thread -> (row = q % 128, octet = q / 128)
#ifdef PCB_ABL_CONV
        if (false)
#endif
        for (int q = t; q < PF_M * (PF_KS / 8); q += PF_NCONV * 32) {
          const int m = q & (PF_M - 1), o = q >> 7;
          float v[8];
          if (m < it.rows) {
            const int blk = m >> a.lkm;
            const float4 x0 = rA4[m * PF_CH + swz_chunk(m, 2 * o)];
            const float4 x1 = rA4[m * PF_CH + swz_chunk(m, 2 * o + 1)];
            const float4 R0 = rR4[blk * (C::kRP / 16) + 2 * o];
            const float4 R1 = rR4[blk * (C::kRP / 16) + 2 * o + 1];
            const float4 c0 = c4[2 * o], c1 = c4[2 * o + 1];
            const float xs[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
            const float Rs[8] = {R0.x, R0.y, R0.z, R0.w, R1.x, R1.y, R1.z, R1.w};
            const float cc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
            for (int e = 0; e < 8; ++e)
              v[e] = (cc[e] == PCB_NEG_INF) ? 0.f : ex2(xs[e] + (Rs[e] - cc[e]));
          } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = 0.f;
          }
          uint4 hi, lo;
          split_pack8(v, hi, lo);
          const uint32_t off = kmajor_off(m, o * 8, PF_KS);
          *reinterpret_cast<uint4*>(oAh + off) = hi;
          *reinterpret_cast<uint4*>(oAl + off) = lo;
        }
        // E: npad rows x 4 octets
        const float4* rB4 = reinterpret_cast<const float4*>(rB);
        const float4* rP4 = reinterpret_cast<const float4*>(rP);
#ifdef PCB_ABL_CONV
        if (false)
#endif
        for (int o = 0; o < PF_KS / 8; ++o)
        for (int n = t; n < npad; n += PF_NCONV * 32) {
          const float4 x0 = rE4[n * PF_CH + swz_chunk(n, 2 * o)];
          const float4 x1 = rE4[n * PF_CH + swz_chunk(n, 2 * o + 1)];
          const float4 c0 = c4[2 * o], c1 = c4[2 * o + 1];
          const float4 p0 = rP4[(n / KN) * (C::kRP / 16) + 2 * o];
          const float4 p1 = rP4[(n / KN) * (C::kRP / 16) + 2 * o + 1];
          const float4 s0 = rB4[2 * o], s1 = rB4[2 * o + 1];
          const float xs[8] = {x0.x + (p0.x - s0.x), x0.y + (p0.y - s0.y), x0.z + (p0.z - s0.z),
                               x0.w + (p0.w - s0.w), x1.x + (p1.x - s1.x), x1.y + (p1.y - s1.y),
                               x1.z + (p1.z - s1.z), x1.w + (p1.w - s1.w)};
          const float cc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            v[e] = (cc[e] == PCB_NEG_INF) ? 0.f : fminf(ex2(fmaf(xs[e], kL2E, cc[e])), 1e37f);
          uint4 hi, lo;
          split_pack8(v, hi, lo);
          const uint32_t off = kmajor_off(n, o * 8, PF_KS);
          *reinterpret_cast<uint4*>(oBh + off) = hi;
          *reinterpret_cast<uint4*>(oBl + off) = lo;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(smem_u32(&raw_empty[rr.slot()]));
          mbar_arrive(smem_u32(&op_full[orr.slot()]));
        }
        rr.next();
        orr.next();
      }
    }
    }  // !PRE
  } else {
    // ------------------------------------------------------------ epilogue
    // NEW / 4 warps per TMEM lane quarter (q4 = warp % 4), each taking every
    // (NEW / 4)-th 16-column chunk
    const int ew = warp - (PRE ? PF_CONV0 : PF_EPI0);
    if (ew < NEW) {  // PRE: converter warps past a multiple of four stay idle
    const int q4 = warp & 3;
    const int h = ew >> 2;          // column phase: chunks h*16, h*16 + CSTEP, ...
    const int er = q4 * 32 + lane;  // sum row within the tile (TMEM lane)
    int* cols = cols_w[ew];
    int acc_u = 0;
    int em_inf = 0, em_bad = 0;
    for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
      const PfItem it = pf_item(a, item);
      if (!pf_active(it)) continue;
      int ncol = 0;
      if (lane == 0) ncol = pf_cols(a, it, C::kCPG, cols);
      ncol = __shfl_sync(0xffffffffu, ncol, 0);
      __syncwarp();
      if (!ncol) continue;
      const bool live = er < it.rows;
      const int s = it.s_lo + (live ? er / a.k_m : 0);
      const int mm = er % a.k_m;
      const int64_t rowbase = (int64_t)__ldg(a.members + it.m0 + s) * a.cap;
      const int as = acc_u & 1;
      // theta of the next 16 columns (one row segment: 4 float4) is loaded
      // before this chunk's TMEM read
      auto tile_of = [&](int c0) {
        return (int64_t)__ldg(a.param_ids + rowbase + cols[c0 / KN]) + mm * KN + (c0 % KN);
      };
      auto load_th = [&](int64_t tile, float* th) {
        const float* tp = a.theta + tile;
        if ((tile & 3) == 0) {
#pragma unroll
          for (int i = 0; i < 16; i += 4) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(tp + i));
            th[i] = q.x, th[i + 1] = q.y, th[i + 2] = q.z, th[i + 3] = q.w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) th[i] = __ldg(tp + i);
        }
      };
      float th[16], thn[16];
      if (live && h * 16 < ncol * KN) load_th(tile_of(h * 16), thn);
      mbar_wait(smem_u32(&acc_full[as]), (uint32_t)((acc_u >> 1) & 1));
      tc_fence_after();
      const uint32_t tbase = tmem + (uint32_t)(as * PF_N) + ((uint32_t)(q4 * 32) << 16);
      if constexpr (KN == 32 && !PRE) {
        if (a.em) {
          // Fused EM, the two warps of a lane quarter (same 32 rows) split
          // the columns in 16-wide chunks as in the plain epilogue and meet
          // at a pair barrier (ids 2..5) for the row total and each 32 x 32
          // product-major tile.
          auto pair_bar = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(2 + q4) : "memory"); };
          // pass 1: the row's group total sum(F + k) over all its columns
          float tot = 0.f;
          for (int c0 = h * 16; c0 < ncol * KN; c0 += 32) {
#pragma unroll
            for (int i = 0; i < 16; ++i) th[i] = thn[i];
            if (live && c0 + 32 < ncol * KN) load_th(tile_of(c0 + 32), thn);
            float v[16];
            tmem_ld16(tbase + c0, v);
            if (!live) continue;
#pragma unroll
            for (int i = 0; i < 16; ++i) tot += ((th[i] != 0.f) ? th[i] * v[i] : 0.f) + a.kappa;
          }
          em_tot[q4][h][lane] = tot;
          pair_bar();
          tot = em_tot[q4][0][lane] + em_tot[q4][1][lane];  // same order on both warps
          const bool inf_row = live && tot > 0.f;
          const float inv = inf_row ? 1.f / tot : 0.f;
          if (h == 0) em_inf += inf_row;
          // pass 2: blend, store theta, pack the sum-major planes; stage the
          // tile for the product-major planes
          if (live) load_th(tile_of(h * 16), thn);
          float* wt = em_wt[q4];
          for (int c0 = h * 16; c0 < ncol * KN; c0 += 32) {
#pragma unroll
            for (int i = 0; i < 16; ++i) th[i] = thn[i];
            if (live && c0 + 32 < ncol * KN) load_th(tile_of(c0 + 32), thn);
            float v[16];
            tmem_ld16(tbase + c0, v);
            const int c = cols[c0 / KN];
            const int j0 = c0 % KN;
            if (live) {
              float nt[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const float f = (th[i] != 0.f) ? th[i] * v[i] : 0.f;
                const float n = (f + a.kappa) * inv;
                nt[i] = inf_row ? ((a.step >= 1.f) ? n : ((1.f - a.step) * th[i] + a.step * n))
                                : th[i];
                if (inf_row && !isfinite(nt[i])) ++em_bad;
              }
              const int64_t tile = __ldg(a.param_ids + rowbase + c);
              float* tp = a.theta_out + tile + mm * KN + j0;
              if ((tile & 3) == 0) {
#pragma unroll
                for (int i = 0; i < 16; i += 4)
                  *reinterpret_cast<float4*>(tp + i) = make_float4(nt[i], nt[i + 1], nt[i + 2], nt[i + 3]);
              } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) tp[i] = nt[i];
              }
              __nv_bfloat16* fpl = a.mma + __ldg(a.slab_f + rowbase + c);
#pragma unroll
              for (int h2 = 0; h2 < 2; ++h2) {
                float e8[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) e8[e] = nt[8 * h2 + e];
                uint4 hi, lo;
                split_pack8(e8, hi, lo);
                uint8_t* dst = reinterpret_cast<uint8_t*>(fpl) +
                               (uint32_t)tile_off(mm, j0 + 8 * h2, KN) * 2u;
                *reinterpret_cast<uint4*>(dst) = hi;
                *reinterpret_cast<uint4*>(dst + a.plane * 2) = lo;
              }
#pragma unroll
              for (int i = 0; i < 16; ++i) wt[lane * 33 + j0 + i] = nt[i];
            }
            pair_bar();  // the pair's 32 x 32 tile is staged
            if (live) {  // k_m == 32: a lane quarter is live or dead as a whole
              __nv_bfloat16* cpl = a.mma + 2 * a.plane + __ldg(a.slab_c + rowbase + c);
#pragma unroll
              for (int k = 2 * h; k < 2 * h + 2; ++k) {
                const int q = lane + 32 * k, j = q >> 2, g8 = (q & 3) * 8;
                float e8[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) e8[e] = wt[(g8 + e) * 33 + j];
                uint4 hi, lo;
                split_pack8(e8, hi, lo);
                uint8_t* dst = reinterpret_cast<uint8_t*>(cpl) + (uint32_t)tile_off(j, g8, KN) * 2u;
                *reinterpret_cast<uint4*>(dst) = hi;
                *reinterpret_cast<uint4*>(dst + a.plane * 2) = lo;
              }
            }
            pair_bar();  // the tile is read before the next one is staged
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&acc_empty[as]));
          ++acc_u;
          continue;
        }
      }
      for (int c0 = h * 16; c0 < ncol * KN; c0 += CSTEP) {
#pragma unroll
        for (int i = 0; i < 16; ++i) th[i] = thn[i];
#ifndef PCB_ABL_EPI
        if (live && c0 + CSTEP < ncol * KN) load_th(tile_of(c0 + CSTEP), thn);
#endif
        float v[16];
        tmem_ld16(tbase + c0, v);
#ifdef PCB_ABL_EPI
        if (v[0] != 12345.f) continue;
#endif
        if (!live) continue;
        const int c = cols[c0 / KN];
        const int j0 = c0 % KN;
        const int64_t tile = __ldg(a.param_ids + rowbase + c) + mm * KN + j0;
        const int64_t flow = __ldg(a.flow_ids + rowbase + c) + mm * KN + j0;
        float* dst = a.f_params + flow;
        float w[16];  // zero-theta terms skipped (an overflowed cum must not make inf * 0)
#pragma unroll
        for (int i = 0; i < 16; ++i) w[i] = (th[i] != 0.f) ? th[i] * v[i] : 0.f;
        const bool vec = ((tile | flow) & 3) == 0;
        if (a.store && vec) {
#pragma unroll
          for (int i = 0; i < 16; i += 4)
            *reinterpret_cast<float4*>(dst + i) = make_float4(w[i], w[i + 1], w[i + 2], w[i + 3]);
        } else if (a.store) {
#pragma unroll
          for (int i = 0; i < 16; ++i) dst[i] = w[i];
        } else if (vec) {
#pragma unroll
          for (int i = 0; i < 16; i += 4)
            atomicAdd(reinterpret_cast<float4*>(dst + i), make_float4(w[i], w[i + 1], w[i + 2], w[i + 3]));
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (w[i] != 0.f) atomicAdd(dst + i, w[i]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&acc_empty[as]));
      ++acc_u;
    }
    if (a.em) {
      for (int o = 16; o > 0; o >>= 1) {
        em_inf += __shfl_xor_sync(0xffffffffu, em_inf, o);
        em_bad += __shfl_xor_sync(0xffffffffu, em_bad, o);
      }
      if (lane == 0 && em_inf) atomicAdd(a.status, em_inf);
      if (lane == 0 && em_bad) atomicAdd(a.status + 1, em_bad);
    }
    }  // ew < NEW
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free(tmem, 512);
}

// batch slices so small layers still cover the SMs; >= 2 chunks per slice
int pf_kslices(int64_t count, int64_t cap, int kn, int B) {
  const int64_t base = count * ((cap * kn + PF_N - 1) / PF_N) * 2;
  const int nchunks = (B + PF_KS - 1) / PF_KS;
  const int ks = (int)((2 * sm_count() + base - 1) / base);
  return max(1, min(ks, nchunks / 2));
}

namespace {

// ---------------------------------------------------------------- pre-conversion
// Dense uniform groups (pf_pre_ok: every sum block over the same child row,
// several 128-sum tiles and 256-child column groups per layer, e.g. HMM
// transitions): each operand is converted once per layer instead of once per
// item that uses it (the B operand 2 x (sum rows / 256) times, the A operand
// (child columns / 256) times).  The shift is one per sample for the whole
// layer, c_b = max over its sum blocks of R (it cancels between the
// operands as the per-tile shift does).
//   prep row 0          c_b
//   A images            per (128-sum tile, 32-sample chunk): hi plane, lo
//                       plane of 2^(r + R - c) in the MMA's K-major layout
//   B images            per (256-child column group, chunk): hi, lo planes
//                       of 2^((o + base_pb - base_sum) log2 e + c)
// CTA = 32 samples x 32 thread rows striding over the sum blocks
__global__ void __launch_bounds__(1024)
    k_pf_shift(int n_sb, int B, int ldb, const float* __restrict__ rmax, float* __restrict__ c) {
  pdl_enter();
  __shared__ float part[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int b = blockIdx.x * 32 + tx;
  float m = PCB_NEG_INF;
  if (b < B)
    for (int k = ty; k < n_sb; k += 32) m = fmaxf(m, __ldg(rmax + (int64_t)k * ldb + b));
  part[ty][tx] = m;
  __syncthreads();
  if (ty == 0 && b < ldb) {
#pragma unroll 8
    for (int y = 1; y < 32; ++y) m = fmaxf(m, part[y][tx]);
    c[b] = m;
  }
}

__global__ void __launch_bounds__(256)
    k_pf_prep(int n_a, int n_e, int k_m, int kn, int nstride, int kc_off, int ldb, int cap,
              const int32_t* __restrict__ prod_row0, const int32_t* __restrict__ param_row0,
              const float* __restrict__ ratio, const float* __restrict__ rmax,
              const float* __restrict__ scratch, const float* __restrict__ pbase,
              const float* __restrict__ vbase, const float* __restrict__ c,
              uint8_t* __restrict__ img_a, uint8_t* __restrict__ img_e) {
  pdl_enter();
  constexpr int kOpA = PF_M * PF_KS * 2, kOpB = PF_N * PF_KS * 2;
  __shared__ int child0, n_real;
  if (threadIdx.x == 0) {
    int first = 0, cnt = 0;
    while (first < cap && __ldg(param_row0 + first) == 0) ++first;
    for (int q = 0; q < cap; ++q) cnt += __ldg(param_row0 + q) != 0;
    child0 = first < cap ? __ldg(prod_row0 + first) : 0;
    n_real = cnt * kn;  // contiguous real child rows (pf_pre_ok)
  }
  __syncthreads();
  const int oct = ldb / 8;
  const int64_t total = (int64_t)(n_a + n_e) * oct;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(t / oct), b0 = (int)(t % oct) * 8;
    const int kc = b0 / PF_KS, k = b0 % PF_KS;
    const float4 c0 = *reinterpret_cast<const float4*>(c + b0);
    const float4 c1 = *reinterpret_cast<const float4*>(c + b0 + 4);
    const float cc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    float v[8];
    uint8_t* dst;
    uint32_t plane;
    if (row < n_a) {
      const float* rr = ratio + (int64_t)row * ldb + b0;
      const float* RR = rmax + (int64_t)(row / k_m) * ldb + b0;
      const float4 x0 = *reinterpret_cast<const float4*>(rr);
      const float4 x1 = *reinterpret_cast<const float4*>(rr + 4);
      const float4 R0 = *reinterpret_cast<const float4*>(RR);
      const float4 R1 = *reinterpret_cast<const float4*>(RR + 4);
      const float xs[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
      const float Rs[8] = {R0.x, R0.y, R0.z, R0.w, R1.x, R1.y, R1.z, R1.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = (cc[e] == PCB_NEG_INF) ? 0.f : ex2(xs[e] + (Rs[e] - cc[e]));
      dst = img_a + ((int64_t)(row / PF_M) * nstride + kc_off + kc) * (2 * kOpA) +
            kmajor_off(row % PF_M, k, PF_KS);
      plane = kOpA;
    } else {
      const int n = row - n_a;
      if (n >= n_real) continue;
      const int srow = child0 + n;
      const float* xr = scratch + (int64_t)srow * ldb + b0;
      const float* pr = pbase + (int64_t)(srow / kn) * ldb + b0;
      const float4 x0 = *reinterpret_cast<const float4*>(xr);
      const float4 x1 = *reinterpret_cast<const float4*>(xr + 4);
      const float4 p0 = *reinterpret_cast<const float4*>(pr);
      const float4 p1 = *reinterpret_cast<const float4*>(pr + 4);
      const float4 s0 = *reinterpret_cast<const float4*>(vbase + b0);
      const float4 s1 = *reinterpret_cast<const float4*>(vbase + b0 + 4);
      const float xs[8] = {x0.x + (p0.x - s0.x), x0.y + (p0.y - s0.y), x0.z + (p0.z - s0.z),
                           x0.w + (p0.w - s0.w), x1.x + (p1.x - s1.x), x1.y + (p1.y - s1.y),
                           x1.z + (p1.z - s1.z), x1.w + (p1.w - s1.w)};
#pragma unroll
      for (int e = 0; e < 8; ++e)
        v[e] = (cc[e] == PCB_NEG_INF) ? 0.f : fminf(ex2(fmaf(xs[e], kL2E, cc[e])), 1e37f);
      dst = img_e + ((int64_t)(n / PF_N) * nstride + kc_off + kc) * (2 * kOpB) +
            kmajor_off(n % PF_N, k, PF_KS);
      plane = kOpB;
    }
    uint4 hi, lo;
    split_pack8(v, hi, lo);
    *reinterpret_cast<uint4*>(dst) = hi;
    *reinterpret_cast<uint4*>(dst + plane) = lo;
  }
}

template <int KN, int RS>
int launch_pf(const PfArgs& a0, const Layer& L, const float* ratio, const float* rmax,
              const float* scratch, const float* vbase, const float* pbase, cudaStream_t s,
              float* prep = nullptr, const PfFuse* fuse = nullptr) {
  using C = PfCfg<KN, RS>;
  const bool pre = prep != nullptr;
  static int attr[kMaxDev] = {}, attr_p[kMaxDev] = {};
  if (ensure_smem((const void*)k_param_flow_ws<KN, RS, false>, C::kBytes, attr) ||
      (pre && ensure_smem((const void*)k_param_flow_ws<KN, RS, true>, C::kBytes, attr_p)))
    return PCB_CUDA;
  PfArgs a = a0;
  a.cgroups = (int)((a.cap * KN + PF_N - 1) / PF_N);
  a.mtiles = 2;  // super-rows hold <= 256 sums
  a.nchunks = (a.B + PF_KS - 1) / PF_KS;
  a.kslices = pf_kslices(a.n_items, a.cap, KN, a.B);  // n_items holds the super-row count here
  const int base = a.n_items * a.cgroups * a.mtiles;
  a.n_items = base * a.kslices;
  auto base_items = [base](const PfArgs&) { return base; };
  a.store = a.store && a.kslices == 1;  // batch slices add partial sums
  if (a.em && (a.kslices != 1 || a.cgroups != 1)) return PCB_USAGE;  // needs whole rows
  CUtensorMap tr, tR, te, tr128, tRt, te256, tvb, tpb, tpbn;
  if (make_rows_map(&tr, ratio, L.n_sb * L.k_m, a.ldb, (int)L.k_m, PF_KS, PF_SWZ) ||
      make_rows_map(&tR, rmax, L.n_sb, a.ldb, 1, C::kRP / 4, 0) ||
      make_rows_map(&te, scratch, L.window, a.ldb, KN, PF_KS, PF_SWZ) ||
      make_rows_map(&tr128, ratio, L.n_sb * L.k_m, a.ldb, PF_M, PF_KS, PF_SWZ) ||
      make_rows_map(&tRt, rmax, L.n_sb, a.ldb, PF_M / (int)L.k_m, C::kRP / 4, 0) ||
      make_rows_map(&te256, scratch, L.window, a.ldb, PF_N, PF_KS, PF_SWZ) ||
      make_rows_map(&tvb, vbase, L.n_sb, a.ldb, 1, C::kRP / 4, 0) ||
      make_rows_map(&tpb, pbase, L.n_pb, a.ldb, 1, C::kRP / 4, 0) ||
      make_rows_map(&tpbn, pbase, L.n_pb, a.ldb, C::kCPG, C::kRP / 4, 0))
    return PCB_CUDA;
  if (pre) {
    // the layer's operands once: shift row, A images (all sum rows), B images.
    // A fusion member writes its segment (chunks rank * nchunks ...) of the
    // group's images; the rank-0 member (last in the backward pass) then runs
    // one contraction over all n segments, storing every flow once
    const int n_a = (int)(L.n_sb * L.k_m), n_e = a.cap * KN;
    const int64_t a_rows = (n_a + PF_M - 1) / PF_M * PF_M;
    const int nseg = fuse ? fuse->n : 1, rank = fuse ? fuse->rank : 0;
    float* base = fuse ? fuse->prep : prep;
    float* c = base + (int64_t)rank * a.ldb;
    uint8_t* img_a = reinterpret_cast<uint8_t*>(base + (int64_t)nseg * a.ldb);
    uint8_t* img_e = reinterpret_cast<uint8_t*>(base + (int64_t)nseg * (1 + a_rows) * a.ldb);
    launch_k(k_pf_shift, dim3((a.ldb + 31) / 32), dim3(1024), 0, s, (int)L.n_sb, a.B, a.ldb, rmax, c);
    if (check_launch()) return PCB_CUDA;
    const int64_t tasks = (int64_t)(n_a + n_e) * (a.ldb / 8);
    launch_k(k_pf_prep, dim3(grid_for(tasks, 256)), dim3(256), 0, s, n_a, n_e, (int)L.k_m, KN,
             nseg * a.nchunks, rank * a.nchunks, a.ldb, a.cap, a.prod_ids, a.param_ids, ratio,
             rmax, scratch, pbase, vbase, c, img_a, img_e);
    if (check_launch()) return PCB_CUDA;
    a.prep_a = img_a;
    a.prep_e = img_e;
    if (fuse) {
      if (rank != 0) return PCB_OK;  // operands staged; the rank-0 member contracts
      a.nchunks *= nseg;
      a.kslices = 1;
      a.n_items = base_items(a);
      a.store = 1;  // the group's tiles have no writer outside this launch
    }
  }
  const int grid = min(a.n_items, sm_count());
  if (pre)
    launch_k((k_param_flow_ws<KN, RS, true>), dim3(grid), dim3(PF_THREADS), C::kBytes, s, 
        a, tr, tR, te, tr128, tRt, te256, tvb, tpb, tpbn);
  else
    launch_k((k_param_flow_ws<KN, RS, false>), dim3(grid), dim3(PF_THREADS), C::kBytes, s, 
        a, tr, tR, te, tr128, tRt, te256, tvb, tpb, tpbn);
  return check_launch();
}

}  // namespace

// PCB_PF_NO_PRE=1: convert per item as for every other group (A/B experiments)
static bool pf_pre_off() {
  static const bool off = getenv("PCB_PF_NO_PRE") != nullptr;
  return off;
}

bool pf_fusable(const Layer& L) {
  return L.pf_fuse >= 0 && L.fwd.size() == 1 && L.fwd[0].pf_pre && L.k_n == 32 && !pf_pre_off() &&
         getenv("PCB_NO_PF_FUSE") == nullptr;
}

int64_t pf_prep_rows(const Layer& L, const FwdGroup& g) {
  // the shift row, A images (sum rows to a 128 multiple), B images (child
  // columns to a 256 multiple); one bf16 hi + lo pair per element = 1 float
  return 1 + (L.n_sb * L.k_m + PF_M - 1) / PF_M * PF_M + (g.cap * L.k_n + PF_N - 1) / PF_N * PF_N;
}

bool pf_ws_supported(const Layer& L) {
  return (L.k_n == 16 || L.k_n == 32 || L.k_n == 64) && (L.k_m == 16 || L.k_m == 32 || L.k_m == 64);
}

// the layer's parameter flows are all plain stores at batch size B (so its
// f_params range needs no zeroing)
bool pf_layer_stores(const pcb_plan* P, const Layer& L, int B) {
  if (P->use_tc != 1 || !pf_ws_supported(L)) return false;
  for (size_t g = 0; g < L.fwd.size(); ++g) {
    const TcRows& T = L.pf_tc[g];
    if (!T.count || !L.fwd[g].exclusive) return false;
    if (pf_kslices(T.count, L.fwd[g].cap, (int)L.k_n, B) != 1) return false;
  }
  return true;
}


int launch_param_flow_ws(const Layer& L, const FwdGroup& g, const TcRows& tc, cudaStream_t s,
                         int B, int ldb, const float* theta, const float* ratio, const float* rmax,
                         const float* scratch, const float* vbase, const float* pbase,
                         float* f_params, const PfEm* em, float* prep, const PfFuse* fuse) {
  ProfScope prof_(KC_PARAM_FLOW, s);
  if (!tc.count || !B) return PCB_OK;
  PfArgs a{};
  a.cap = (int)g.cap;
  a.k_m = (int)L.k_m;
  a.lkm = __builtin_ctz((unsigned)L.k_m);
  a.B = B;
  a.ldb = ldb;
  a.n_items = (int)tc.count;
  a.sb_base = L.sb_base;
  a.row_off = tc.row_off;
  a.members = tc.members;
  a.sum_ids = g.sum_ids;
  a.prod_ids = g.prod_ids;
  a.param_ids = g.param_ids;
  a.flow_ids = g.flow_ids;
  a.flags = tc.flags;
  a.theta = theta;
  a.f_params = f_params;
  a.store = g.exclusive;
  if (em) {
    a.em = 1;
    a.kappa = em->kappa;
    a.step = em->step;
    a.status = em->status;
    a.mma = em->mma;
    a.plane = em->plane;
    a.slab_f = g.param_slab;
    a.slab_c = g.param_slab_c;
    a.theta_out = em->theta;
  }
  // dense layers (several 256-child column groups) re-read operands from L2:
  // a deeper raw ring pays there
  const bool dense = g.cap * L.k_n > PF_N;
  switch (L.k_n) {
    case 16: return dense ? launch_pf<16, 3>(a, L, ratio, rmax, scratch, vbase, pbase, s)
                          : launch_pf<16, 2>(a, L, ratio, rmax, scratch, vbase, pbase, s);
#ifndef PCB_PF_RS32
#define PCB_PF_RS32 2
#endif
#ifndef PCB_PF_DENSE_RS
#define PCB_PF_DENSE_RS 2
#endif
    case 32: {
      // PRE (operands converted once per layer): every stage is an operand
      // stage.  Dense without PRE (RAT-SPN's 1024-child rows): keep two
      // operand stages -- three raw stages leave one, which serialises the
      // converters and the MMAs
      const bool pre = g.pf_pre && !em && !pf_pre_off();
      if (dense && pre)
        return launch_pf<32, 3>(a, L, ratio, rmax, scratch, vbase, pbase, s, prep, fuse);
      if (dense) return launch_pf<32, PCB_PF_DENSE_RS>(a, L, ratio, rmax, scratch, vbase, pbase, s);
      return launch_pf<32, PCB_PF_RS32>(a, L, ratio, rmax, scratch, vbase, pbase, s);
    }
    case 64: return dense ? launch_pf<64, 3>(a, L, ratio, rmax, scratch, vbase, pbase, s)
                          : launch_pf<64, 2>(a, L, ratio, rmax, scratch, vbase, pbase, s);
    default: return PCB_USAGE;
  }
}

}  // namespace pcb
