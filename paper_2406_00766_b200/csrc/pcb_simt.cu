// SIMT kernels of the hot path: inputs, products, the generic (any block
// size, incl. demoted K=1) sum-layer forward / parameter-flow / child-flow
// kernels, flow bookkeeping, replica reduction and EM.
//
// Numerics follow pcirc/runtime/engine.py exactly (Appendix B of SURVEY.md):
// streaming (lin, top) merge with dead-tile skipping, log-flow rescaling by a
// per-sample block maximum, zero flow for impossible nodes; fp32 throughout.
#include <math.h>
#include <stdlib.h>

#include "pcb_internal.cuh"
#include "pcb_tc.cuh"

namespace pcb {

unsigned long long g_launches = 0;

bool pdl_enabled() {
  static const bool on = getenv("PCB_NO_PDL") == nullptr;
  return on;
}

int check_launch() {
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PCB_OK : PCB_CUDA;
}

// ---------------------------------------------------------------- profiling
namespace {
struct ProfRec {
  int cls;
  cudaEvent_t a, b;
  unsigned long long launches;
};
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_event_pool;
cudaEvent_t take_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

ProfScope::ProfScope(int c, cudaStream_t st) : cls(c), s(st), l0(g_launches), slot(-1) {
  if (!g_prof_on) return;
  ProfRec r{c, take_event(), take_event(), 0};
  cudaEventRecord(r.a, s);
  slot = (int)g_prof.size();
  g_prof.push_back(r);
}

ProfScope::~ProfScope() {
  if (slot < 0) return;
  cudaEventRecord(g_prof[slot].b, s);
  g_prof[slot].launches = g_launches - l0;
}

}  // namespace pcb

extern "C" int pcb_profile_enable(int on) {
  pcb::g_prof_on = on != 0;
  return PCB_OK;
}

// Per class: total milliseconds, number of wrapper scopes, number of kernel
// launches since the last read.  Synchronises on the recorded events.
extern "C" int pcb_profile_read(double* ms, int64_t* scopes, int64_t* launches, int n) {
  using namespace pcb;
  for (int i = 0; i < n; ++i) {
    ms[i] = 0;
    scopes[i] = 0;
    launches[i] = 0;
  }
  int st = PCB_OK;
  for (auto& r : g_prof) {
    float t = 0.f;
    if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess)
      st = PCB_CUDA;
    if (r.cls < n) {
      ms[r.cls] += t;
      scopes[r.cls] += 1;
      launches[r.cls] += (int64_t)r.launches;
    }
    g_event_pool.push_back(r.a);
    g_event_pool.push_back(r.b);
  }
  g_prof.clear();
  return st;
}

namespace pcb {

// ---------------------------------------------------------------- K1 inputs
// values[slot_i, b] = log theta[pmf_i + x[var_i, b]], 0 when x is missing
// (engine.py:55-65).  Threads run along the batch so x and values coalesce.
__global__ void k_input_fwd(int64_t n, int B, int ldb, const int32_t* __restrict__ slots,
                            const int32_t* __restrict__ vars, const int32_t* __restrict__ pids,
                            const int32_t* __restrict__ xT, const float* __restrict__ theta,
                            float* __restrict__ values) {
  pdl_enter();
  int64_t total = n * (int64_t)B;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / B;
    int b = (int)(t - i * B);
    int x = xT[(int64_t)vars[i] * ldb + b];
    float v = 0.f;
    if (x >= 0) v = logf(__ldg(theta + pids[i] + x));
    values[(int64_t)slots[i] * ldb + b] = v;
  }
}

// Staged inputs (one CTA per block of <= 128 inputs on one variable): the
// block's pmfs are read once, coalesced, as log-pmfs into shared memory; every
// sample then reads its category's log-probability from smem and the values
// rows are written coalesced along the batch.  Replaces 4-byte gathers that
// each pull a 32-byte sector of a pmf table far larger than L2.
constexpr int IN_THREADS = 512;
constexpr int SP_THREADS = 1024;  // shared-pmf input kernels
#ifndef PCB_SP_UNROLL
#define PCB_SP_UNROLL 16
#endif
#ifndef PCB_SP_ITEMS
#define PCB_SP_ITEMS 8
#endif
constexpr int SP_UNROLL = PCB_SP_UNROLL;  // row loads in flight per thread
constexpr int SP_ITEMS = PCB_SP_ITEMS;    // (input, sample) loads in flight per thread

#ifndef PCB_IN_PREFETCH
#define PCB_IN_PREFETCH 1
#endif
// TMA L2 prefetch of floats [p, p + n) (16-byte-aligned body only)
__device__ __forceinline__ void l2_prefetch(const float* p, int64_t n) {
  const uintptr_t a = (reinterpret_cast<uintptr_t>(p) + 15) & ~(uintptr_t)15;
  const uintptr_t e = reinterpret_cast<uintptr_t>(p + n) & ~(uintptr_t)15;
  for (uintptr_t o = a; o < e; o += 16384) {
    const uint32_t bytes = (uint32_t)(e - o < 16384 ? e - o : 16384);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(o), "r"(bytes) : "memory");
  }
}

__global__ void __launch_bounds__(IN_THREADS)
    k_input_fwd_block(int B, int ldb, const int32_t* __restrict__ bvar,
                      const int32_t* __restrict__ bncat, const int32_t* __restrict__ bslot0,
                      const int32_t* __restrict__ bcount, const int32_t* __restrict__ bpoff,
                      const int32_t* __restrict__ pids, const int32_t* __restrict__ xT,
                      const float* __restrict__ theta, float* __restrict__ values,
                      const int32_t* __restrict__ arow, const int32_t* __restrict__ adir,
                      float* __restrict__ ascratch, float* __restrict__ abmax, int kn) {
  pdl_enter();
  extern __shared__ float tbl[];
  const int blk = blockIdx.x;
  const int ncat = bncat[blk], cnt = bcount[blk], var = bvar[blk];
  const int64_t slot0 = bslot0[blk];
  const int32_t* pid = pids + bpoff[blk];
  const int total = cnt * ncat;
#if PCB_IN_PREFETCH
  // every pmf row of the block into L2 at once (TMA), ahead of the staging
  // loads below, which then hit L2
  for (int i = threadIdx.x; i < cnt; i += IN_THREADS) l2_prefetch(theta + __ldg(pid + i), ncat);
#endif
  // stage log-pmfs: a warp per input row, float4 loads when the pmf is
  // 16-byte aligned (4 rows in flight per warp), else scalar loads
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = IN_THREADS / 32;
  if ((ncat & 3) == 0) {
    for (int i0 = warp; i0 < cnt; i0 += NW * 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * NW;
        if (i >= cnt) continue;
        const float* src = theta + __ldg(pid + i);
        float* dst = tbl + i * ncat;
        const bool al = (reinterpret_cast<uintptr_t>(src) & 15) == 0;
        for (int c = lane * 4; c < ncat; c += 128) {
          float4 v = al ? __ldg(reinterpret_cast<const float4*>(src + c))
                        : make_float4(__ldg(src + c), __ldg(src + c + 1), __ldg(src + c + 2),
                                      __ldg(src + c + 3));
          dst[c] = __logf(v.x);
          dst[c + 1] = __logf(v.y);
          dst[c + 2] = __logf(v.z);
          dst[c + 3] = __logf(v.w);
        }
      }
    }
  } else {
    for (int q0 = threadIdx.x; q0 < total; q0 += 4 * IN_THREADS) {
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + u * IN_THREADS;
        v[u] = (q < total) ? __ldg(theta + pid[q / ncat] + (q % ncat)) : 1.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + u * IN_THREADS;
        if (q < total) tbl[q] = __logf(v[u]);
      }
    }
  }
  __syncthreads();
  const int r0 = arow ? __ldg(arow + blk) : -1;
  if (r0 >= 0) {
    // leaf alias (lean step): the inputs' log values are the product rows of
    // the first layer's window (row r0 + dir * i); whole product blocks, so
    // the block bases (floor of the block maximum) are formed here and the
    // rows hold offsets from them
    const int64_t step = (int64_t)__ldg(adir + blk) * ldb;
    for (int b = threadIdx.x; b < B; b += IN_THREADS) {
      const int x = xT[(int64_t)var * ldb + b];
      const float* t = tbl + (x < 0 ? 0 : x);
      float* dst = ascratch + (int64_t)r0 * ldb + b;
      for (int i0 = 0; i0 < cnt; i0 += kn) {
        float mx = PCB_NEG_INF;
#pragma unroll 8
        for (int i = i0; i < i0 + kn; ++i) mx = fmaxf(mx, x < 0 ? 0.f : t[i * ncat]);
        const float base = floorf(mx);  // -inf stays -inf
        const bool dead = mx == PCB_NEG_INF;
#pragma unroll 8
        for (int i = i0; i < i0 + kn; ++i)
          dst[i * step] = dead ? PCB_NEG_INF : (x < 0 ? 0.f : t[i * ncat]) - base;
        abmax[(int64_t)((r0 + (step > 0 ? i0 : -i0)) / kn) * ldb + b] = base;
      }
    }
    return;
  }
  for (int b = threadIdx.x; b < B; b += IN_THREADS) {
    const int x = xT[(int64_t)var * ldb + b];
    float* dst = values + slot0 * ldb + b;
    if (x < 0) {
      for (int i = 0; i < cnt; ++i) dst[(int64_t)i * ldb] = 0.f;
    } else {
#pragma unroll 8
      for (int i = 0; i < cnt; ++i) dst[(int64_t)i * ldb] = tbl[i * ncat + x];
    }
  }
}

// Shared pmfs (plan.shared_pmf_table): one CTA per pmf stages its log-pmf in
// shared memory once and serves every (input, sample) of the inputs that use
// it from there -- instead of one random 32-byte-sector gather of the pmf
// table per (input, sample).  The row (up to 201 KB for HMM emissions) comes
// in by 1-D TMA bulk copies from its 16-byte-aligned start (the ragged tail
// by plain loads), so the whole row is in flight at once rather than a few
// loads per thread; the logs are then taken in place.
#ifndef PCB_SP_FWD_BULK
#define PCB_SP_FWD_BULK 1
#endif
constexpr int SP_BULK_CHUNK = 16384;  // bytes per bulk copy / L2 prefetch
#ifndef PCB_SP_FLOW_PREFETCH
#define PCB_SP_FLOW_PREFETCH 1
#endif
#ifndef PCB_SP_NEXT
#define PCB_SP_NEXT 1
#endif
// L2 prefetch (TMA) of the 16-byte-aligned body of floats [p0, p1)
__device__ __forceinline__ void l2_prefetch_row(const float* base, int64_t p0, int64_t p1) {
  const int64_t a0 = (p0 + 3) & ~(int64_t)3, a1 = p1 & ~(int64_t)3;
  for (int64_t o = a0; o < a1; o += SP_BULK_CHUNK / 4) {
    const uint32_t bytes = (uint32_t)(min((int64_t)SP_BULK_CHUNK / 4, a1 - o) * 4);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + o), "r"(bytes)
                 : "memory");
  }
}

__global__ void __launch_bounds__(SP_THREADS)
    k_input_fwd_shared(int ncat, int B, int ldb, const int32_t* __restrict__ u_pid,
                       const int32_t* __restrict__ u_off, const int32_t* __restrict__ u_slot,
                       const int32_t* __restrict__ u_var, const int32_t* __restrict__ xT,
                       const float* __restrict__ theta, float* __restrict__ values,
                       int n_u, int nsm) {
  pdl_enter();
  extern __shared__ __align__(16) float tbl_raw[];
  const int u = blockIdx.x, tid = threadIdx.x;
  const int64_t pid = __ldg(u_pid + u);
#if PCB_SP_FWD_BULK
  __shared__ __align__(8) uint64_t mbar;
  const int64_t a0 = pid & ~(int64_t)3, end = pid + ncat;
  const int64_t a1 = end & ~(int64_t)3;  // the body [a0, a1) by TMA
  const int lead = (int)(pid - a0);
  float* tbl = tbl_raw + lead;           // tbl[c] = pmf entry c
  const uint32_t mb = tc::smem_u32(&mbar);
  if (tid == 0) {
    tc::mbar_init(mb, 1);
    tc::fence_mbar_init();
    const uint32_t body = (uint32_t)((a1 - a0) * 4);
    tc::mbar_arrive_expect_tx(mb, body);
    for (uint32_t off = 0; off < body; off += SP_BULK_CHUNK)
      tc::bulk_g2s(tc::smem_u32(tbl_raw) + off, theta + a0 + off / 4, min(SP_BULK_CHUNK, (int)(body - off)),
               mb);
#if PCB_SP_NEXT
    // the row of the CTA that takes this SM next, into L2 under this one's work
    if (u + nsm < n_u) {
      const int64_t nx = __ldg(u_pid + u + nsm);
      l2_prefetch_row(theta, nx, nx + ncat);
    }
#endif
  }
  for (int64_t c = (a1 > pid ? a1 : pid) + tid; c < end; c += SP_THREADS)
    tbl_raw[c - a0] = __ldg(theta + c);
  __syncthreads();  // mbarrier initialised, tail stored
  tc::mbar_wait(mb, 0);
  for (int c = tid; c < ncat; c += SP_THREADS) tbl[c] = __logf(tbl[c]);
#else
  float* tbl = tbl_raw;
  const float* th = theta + pid;
  for (int c = tid; c < ncat; c += SP_THREADS) tbl[c] = __logf(__ldg(th + c));
#endif
  __syncthreads();
  const int e0 = __ldg(u_off + u), e1 = __ldg(u_off + u + 1);
  const int n_items = (e1 - e0) * B;
  // branch-free batches (indices clamped to the last item) so every item's
  // loads issue before the first one is used
  for (int t0 = tid; t0 < n_items; t0 += SP_ITEMS * SP_THREADS) {
    int x[SP_ITEMS];
    int64_t o[SP_ITEMS];
#pragma unroll
    for (int k = 0; k < SP_ITEMS; ++k) {
      const int t = min(t0 + k * SP_THREADS, n_items - 1);
      const int e = e0 + t / B, b = t - (t / B) * B;
      o[k] = (int64_t)__ldg(u_slot + e) * ldb + b;
      x[k] = __ldg(xT + (int64_t)__ldg(u_var + e) * ldb + b);
    }
#pragma unroll
    for (int k = 0; k < SP_ITEMS; ++k)
      if (t0 + k * SP_THREADS < n_items) values[o[k]] = x[k] < 0 ? 0.f : tbl[x[k]];
  }
}

int launch_input_fwd(const pcb_plan* p, cudaStream_t s, int B, int ldb, const int32_t* xT,
                     const float* theta, float* values, float* scratch_all, float* pbase_all,
                     bool alias) {
  ProfScope prof_(KC_INPUT_FWD, s);
  const InBlocks& ib = p->in_blocks;
  if (ib.n) {
    const int bytes = (int)ib.max_elems * 4;
    static int attr[kMaxDev] = {};
    if (ensure_smem((const void*)k_input_fwd_block, bytes, attr)) return PCB_CUDA;
    alias = alias && p->leaf_alias;
    const Layer* L0 = alias ? &p->layers[0] : nullptr;
    launch_k(k_input_fwd_block, dim3((unsigned)ib.n), dim3(IN_THREADS), bytes, s, 
        B, ldb, ib.var, ib.ncat, ib.slot0, ib.count, ib.pid_off, ib.pids, xT, theta, values,
        alias ? ib.alias_row : nullptr, ib.alias_dir,
        alias ? scratch_all + L0->scratch_off * (int64_t)ldb : nullptr,
        alias ? pbase_all + L0->pb_off * (int64_t)ldb : nullptr,
        alias ? (int)L0->k_n : 1);
    if (check_launch()) return PCB_CUDA;
  }
  for (auto& c : p->inputs) {
    int64_t total = c.n * B;
    if (!total) continue;
    if (c.n_u) {
      const int bytes = (int)(c.ncat + 4) * 4;  // + the aligned row start's lead
      static int attr_sp[kMaxDev] = {};
      if (ensure_smem((const void*)k_input_fwd_shared, bytes, attr_sp)) return PCB_CUDA;
      launch_k(k_input_fwd_shared, dim3((unsigned)c.n_u), dim3(SP_THREADS), bytes, s, 
          (int)c.ncat, B, ldb, c.u_pid, c.u_off, c.u_slot, c.u_var, xT, theta, values,
          (int)c.n_u, sm_count());
      if (check_launch()) return PCB_CUDA;
      continue;
    }
    launch_k(k_input_fwd, dim3(grid_for(total, 256)), dim3(256), 0, s, c.n, B, ldb, c.slots, c.vars, c.pids, xT,
                                                      theta, values);
    if (check_launch()) return PCB_CUDA;
  }
  return PCB_OK;
}

// ---------------------------------------------------------------- K2 products
__global__ void k_fill_rows(int64_t n, int B, int ldb, const int32_t* __restrict__ rows,
                            float* __restrict__ buf, float v) {
  pdl_enter();
  int64_t total = n * (int64_t)B;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = t / B;
    int b = (int)(t - j * B);
    buf[(int64_t)rows[j] * ldb + b] = v;
  }
}

int launch_fill(cudaStream_t s, const int32_t* rows, int64_t n, int B, int ldb, float* buf,
                float v) {
  if (!n) return PCB_OK;
  launch_k(k_fill_rows, dim3(grid_for(n * B, 256)), dim3(256), 0, s, n, B, ldb, rows, buf, v);
  return check_launch();
}

__global__ void k_fill_range(int64_t row0, int64_t n, int B, int ldb, float* __restrict__ buf,
                             float v) {
  pdl_enter();
  int64_t total = n * (int64_t)B;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = t / B;
    int b = (int)(t - j * B);
    buf[(row0 + j) * ldb + b] = v;
  }
}

// zero rows [start_r, start_r + len_r) of a [rows x ldb] buffer for every range r
__global__ void k_zero_ranges(int64_t n, const int32_t* __restrict__ start,
                              const int32_t* __restrict__ len, int ldb, float* __restrict__ buf) {
  pdl_enter();
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t r = blockIdx.x; r < n; r += gridDim.x) {
    float4* p = reinterpret_cast<float4*>(buf + (int64_t)__ldg(start + r) * ldb);
    const int64_t total = (int64_t)__ldg(len + r) * ldb / 4;
    for (int64_t q = threadIdx.x; q < total; q += blockDim.x) p[q] = z;
  }
}

int launch_zero_ranges(cudaStream_t s, int64_t n, const int32_t* start, const int32_t* len,
                       int ldb, float* buf) {
  if (!n) return PCB_OK;
  launch_k(k_zero_ranges, dim3(grid_for(n, 1, 148 * 16)), dim3(256), 0, s, n, start, len, ldb, buf);
  return check_launch();
}

int launch_fill_range(cudaStream_t s, int64_t row0, int64_t n, int B, int ldb, float* buf,
                      float v) {
  ProfScope prof_(KC_MISC, s);
  if (!n || !B) return PCB_OK;
  launch_k(k_fill_range, dim3(grid_for(n * B, 256)), dim3(256), 0, s, row0, n, B, ldb, buf, v);
  return check_launch();
}

// One CTA per (product block, 128-sample slab): 8 warps stride over the
// block's scratch rows, lane = 4 consecutive samples (float4).  A product's
// log value is the sum of its children's (engine.py:68-71): the integer
// bases add exactly (beta), the offsets in fp32 (o).  The block base is
// floor(max_j beta_j + o_j) (reduced across warps in shared memory; it is
// also the shift the sum contraction needs, so no max pre-pass), and the
// rows store (beta_j - base) + o_j.  -inf rows: window padding.
constexpr int VB = 4;              // samples per lane (float4)
constexpr int SLAB = 32 * VB;      // samples per CTA
constexpr int RW = 8;              // warps per CTA (rows in flight)
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float4 f4max(float4 a, float4 b) {
  return make_float4(fmaxf(a.x, b.x), fmaxf(a.y, b.y), fmaxf(a.z, b.z), fmaxf(a.w, b.w));
}

__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

// max over the RW warps' float4 partials, broadcast to every warp
__device__ __forceinline__ float4 block_max_all(float4 mx) {
  __shared__ float4 red[RW][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  red[warp][lane] = mx;
  __syncthreads();
#pragma unroll
  for (int w = 0; w < RW; ++w) mx = f4max(mx, red[w][lane]);
  return mx;
}

__device__ __forceinline__ float rebase(float beta, float o, float base) {
  return base == PCB_NEG_INF ? PCB_NEG_INF : (beta - base) + o;
}

// UNI: every row of a block takes its children's bases from row 0's base
// rows (plan.prod_blocks_uniform), so the summed base is formed once per
// sample and only the offsets stay in registers.
// 4 resident CTAs per SM (64 registers): 5 / 6 spill the gathered rows
// (HCLT-256 products 0.87 -> 0.97 / 1.25 ms)
#ifndef PCB_PB_MINB
#define PCB_PB_MINB 4
#endif
template <int PER, bool UNI>
__global__ void __launch_bounds__(RW * 32, (UNI && PER == 4) ? PCB_PB_MINB : 2)
    k_prod_block(int k_n, int B, int ldb, const int32_t* __restrict__ row_off,
                 const int32_t* __restrict__ ch, const int32_t* __restrict__ cb,
                 const float* __restrict__ values, const float* __restrict__ vbase,
                 float* __restrict__ scratch, float* __restrict__ pbase) {
  pdl_enter();
  const int blk = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = blockIdx.y * SLAB + lane * VB;
  const bool live = b < B;
  const float ninf = PCB_NEG_INF;
  float4 mx = make_float4(ninf, ninf, ninf, ninf);
  float4 be[UNI ? 1 : PER], of[PER];
  if (UNI) {
    // rows share one fan-in (row 0's): slot by slot, every row's child index
    // and value loads are issued together (PER independent gathers)
    be[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    int ra[PER];
    bool rl[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int j = warp + u * RW;
      const int r = blk * k_n + j;
      rl[u] = live && j < k_n && __ldg(row_off + r) < __ldg(row_off + r + 1);
      ra[u] = (j < k_n) ? __ldg(row_off + r) : 0;
      of[u] = rl[u] ? make_float4(0.f, 0.f, 0.f, 0.f) : make_float4(ninf, ninf, ninf, ninf);
    }
    const int a0 = __ldg(row_off + blk * k_n), f = __ldg(row_off + blk * k_n + 1) - a0;
    for (int q = 0; q < f; ++q) {
      int idx[PER];
#pragma unroll
      for (int u = 0; u < PER; ++u) idx[u] = rl[u] ? __ldg(ch + ra[u] + q) : 0;
      const int c = live ? __ldg(cb + a0 + q) : -1;
      float4 v[PER];
#pragma unroll
      for (int u = 0; u < PER; ++u)
        if (rl[u]) v[u] = *reinterpret_cast<const float4*>(values + (int64_t)idx[u] * ldb + b);
      if (c >= 0) be[0] = f4add(be[0], *reinterpret_cast<const float4*>(vbase + (int64_t)c * ldb + b));
#pragma unroll
      for (int u = 0; u < PER; ++u)
        if (rl[u]) of[u] = f4add(of[u], v[u]);
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) mx = f4max(mx, of[u]);
  } else {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int j = warp + u * RW;
      be[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      of[u] = make_float4(ninf, ninf, ninf, ninf);
      if (j >= k_n || !live) continue;
      const int r = blk * k_n + j;
      const int a = __ldg(row_off + r), z = __ldg(row_off + r + 1);
      if (a < z) {
        of[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int q = a; q < z; ++q) {
          of[u] = f4add(of[u], *reinterpret_cast<const float4*>(values + (int64_t)__ldg(ch + q) * ldb + b));
          const int c = __ldg(cb + q);
          if (c >= 0) be[u] = f4add(be[u], *reinterpret_cast<const float4*>(vbase + (int64_t)c * ldb + b));
        }
      }
      mx = f4max(mx, f4add(be[u], of[u]));
    }
  }
  mx = block_max_all(mx);
  if (!live) return;
  if (UNI) mx = f4add(mx, be[0]);
  const float4 base = make_float4(floorf(mx.x), floorf(mx.y), floorf(mx.z), floorf(mx.w));
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int j = warp + u * RW;
    if (j >= k_n) continue;
    const float4 e = be[UNI ? 0 : u];
    const float4 o = make_float4(rebase(e.x, of[u].x, base.x), rebase(e.y, of[u].y, base.y),
                                 rebase(e.z, of[u].z, base.z), rebase(e.w, of[u].w, base.w));
    *reinterpret_cast<float4*>(scratch + (int64_t)(blk * k_n + j) * ldb + b) = o;
  }
  if (warp == 0) *reinterpret_cast<float4*>(pbase + (int64_t)blk * ldb + b) = base;
}

int launch_prod_eval(const Layer& L, cudaStream_t s, int B, int ldb, const float* values,
                     const float* vbase_all, float* scratch, float* pbase) {
  ProfScope prof_(KC_PROD_EVAL, s);
  if (!B || !L.n_pb) return PCB_OK;
  dim3 grid((unsigned)L.n_pb, (unsigned)((B + SLAB - 1) / SLAB));
#define PCB_PB(PER)                                                                          \
  (L.prod_uniform                                                                            \
       ? launch_k((k_prod_block<PER, true>), dim3(grid), dim3(RW * 32), 0, s, (int)L.k_n, B, ldb, L.prow_off,    \
                                                          L.prow_ch, L.prow_cb, values,     \
                                                          vbase_all, scratch, pbase)        \
       : launch_k((k_prod_block<PER, false>), dim3(grid), dim3(RW * 32), 0, s, (int)L.k_n, B, ldb, L.prow_off,   \
                                                           L.prow_ch, L.prow_cb, values,    \
                                                           vbase_all, scratch, pbase))
  if (L.k_n <= RW) PCB_PB(1);
  else if (L.k_n <= 2 * RW) PCB_PB(2);
  else if (L.k_n <= 4 * RW) PCB_PB(4);
  else if (L.k_n <= 8 * RW) PCB_PB(8);
  else return PCB_USAGE;
#undef PCB_PB
  return check_launch();
}

// Flow ratios of one sum block (engine.py:114-117), in log2 units:
//   R[sb, b]  = max over the block's sums of lg2(flow) - value * log2(e)
//               (-inf when every sum is impossible or flowless): the shift;
//   r[m, b]   = lg2(flow_m) - fma(value_m, log2 e, R)  (<= 0; -inf for
//               impossible / zero-flow sums), r rows indexed from sb_base.
// The shift only has to be applied consistently: every product of a large
// log value with log2(e) is fused with the subtraction of R, so r keeps full
// precision even at |log p| ~ 1e4.  The tensor-core flow kernels read r (one
// row per sum instead of flows + values) and R.
constexpr int KM_MAX = 64;
__global__ void __launch_bounds__(RW * 32, 5)
    k_ratio(int k_m, int B, int ldb, int64_t sb_base, const float* __restrict__ values,
            const float* __restrict__ flows, float* __restrict__ rmax, float* __restrict__ ratio) {
  pdl_enter();
  constexpr int PER = KM_MAX / RW;
  const int blk = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = blockIdx.y * SLAB + lane * VB;
  const bool live = b < B;
  const float ninf = PCB_NEG_INF;
  float4 t[PER];
  float4 mx = make_float4(ninf, ninf, ninf, ninf);
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int m = warp + u * RW;
    t[u] = make_float4(ninf, ninf, ninf, ninf);
    if (live && m < k_m) {
      const int64_t o = (sb_base + (int64_t)blk * k_m + m) * ldb + b;
      const float4 f = *reinterpret_cast<const float4*>(flows + o);
      const float4 l = *reinterpret_cast<const float4*>(values + o);
      // t = lg2 f, with l folded in only for the (imprecise) max
      t[u].x = (l.x == ninf || !(f.x > 0.f)) ? ninf : __log2f(f.x);
      t[u].y = (l.y == ninf || !(f.y > 0.f)) ? ninf : __log2f(f.y);
      t[u].z = (l.z == ninf || !(f.z > 0.f)) ? ninf : __log2f(f.z);
      t[u].w = (l.w == ninf || !(f.w > 0.f)) ? ninf : __log2f(f.w);
      if (t[u].x != ninf) mx.x = fmaxf(mx.x, t[u].x - l.x * kLog2e);
      if (t[u].y != ninf) mx.y = fmaxf(mx.y, t[u].y - l.y * kLog2e);
      if (t[u].z != ninf) mx.z = fmaxf(mx.z, t[u].z - l.z * kLog2e);
      if (t[u].w != ninf) mx.w = fmaxf(mx.w, t[u].w - l.w * kLog2e);
    }
  }
  __shared__ float4 red[RW][32];
  red[warp][lane] = mx;
  __syncthreads();
#pragma unroll
  for (int w = 0; w < RW; ++w) mx = f4max(mx, red[w][lane]);
  if (!live) return;
  if (warp == 0) *reinterpret_cast<float4*>(rmax + (int64_t)blk * ldb + b) = mx;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int m = warp + u * RW;
    if (m < k_m) {
      const int64_t row = (int64_t)blk * k_m + m;
      const float4 l = *reinterpret_cast<const float4*>(values + (sb_base + row) * ldb + b);
      float4 r;
      r.x = (t[u].x == ninf) ? ninf : t[u].x - fmaf(l.x, kLog2e, mx.x);
      r.y = (t[u].y == ninf) ? ninf : t[u].y - fmaf(l.y, kLog2e, mx.y);
      r.z = (t[u].z == ninf) ? ninf : t[u].z - fmaf(l.z, kLog2e, mx.z);
      r.w = (t[u].w == ninf) ? ninf : t[u].w - fmaf(l.w, kLog2e, mx.w);
      *reinterpret_cast<float4*>(ratio + row * ldb + b) = r;
    }
  }
}

int launch_ratio_max(const Layer& L, cudaStream_t s, int B, int ldb, const float* values,
                     const float* flows, float* rmax, float* ratio) {
  ProfScope prof_(KC_PARAM_FLOW, s);
  if (!B || !L.n_sb) return PCB_OK;
  if (L.k_m > KM_MAX) return PCB_USAGE;
  dim3 grid((unsigned)L.n_sb, (unsigned)((B + SLAB - 1) / SLAB));
  launch_k(k_ratio, dim3(grid), dim3(RW * 32), 0, s, (int)L.k_m, B, ldb, L.sb_base, values, flows, rmax, ratio);
  return check_launch();
}

// Fused flow push + flow ratio (lean steps): one CTA per (fan-in slot of a
// push block of K products, 128-sample slab).  The slot's K children are
// consecutive single-push slots: either plain flow stores of the block's K
// product flows, or one whole sum block of a pre-ratioed layer, whose ratio
// rows r (k_ratio's arithmetic, bit for bit) overwrite the flow rows and
// whose shift R goes to its rmax_all row.  Replaces the push's flow stores
// plus the ratio pass's re-read of flows and values.  The block's product
// flows are read once per slot (the slots of a block are adjacent CTAs: L2).
// 6 resident CTAs per SM (40 registers, a small spill): each CTA's life is
// ~3 dependent latency rounds for 48 KB, so residency sets the bandwidth
// (HCLT-256: 1.31 ms at 4 CTAs / SM -> 1.05 ms; 5: 1.23, 7 / 8: 1.53)
#ifndef PCB_PR_MINB
#define PCB_PR_MINB 6
#endif
template <int K>
__global__ void __launch_bounds__(RW * 32, PCB_PR_MINB)
    k_push_ratio(int B, int ldb, const int32_t* __restrict__ qblk,
                 const int32_t* __restrict__ prow, const int32_t* __restrict__ qbase,
                 const int32_t* __restrict__ qkind, const int32_t* __restrict__ qrrow,
                 const float* __restrict__ fs, const float* __restrict__ values,
                 float* __restrict__ flows, float* __restrict__ rmax_all) {
  pdl_enter();
  constexpr int PER = (K + RW - 1) / RW;
  const int q = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = blockIdx.y * SLAB + lane * VB;
  const bool live = b < B;
  const float ninf = PCB_NEG_INF;
  const int64_t r0 = __ldg(prow + __ldg(qblk + q)), cb = __ldg(qbase + q);
  const bool ratio = __ldg(qkind + q) != 0;
  float4 p[PER], l[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int m = warp + u * RW;
    p[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    l[u] = make_float4(ninf, ninf, ninf, ninf);
    if (live && m < K) {
      p[u] = *reinterpret_cast<const float4*>(fs + (r0 + m) * ldb + b);
      if (ratio) l[u] = *reinterpret_cast<const float4*>(values + (cb + m) * ldb + b);
    }
  }
  if (!ratio) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int m = warp + u * RW;
      if (live && m < K) *reinterpret_cast<float4*>(flows + (cb + m) * ldb + b) = p[u];
    }
    return;
  }
  float4 mx = make_float4(ninf, ninf, ninf, ninf);
#pragma unroll
  for (int u = 0; u < PER; ++u) {  // p <- lg2 f (k_ratio's t)
    p[u].x = (l[u].x == ninf || !(p[u].x > 0.f)) ? ninf : __log2f(p[u].x);
    p[u].y = (l[u].y == ninf || !(p[u].y > 0.f)) ? ninf : __log2f(p[u].y);
    p[u].z = (l[u].z == ninf || !(p[u].z > 0.f)) ? ninf : __log2f(p[u].z);
    p[u].w = (l[u].w == ninf || !(p[u].w > 0.f)) ? ninf : __log2f(p[u].w);
    if (p[u].x != ninf) mx.x = fmaxf(mx.x, p[u].x - l[u].x * kLog2e);
    if (p[u].y != ninf) mx.y = fmaxf(mx.y, p[u].y - l[u].y * kLog2e);
    if (p[u].z != ninf) mx.z = fmaxf(mx.z, p[u].z - l[u].z * kLog2e);
    if (p[u].w != ninf) mx.w = fmaxf(mx.w, p[u].w - l[u].w * kLog2e);
  }
  __shared__ float4 red[RW][32];
  red[warp][lane] = mx;
  __syncthreads();
#pragma unroll
  for (int w = 0; w < RW; ++w) mx = f4max(mx, red[w][lane]);
  if (!live) return;
  if (warp == 0) *reinterpret_cast<float4*>(rmax_all + (int64_t)__ldg(qrrow + q) * ldb + b) = mx;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int m = warp + u * RW;
    if (m < K) {
      float4 r;
      r.x = (p[u].x == ninf) ? ninf : p[u].x - fmaf(l[u].x, kLog2e, mx.x);
      r.y = (p[u].y == ninf) ? ninf : p[u].y - fmaf(l[u].y, kLog2e, mx.y);
      r.z = (p[u].z == ninf) ? ninf : p[u].z - fmaf(l[u].z, kLog2e, mx.z);
      r.w = (p[u].w == ninf) ? ninf : p[u].w - fmaf(l[u].w, kLog2e, mx.w);
      *reinterpret_cast<float4*>(flows + (cb + m) * ldb + b) = r;
    }
  }
}

int launch_push_ratio(const Layer& L, cudaStream_t s, int B, int ldb, const float* flow_scratch,
                      const float* values, float* flows, float* rmax_all) {
  ProfScope prof_(KC_ACCUM_PUSH, s);
  if (!B || !L.n_pq) return PCB_OK;
  dim3 grid((unsigned)L.n_pq, (unsigned)((B + SLAB - 1) / SLAB));
#define PCB_PR(K)                                                                              \
  launch_k((k_push_ratio<K>), dim3(grid), dim3(RW * 32), 0, s, B, ldb, L.q_blk, L.pb_row, L.q_base, L.q_kind,      \
                                           L.q_rrow, flow_scratch, values, flows, rmax_all)
  switch (L.k_n) {
    case 16: PCB_PR(16); break;
    case 32: PCB_PR(32); break;
    case 64: PCB_PR(64); break;
    default: return PCB_USAGE;
  }
#undef PCB_PR
  return check_launch();
}

// ---------------------------------------------------------------- K3 (SIMT)
// Alg. 1 for one sum-block row and a 32-sample tile (engine.py:74-102).
// block (32, 8): tx = sample, ty strides over the k_m sums of the block.
// The row's base G is the max of its real child blocks' bases; child values
// enter as offset + (base - G) (an exact integer difference), the streaming
// (lin, top) merge runs on those, and the outputs are offsets from G.
constexpr int TB = 32;
constexpr int TY = 8;
constexpr int KMAX = 64;

__global__ void __launch_bounds__(TB* TY)
    k_sum_fwd_simt(int cap, int k_m, int k_n, int B, int ldb, int64_t sb_base,
                   const int32_t* __restrict__ sum_ids, const int32_t* __restrict__ prod_ids,
                   const int32_t* __restrict__ param_ids, const float* __restrict__ theta,
                   const float* __restrict__ scratch, const float* __restrict__ pbase,
                   float* __restrict__ values, float* __restrict__ vbase) {
  pdl_enter();
  __shared__ float ex[KMAX][TB];
  __shared__ float th[KMAX * KMAX];
  __shared__ float cm[TB];
  const int r = blockIdx.y;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * TB + tx;
  const int b = blockIdx.x * TB + tx;
  const bool live_b = b < B;
  float G = PCB_NEG_INF;
  if (live_b)
    for (int c = 0; c < cap; ++c)
      if (param_ids[(int64_t)r * cap + c] != 0)
        G = fmaxf(G, pbase[(int64_t)(prod_ids[(int64_t)r * cap + c] / k_n) * ldb + b]);
  if (G == PCB_NEG_INF) G = 0.f;  // every child block -inf: the offsets say so
  float lin[KMAX / TY];
#pragma unroll
  for (int i = 0; i < KMAX / TY; ++i) lin[i] = 0.f;
  float top = PCB_NEG_INF;
  for (int c = 0; c < cap; ++c) {
    const int pid = prod_ids[(int64_t)r * cap + c];
    const int tid0 = param_ids[(int64_t)r * cap + c];
    if (tid0 == 0) continue;  // padded column: -inf child block, zero tile
    const float d = live_b ? pbase[(int64_t)(pid / k_n) * ldb + b] - G : PCB_NEG_INF;
    for (int j = ty; j < k_n; j += TY)
      ex[j][tx] = live_b ? scratch[(int64_t)(pid + j) * ldb + b] + d : PCB_NEG_INF;
    for (int q = tid; q < k_m * k_n; q += TB * TY) th[q] = __ldg(theta + tid0 + q);
    __syncthreads();
    if (ty == 0) {
      float m = PCB_NEG_INF;
      for (int j = 0; j < k_n; ++j) m = fmaxf(m, ex[j][tx]);
      cm[tx] = m;
    }
    __syncthreads();
    const float cmax = cm[tx];
    const bool dead = (cmax == PCB_NEG_INF);
    for (int j = ty; j < k_n; j += TY) ex[j][tx] = dead ? 0.f : expf(ex[j][tx] - cmax);
    __syncthreads();
    if (!dead) {
      const float s_old = (cmax > top) ? expf(top - cmax) : 1.f;
      const float s_new = (cmax > top) ? 1.f : expf(cmax - top);
#pragma unroll
      for (int i = 0; i < KMAX / TY; ++i) {
        const int m = ty + i * TY;
        if (m < k_m) {
          float part = 0.f;
          for (int j = 0; j < k_n; ++j) part = fmaf(th[m * k_n + j], ex[j][tx], part);
          lin[i] = lin[i] * s_old + part * s_new;
        }
      }
      top = fmaxf(top, cmax);
    }
    __syncthreads();
  }
  if (!live_b) return;
  const int sid = sum_ids[r];
#pragma unroll
  for (int i = 0; i < KMAX / TY; ++i) {
    const int m = ty + i * TY;
    if (m < k_m) values[(int64_t)(sid + m) * ldb + b] = logf(lin[i]) + top;
  }
  if (ty == 0) vbase[(int64_t)((sid - sb_base) / k_m) * ldb + b] = G;
}

// Single-sum rows (k_m = 1, e.g. an HMM or mixture root over thousands of
// children): TY1 thread rows split the child blocks (each its own
// streaming (lin, top) pair, merged in shared memory at the end) instead of
// one thread row walking all of them; 32 rows: a 128-block root (HMM-4096)
// is 4 blocks per thread.
constexpr int TY1 = 32;
__global__ void __launch_bounds__(TB* TY1)
    k_sum_fwd_simt1(int cap, int k_n, int B, int ldb, int64_t sb_base,
                    const int32_t* __restrict__ sum_ids, const int32_t* __restrict__ prod_ids,
                    const int32_t* __restrict__ param_ids, const float* __restrict__ theta,
                    const float* __restrict__ scratch, const float* __restrict__ pbase,
                    float* __restrict__ values, float* __restrict__ vbase) {
  pdl_enter();
  __shared__ float lin_s[TY1][TB], top_s[TY1][TB], g_s[TY1][TB];
  const int r = blockIdx.y;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int b = blockIdx.x * TB + tx;
  const bool live = b < B;
  const int32_t* prow = prod_ids + (int64_t)r * cap;
  const int32_t* trow = param_ids + (int64_t)r * cap;
  float G = PCB_NEG_INF;
  if (live)
    for (int c = ty; c < cap; c += TY1)
      if (trow[c] != 0) G = fmaxf(G, pbase[(int64_t)(prow[c] / k_n) * ldb + b]);
  g_s[ty][tx] = G;
  __syncthreads();
  G = PCB_NEG_INF;
#pragma unroll
  for (int y = 0; y < TY1; ++y) G = fmaxf(G, g_s[y][tx]);
  if (G == PCB_NEG_INF) G = 0.f;
  float lin = 0.f, top = PCB_NEG_INF;
  if (live)
    for (int c = ty; c < cap; c += TY1) {
      const int t0 = trow[c];
      if (t0 == 0) continue;
      const int pid = prow[c];
      const float d = pbase[(int64_t)(pid / k_n) * ldb + b] - G;
      float cmax = PCB_NEG_INF;
      for (int j = 0; j < k_n; ++j) cmax = fmaxf(cmax, scratch[(int64_t)(pid + j) * ldb + b] + d);
      if (cmax == PCB_NEG_INF) continue;
      float part = 0.f;
      for (int j = 0; j < k_n; ++j)
        part = fmaf(__ldg(theta + t0 + j), expf(scratch[(int64_t)(pid + j) * ldb + b] + d - cmax),
                    part);
      if (cmax > top) {
        lin = lin * expf(top - cmax) + part;
        top = cmax;
      } else {
        lin += part * expf(cmax - top);
      }
    }
  lin_s[ty][tx] = lin;
  top_s[ty][tx] = top;
  __syncthreads();
  if (ty != 0 || !live) return;
  float T = PCB_NEG_INF;
#pragma unroll
  for (int y = 0; y < TY1; ++y) T = fmaxf(T, top_s[y][tx]);
  float acc = 0.f;
  if (T != PCB_NEG_INF)
#pragma unroll
    for (int y = 0; y < TY1; ++y)
      if (top_s[y][tx] != PCB_NEG_INF) acc += lin_s[y][tx] * expf(top_s[y][tx] - T);
  const int sid = sum_ids[r];
  values[(int64_t)sid * ldb + b] = logf(acc) + T;
  vbase[(int64_t)(sid - sb_base) * ldb + b] = G;
}

int launch_sum_fwd_simt(const Layer& L, const FwdGroup& g, cudaStream_t s, int B, int ldb,
                        const float* theta, const float* scratch, const float* pbase,
                        float* values, float* vbase) {
  ProfScope prof_(KC_SUM_FWD_SIMT, s);
  if (!g.rows) return PCB_OK;
  if (L.k_m == 1 && g.cap >= 2) {  // thread rows split the child blocks
    dim3 grid((B + TB - 1) / TB, (unsigned)g.rows);
    launch_k(k_sum_fwd_simt1, dim3(grid), dim3(dim3(TB, TY1)), 0, s, (int)g.cap, (int)L.k_n, B, ldb, L.sb_base,
                                                  g.sum_ids, g.prod_ids, g.param_ids, theta,
                                                  scratch, pbase, values, vbase);
    return check_launch();
  }
  dim3 grid((B + TB - 1) / TB, (unsigned)g.rows);
  launch_k(k_sum_fwd_simt, dim3(grid), dim3(dim3(TB, TY)), 0, s, (int)g.cap, (int)L.k_m, (int)L.k_n, B, ldb,
                                               L.sb_base, g.sum_ids, g.prod_ids, g.param_ids,
                                               theta, scratch, pbase, values, vbase);
  return check_launch();
}

// log-flow ratio of a sum node: -inf for impossible nodes (engine.py:114-117)
__device__ __forceinline__ float log_ratio(float f, float l) {
  return (l == PCB_NEG_INF) ? PCB_NEG_INF : (logf(f) - l);
}

// ---------------------------------------------------------------- K4 (SIMT)
// Alg. 3 for one (sum-block row, child column) tile (engine.py:105-126):
// cum[m, n] = sum_b exp(lnf[m,b] - nmax[b]) * exp(child[n,b] + nmax[b]);
// f_params[flow + m*k_n + n] += theta * cum.  lnf uses the sums' offsets;
// the child side adds the exact base difference (product block - sum block).
constexpr int PF_THREADS = 256;

__global__ void __launch_bounds__(PF_THREADS)
    k_param_flow_simt(int cap, int k_m, int k_n, int B, int ldb, int64_t sb_base,
                      const int32_t* __restrict__ sum_ids, const int32_t* __restrict__ prod_ids,
                      const int32_t* __restrict__ param_ids, const int32_t* __restrict__ flow_ids,
                      const float* __restrict__ theta, const float* __restrict__ values,
                      const float* __restrict__ flows, const float* __restrict__ scratch,
                      const float* __restrict__ pbase, const float* __restrict__ vbase,
                      float* __restrict__ f_params) {
  pdl_enter();
  __shared__ float sc[KMAX][TB];
  __shared__ float em[KMAX][TB];
  __shared__ float nm[TB];
  const int r = blockIdx.y, c = blockIdx.x;
  const int tid0 = param_ids[(int64_t)r * cap + c];
  if (tid0 == 0) return;
  const int pid = prod_ids[(int64_t)r * cap + c];
  const int fid = flow_ids[(int64_t)r * cap + c];
  const int sid = sum_ids[r];
  const float* pb = pbase + (int64_t)(pid / k_n) * ldb;
  const float* vb = vbase + (int64_t)((sid - sb_base) / k_m) * ldb;
  const int tid = threadIdx.x;
  const int tx = tid % TB, ty = tid / TB;  // 32 x 8
  const int tile = k_m * k_n;
  constexpr int PER = KMAX * KMAX / PF_THREADS;
  float cum[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) cum[i] = 0.f;
  for (int b0 = 0; b0 < B; b0 += TB) {
    const int b = b0 + tx;
    const bool live = b < B;
    for (int m = ty; m < k_m; m += PF_THREADS / TB) {
      const int64_t o = (int64_t)(sid + m) * ldb + b;
      sc[m][tx] = live ? log_ratio(flows[o], values[o]) : PCB_NEG_INF;
    }
    __syncthreads();
    if (ty == 0) {
      float mx = PCB_NEG_INF;
      for (int m = 0; m < k_m; ++m) mx = fmaxf(mx, sc[m][tx]);
      nm[tx] = mx;
    }
    __syncthreads();
    const float nmax = nm[tx];
    const bool dead = (nmax == PCB_NEG_INF) || !live;
    const float d = dead ? 0.f : pb[b] - vb[b];
    for (int m = ty; m < k_m; m += PF_THREADS / TB) sc[m][tx] = dead ? 0.f : expf(sc[m][tx] - nmax);
    for (int n = ty; n < k_n; n += PF_THREADS / TB)
      em[n][tx] = dead ? 0.f : expf((scratch[(int64_t)(pid + n) * ldb + b] + d) + nmax);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int q = tid + i * PF_THREADS;
      if (q < tile) {
        const int m = q / k_n, n = q - m * k_n;
        float a = cum[i];
        for (int t = 0; t < TB; ++t) a = fmaf(sc[m][t], em[n][t], a);
        cum[i] = a;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int q = tid + i * PF_THREADS;
    if (q < tile) {
      const float th = __ldg(theta + tid0 + q);
      if (th != 0.f) atomicAdd(f_params + fid + q, th * cum[i]);
    }
  }
}

// Single-sum rows (k_m = 1, e.g. an HCLT / HMM root): the ratio shift is the
// row's own log ratio, so cum[n] = sum_b exp(child[n,b] + d_b + lr_b).  The
// eight warps take interleaved 32-sample chunks (lane = sample, coalesced
// child rows), keep k_n partial sums each, and meet in a fixed-order
// reduction (warp shuffles, then warp 0..7 in order): deterministic.
__global__ void __launch_bounds__(PF_THREADS)
    k_param_flow_simt1(int cap, int k_n, int B, int ldb, int64_t sb_base,
                       const int32_t* __restrict__ sum_ids, const int32_t* __restrict__ prod_ids,
                       const int32_t* __restrict__ param_ids, const int32_t* __restrict__ flow_ids,
                       const float* __restrict__ theta, const float* __restrict__ values,
                       const float* __restrict__ flows, const float* __restrict__ scratch,
                       const float* __restrict__ pbase, const float* __restrict__ vbase,
                       float* __restrict__ f_params) {
  pdl_enter();
  constexpr int NW = PF_THREADS / 32;
  __shared__ float red[NW][KMAX];
  const int r = blockIdx.y, c = blockIdx.x;
  const int tid0 = param_ids[(int64_t)r * cap + c];
  if (tid0 == 0) return;
  const int pid = prod_ids[(int64_t)r * cap + c];
  const int fid = flow_ids[(int64_t)r * cap + c];
  const int sid = sum_ids[r];
  const float* pb = pbase + (int64_t)(pid / k_n) * ldb;
  const float* vb = vbase + (int64_t)(sid - sb_base) * ldb;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float acc[KMAX];
#pragma unroll
  for (int n = 0; n < KMAX; ++n) acc[n] = 0.f;
  for (int b = w * 32 + lane; b < B; b += NW * 32) {
    const int64_t o = (int64_t)sid * ldb + b;
    const float lr = log_ratio(flows[o], values[o]);
    if (lr == PCB_NEG_INF) continue;
    const float e = lr + (pb[b] - vb[b]);
#pragma unroll
    for (int n = 0; n < KMAX; ++n)
      if (n < k_n) acc[n] += expf(scratch[(int64_t)(pid + n) * ldb + b] + e);
  }
#pragma unroll
  for (int n = 0; n < KMAX; ++n) {
    if (n >= k_n) break;
    float v = acc[n];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[w][n] = v;
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t < k_n) {
    float sum = 0.f;
#pragma unroll
    for (int q = 0; q < NW; ++q) sum += red[q][t];
    const float th = __ldg(theta + tid0 + t);
    if (th != 0.f) atomicAdd(f_params + fid + t, th * sum);
  }
}

int launch_param_flow_simt(const Layer& L, const FwdGroup& g, cudaStream_t s, int B, int ldb,
                           const float* theta, const float* values, const float* flows,
                           const float* scratch, const float* pbase, const float* vbase,
                           float* f_params) {
  ProfScope prof_(KC_PARAM_FLOW, s);
  if (!g.rows || !g.cap) return PCB_OK;
  dim3 grid((unsigned)g.cap, (unsigned)g.rows);
  if (L.k_m == 1) {
    launch_k(k_param_flow_simt1, dim3(grid), dim3(PF_THREADS), 0, s, (int)g.cap, (int)L.k_n, B, ldb, L.sb_base,
                                                   g.sum_ids, g.prod_ids, g.param_ids, g.flow_ids,
                                                   theta, values, flows, scratch, pbase, vbase,
                                                   f_params);
    return check_launch();
  }
  launch_k(k_param_flow_simt, dim3(grid), dim3(PF_THREADS), 0, s, (int)g.cap, (int)L.k_m, (int)L.k_n, B, ldb,
                                                L.sb_base, g.sum_ids, g.prod_ids, g.param_ids,
                                                g.flow_ids, theta, values, flows, scratch, pbase,
                                                vbase, f_params);
  return check_launch();
}

// ---------------------------------------------------------------- K5 (SIMT)
// Alg. 4 for one product-block row and a 32-sample tile (engine.py:129-165).
// Parent ratios (offsets) are moved onto the product block's base: lnf +
// (base_pb - base_sb), an exact integer difference per parent block.
__global__ void __launch_bounds__(TB* TY)
    k_child_flow_simt(int cap, int k_m, int k_n, int B, int ldb, int64_t sb_base,
                      const int32_t* __restrict__ ch_ids, const int32_t* __restrict__ par_ids,
                      const int32_t* __restrict__ ppids, const float* __restrict__ theta,
                      const float* __restrict__ values, const float* __restrict__ flows,
                      const float* __restrict__ scratch, const float* __restrict__ pbase,
                      const float* __restrict__ vbase, float* __restrict__ flow_scratch) {
  pdl_enter();
  __shared__ float sc[KMAX][TB];
  __shared__ float th[KMAX * KMAX];
  __shared__ float nm[TB];
  const int r = blockIdx.y;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * TB + tx;
  const int b = blockIdx.x * TB + tx;
  const bool live_b = b < B;
  const int ch = ch_ids[r];
  const float bp = live_b ? pbase[(int64_t)(ch / k_n) * ldb + b] : PCB_NEG_INF;
  float lin[KMAX / TY];
#pragma unroll
  for (int i = 0; i < KMAX / TY; ++i) lin[i] = 0.f;
  float top = PCB_NEG_INF;
  for (int p = 0; p < cap; ++p) {
    const int tid0 = ppids[(int64_t)r * cap + p];
    if (tid0 == 0) continue;
    const int par = par_ids[(int64_t)r * cap + p];
    const float d = (live_b && bp != PCB_NEG_INF)
                        ? bp - vbase[(int64_t)((par - sb_base) / k_m) * ldb + b]
                        : PCB_NEG_INF;
    for (int m = ty; m < k_m; m += TY) {
      const int64_t o = (int64_t)(par + m) * ldb + b;
      sc[m][tx] = live_b ? log_ratio(flows[o], values[o]) + d : PCB_NEG_INF;
    }
    for (int q = tid; q < k_m * k_n; q += TB * TY) th[q] = __ldg(theta + tid0 + q);
    __syncthreads();
    if (ty == 0) {
      float mx = PCB_NEG_INF;
      for (int m = 0; m < k_m; ++m) mx = fmaxf(mx, sc[m][tx]);
      nm[tx] = mx;
    }
    __syncthreads();
    const float nmax = nm[tx];
    const bool dead = (nmax == PCB_NEG_INF);
    for (int m = ty; m < k_m; m += TY) sc[m][tx] = dead ? 0.f : expf(sc[m][tx] - nmax);
    __syncthreads();
    if (!dead) {
      const float s_old = (nmax > top) ? expf(top - nmax) : 1.f;
      const float s_new = (nmax > top) ? 1.f : expf(nmax - top);
#pragma unroll
      for (int i = 0; i < KMAX / TY; ++i) {
        const int n = ty + i * TY;
        if (n < k_n) {
          float part = 0.f;
          for (int m = 0; m < k_m; ++m) part = fmaf(th[m * k_n + n], sc[m][tx], part);
          lin[i] = lin[i] * s_old + part * s_new;
        }
      }
      top = fmaxf(top, nmax);
    }
    __syncthreads();
  }
  if (!live_b) return;
#pragma unroll
  for (int i = 0; i < KMAX / TY; ++i) {
    const int n = ty + i * TY;
    if (n < k_n) {
      const int64_t o = (int64_t)(ch + n) * ldb + b;
      const float lp = scratch[o];
      // lin * exp(top + offset) computed in log space to avoid overflow
      flow_scratch[o] = (lin[i] > 0.f) ? expf(logf(lin[i]) + top + lp) : 0.f;
    }
  }
}

int launch_child_flow_simt(const Layer& L, const BwdGroup& g, cudaStream_t s, int B, int ldb,
                           const float* theta, const float* values, const float* flows,
                           const float* scratch, const float* pbase, const float* vbase,
                           float* flow_scratch) {
  ProfScope prof_(KC_CHILD_FLOW, s);
  if (!g.rows) return PCB_OK;
  dim3 grid((B + TB - 1) / TB, (unsigned)g.rows);
  launch_k(k_child_flow_simt, dim3(grid), dim3(dim3(TB, TY)), 0, s, (int)g.cap, (int)L.k_m, (int)L.k_n, B, ldb,
                                                  L.sb_base, g.ch_ids, g.par_ids,
                                                  g.par_param_ids, theta, values, flows, scratch,
                                                  pbase, vbase, flow_scratch);
  return check_launch();
}

// ---------------------------------------------------------------- K6
// prod_flows[row_j] += flow_scratch[slot_j] (engine.py:249-250)
__global__ void k_prod_accum(int64_t n, int B, int ldb, const int32_t* __restrict__ slots,
                             const int32_t* __restrict__ rows, const float* __restrict__ fs,
                             float* __restrict__ pf) {
  pdl_enter();
  int64_t total = n * (int64_t)B;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = t / B;
    int b = (int)(t - j * B);
    pf[(int64_t)rows[j] * ldb + b] += fs[(int64_t)slots[j] * ldb + b];
  }
}

// flows[child] += prod_flows[row] for every child of a finished product (engine.py:251-254)
__global__ void k_push(int64_t n, int f, int B, int ldb, const int32_t* __restrict__ rows,
                       const int32_t* __restrict__ ch, const float* __restrict__ pf,
                       float* __restrict__ flows) {
  pdl_enter();
  int64_t total = n * (int64_t)B;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = t / B;
    int b = (int)(t - j * B);
    float v = pf[(int64_t)rows[j] * ldb + b];
    if (v == 0.f) continue;
    const int32_t* c = ch + j * f;
    for (int q = 0; q < f; ++q) atomicAdd(flows + (int64_t)c[q] * ldb + b, v);
  }
}

// Fused (engine.py:249-254): for every product evaluated in the layer,
// prod_flows[row] += flow_scratch[slot] (a store for the row's first
// accumulation in the pass); if the layer is its pushing layer, add the
// finished row to each child's flow — a plain store for children with a
// single push in the whole pass, else a vector (float4) atomic.  One warp per
// product row, lane = 4 consecutive samples; a CTA covers RW rows x 128 samples.
__global__ void __launch_bounds__(RW * 32)
    k_flow_push(int64_t n, int B, int ldb, const int32_t* __restrict__ slots,
                const int32_t* __restrict__ rows, const int32_t* __restrict__ flag,
                const int32_t* __restrict__ poff, const int32_t* __restrict__ pch,
                const float* __restrict__ fs, float* __restrict__ pf, float* __restrict__ flows) {
  pdl_enter();
  // each warp takes PU consecutive product rows; their index loads, then
  // their flow loads, are issued together before any store
  constexpr int PU = 4;
  const int64_t j0 = ((int64_t)blockIdx.x * RW + (threadIdx.x >> 5)) * PU;
  const int b = blockIdx.y * SLAB + (threadIdx.x & 31) * VB;
  if (j0 >= n || b >= B) return;
  int fl[PU], rw[PU], sl[PU];
#pragma unroll
  for (int u = 0; u < PU; ++u) {
    const bool ok = j0 + u < n;
    fl[u] = ok ? __ldg(flag + j0 + u) : 0;
    rw[u] = ok ? __ldg(rows + j0 + u) : 0;
    sl[u] = ok ? __ldg(slots + j0 + u) : -1;
  }
  float4 p[PU];
#pragma unroll
  for (int u = 0; u < PU; ++u) {
    p[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (sl[u] >= 0) p[u] = *reinterpret_cast<const float4*>(fs + (int64_t)sl[u] * ldb + b);
    if (sl[u] >= 0 && pf && !(fl[u] & 2)) {
      const float4 o = *reinterpret_cast<const float4*>(pf + (int64_t)rw[u] * ldb + b);
      p[u].x += o.x;
      p[u].y += o.y;
      p[u].z += o.z;
      p[u].w += o.w;
    }
  }
  const bool full = b + VB <= B;
#pragma unroll
  for (int u = 0; u < PU; ++u) {
    if (sl[u] < 0) continue;
    if (pf) *reinterpret_cast<float4*>(pf + (int64_t)rw[u] * ldb + b) = p[u];
    if (!(fl[u] & 1)) continue;
    const int q1 = __ldg(poff + j0 + u + 1);
    for (int q = __ldg(poff + j0 + u); q < q1; ++q) {
      const int code = __ldg(pch + q);
      float* dst = flows + (int64_t)(code >> 1) * ldb + b;
      if (code & 1) {
        *reinterpret_cast<float4*>(dst) = p[u];
      } else if (full) {
        atomicAdd(reinterpret_cast<float4*>(dst), p[u]);
      } else {
        const float pv[4] = {p[u].x, p[u].y, p[u].z, p[u].w};
#pragma unroll
        for (int e = 0; e < VB; ++e)
          if (b + e < B) atomicAdd(dst + e, pv[e]);
      }
    }
  }
}

int launch_prod_accum_push(const Layer& L, cudaStream_t s, int B, int ldb,
                           const float* flow_scratch, float* prod_flows, float* flows) {
  ProfScope prof_(KC_ACCUM_PUSH, s);
  if (!B || !L.n_prod) return PCB_OK;
  dim3 grid((unsigned)((L.n_prod + RW * 4 - 1) / (RW * 4)), (unsigned)((B + SLAB - 1) / SLAB));
  launch_k(k_flow_push, dim3(grid), dim3(RW * 32), 0, s, L.n_prod, B, ldb, L.prod_slots, L.prod_rows, L.push_flag,
                                       L.push_off, L.push_ch, flow_scratch, prod_flows, flows);
  return check_launch();
}

int launch_prod_accum_push_buckets(const Layer& L, cudaStream_t s, int B, int ldb,
                                   const float* flow_scratch, float* prod_flows, float* flows) {
  if (L.n_prod) {
    launch_k(k_prod_accum, dim3(grid_for(L.n_prod * B, 256)), dim3(256), 0, s, L.n_prod, B, ldb, L.prod_slots,
                                                              L.prod_rows, flow_scratch, prod_flows);
    if (check_launch()) return PCB_CUDA;
  }
  for (auto& p : L.pushes) {
    if (!p.n) continue;
    launch_k(k_push, dim3(grid_for(p.n * B, 256)), dim3(256), 0, s, p.n, (int)p.f, B, ldb, p.idx, p.children,
                                                   prod_flows, flows);
    if (check_launch()) return PCB_CUDA;
  }
  return PCB_OK;
}

// ---------------------------------------------------------------- K7
// Input parameter flows (engine.py:168-183): observed -> f[pmf + x] += flow;
// missing -> spread sum(flow) * theta over the pmf.  One CTA per input node.
__global__ void k_input_param_flow(int64_t n, int ncat, int B, int ldb,
                                   const int32_t* __restrict__ slots,
                                   const int32_t* __restrict__ vars, const int32_t* __restrict__ pids,
                                   const int32_t* __restrict__ xT, const float* __restrict__ theta,
                                   const float* __restrict__ flows, float* __restrict__ f_params) {
  pdl_enter();
  // one warp per input node: lanes run along the batch (coalesced flows / x)
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
    const int64_t slot = __ldg(slots + i), var = __ldg(vars + i), pid = __ldg(pids + i);
    float miss = 0.f;
    for (int b = lane; b < B; b += 32) {
      const float f = flows[slot * ldb + b];
      const int x = __ldg(xT + var * ldb + b);
      if (x >= 0) {
        if (f != 0.f) atomicAdd(f_params + pid + x, f);
      } else {
        miss += f;
      }
    }
    for (int o = 16; o > 0; o >>= 1) miss += __shfl_xor_sync(0xffffffffu, miss, o);
    if (miss != 0.f)
      for (int q = lane; q < ncat; q += 32) atomicAdd(f_params + pid + q, miss * __ldg(theta + pid + q));
  }
}

// Staged input flows: a shared-memory histogram [inputs x categories] of the
// block's observed flows (smem atomics), plus the per-input missing-sample
// flow spread over its pmf; the block owns its pmf ranges exclusively, so the
// result is stored to f_params (coalesced, no read-modify-write).
__global__ void __launch_bounds__(IN_THREADS)
    k_input_flow_block(int B, int ldb, const int32_t* __restrict__ bvar,
                       const int32_t* __restrict__ bncat, const int32_t* __restrict__ bslot0,
                       const int32_t* __restrict__ bcount, const int32_t* __restrict__ bpoff,
                       const int32_t* __restrict__ pids, const int32_t* __restrict__ xT,
                       const float* __restrict__ theta, const float* __restrict__ flows,
                       const int32_t* __restrict__ arow, const int32_t* __restrict__ adir,
                       const float* __restrict__ aflows, float* __restrict__ f_params) {
  pdl_enter();
  extern __shared__ float hist[];
  __shared__ float miss[128];
  const int blk = blockIdx.x;
  const int ncat = bncat[blk], cnt = bcount[blk], var = bvar[blk];
  const int64_t slot0 = bslot0[blk];
  const int32_t* pid = pids + bpoff[blk];
  for (int q = threadIdx.x; q < cnt * ncat; q += IN_THREADS) hist[q] = 0.f;
  for (int q = threadIdx.x; q < cnt; q += IN_THREADS) miss[q] = 0.f;
  __syncthreads();
  // input i's flow row: flows[slot0 + i], or the aliased product-flow row
  const int r0 = arow ? __ldg(arow + blk) : -1;
  const float* fbase = r0 >= 0 ? aflows + (int64_t)r0 * ldb : flows + slot0 * ldb;
  const int64_t fstep = r0 >= 0 ? (int64_t)__ldg(adir + blk) * ldb : (int64_t)ldb;
  for (int b = threadIdx.x; b < B; b += IN_THREADS) {
    const int x = xT[(int64_t)var * ldb + b];
    const float* src = fbase + b;
    float* row = (x < 0) ? miss : hist + x;
    const int step = (x < 0) ? 1 : ncat;
    for (int i0 = 0; i0 < cnt; i0 += 8) {
      float f[8];  // 8 independent loads in flight before the smem atomics
#pragma unroll
      for (int u = 0; u < 8; ++u) f[u] = (i0 + u < cnt) ? src[(i0 + u) * fstep] : 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (f[u] != 0.f) atomicAdd(row + (i0 + u) * step, f[u]);
    }
  }
  __syncthreads();
  const int total = cnt * ncat;
  for (int q = threadIdx.x; q < total; q += IN_THREADS) {
    const int i = q / ncat, c = q - i * ncat;
    const float m = miss[i];
    // exclusive pmf range (plan.input_blocks): a store, no read-modify-write
    f_params[pid[i] + c] = hist[q] + (m != 0.f ? m * __ldg(theta + pid[i] + c) : 0.f);
  }
}

// Staged input flows without floating-point atomics (shared-memory float
// atomics are CAS loops on sm_100): the block's samples are counting-sorted
// by category once (native int atomics; missing = bucket ncat), then each warp
// takes input rows: it stages the row's flows in its shared-memory slot
// (coalesced float4) and every lane sums the sorted segments of its
// categories, adding the missing-flow spread, with one coalesced store per
// pmf entry (the block owns its pmf ranges exclusively).
constexpr int IS_THREADS = 256, IS_WARPS = IS_THREADS / 32;
#ifdef PCB_IS_MINB
__global__ void __launch_bounds__(IS_THREADS, PCB_IS_MINB)
#else
__global__ void __launch_bounds__(IS_THREADS)
#endif
    k_input_flow_sorted(int B, int ldb, const int32_t* __restrict__ bvar,
                        const int32_t* __restrict__ bncat, const int32_t* __restrict__ bslot0,
                        const int32_t* __restrict__ bcount, const int32_t* __restrict__ bpoff,
                        const int32_t* __restrict__ pids, const int32_t* __restrict__ xT,
                        const float* __restrict__ theta, const float* __restrict__ flows,
                        const int32_t* __restrict__ arow, const int32_t* __restrict__ adir,
                        const float* __restrict__ aflows, float* __restrict__ f_params,
                        float* __restrict__ em_theta, float kappa, float step,
                        int32_t* __restrict__ status) {
  pdl_enter();
  extern __shared__ __align__(16) uint8_t sm_raw[];
  const int blk = blockIdx.x;
  int informative = 0, bad = 0;
  const int ncat = __ldg(bncat + blk), cnt = __ldg(bcount + blk), var = __ldg(bvar + blk);
  const int64_t slot0 = __ldg(bslot0 + blk);
  const int32_t* pid = pids + __ldg(bpoff + blk);
  const int nb = ncat + 1;                      // buckets incl. missing
  float* rowbuf = reinterpret_cast<float*>(sm_raw);              // [IS_WARPS][ldb]
  int* start = reinterpret_cast<int*>(rowbuf + IS_WARPS * ldb);  // [nb + 1]
  int* fill = start + nb + 1;                   // [nb]
  int* order = fill + nb;                       // [B]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int c = tid; c < nb; c += IS_THREADS) fill[c] = 0;
  __syncthreads();
  const int32_t* xrow = xT + (int64_t)var * ldb;
  for (int b = tid; b < B; b += IS_THREADS) {
    const int x = __ldg(xrow + b);
    atomicAdd(fill + (x < 0 ? ncat : x), 1);
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the bucket sizes
    int run = 0;
    for (int c0 = 0; c0 < nb; c0 += 32) {
      const int c = c0 + lane;
      const int v = c < nb ? fill[c] : 0;
      int inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (c < nb) start[c] = run + inc - v;
      run += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) start[nb] = run;
  }
  __syncthreads();
  for (int c = tid; c < nb; c += IS_THREADS) fill[c] = 0;
  __syncthreads();
  for (int b = tid; b < B; b += IS_THREADS) {
    const int x = __ldg(xrow + b);
    const int k = x < 0 ? ncat : x;
    order[start[k] + atomicAdd(fill + k, 1)] = b;
  }
  __syncthreads();
  float* row = rowbuf + warp * ldb;
  const int m0 = start[ncat], m1 = start[nb];
  // input i's flow row: flows[slot0 + i], or the aliased product-flow row
  const int r0 = arow ? __ldg(arow + blk) : -1;
  const float* fbase = r0 >= 0 ? aflows + (int64_t)r0 * ldb : flows + slot0 * ldb;
  const int64_t fstep = r0 >= 0 ? (int64_t)__ldg(adir + blk) * ldb : (int64_t)ldb;
  for (int i = warp; i < cnt; i += IS_WARPS) {
    const float4* src = reinterpret_cast<const float4*>(fbase + i * fstep);
    for (int q0 = lane; q0 < ldb / 4; q0 += 128) {  // 4 loads in flight per lane
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (q0 + 32 * u < ldb / 4) v[u] = src[q0 + 32 * u];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (q0 + 32 * u < ldb / 4) reinterpret_cast<float4*>(row)[q0 + 32 * u] = v[u];
    }
    __syncwarp();
    float miss = 0.f;
    for (int p = m0 + lane; p < m1; p += 32) miss += row[order[p]];
    for (int o = 16; o > 0; o >>= 1) miss += __shfl_xor_sync(0xffffffffu, miss, o);
    const int64_t base = __ldg(pid + i);
    if (em_theta) {
      // inline EM of the input's pmf (one simplex group, ncat <= 256):
      // k_em's arithmetic on the flows just formed, theta updated in place
      float v[8], o[8], tot = 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u) {  // old theta first: its loads overlap the sums
        const int c = lane + 32 * u;
        o[u] = c < ncat ? em_theta[base + c] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = lane + 32 * u;
        v[u] = 0.f;
        if (c < ncat) {
          float h = 0.f;
          const int p1 = start[c + 1];
          for (int p = start[c]; p < p1; ++p) h += row[order[p]];
          v[u] = h + (miss != 0.f ? miss * o[u] : 0.f) + kappa;
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) tot += v[u];
      for (int o2 = 16; o2 > 0; o2 >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o2);
      if (tot > 0.f) {
        ++informative;
        const float inv = 1.f / tot;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = lane + 32 * u;
          if (c >= ncat) continue;
          const float nv = v[u] * inv;
          const float th = (step >= 1.f) ? nv : ((1.f - step) * o[u] + step * nv);
          if (!isfinite(th)) ++bad;
          em_theta[base + c] = th;
        }
      }
      __syncwarp();
      continue;
    }
    for (int c = lane; c < ncat; c += 32) {
      float h = 0.f;
      const int p1 = start[c + 1];
      for (int p = start[c]; p < p1; ++p) h += row[order[p]];
      f_params[base + c] = h + (miss != 0.f ? miss * __ldg(theta + base + c) : 0.f);
    }
    __syncwarp();
  }
  if (em_theta) {
    for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
    if (lane == 0 && informative) atomicAdd(status, informative);
    if (lane == 0 && bad) atomicAdd(status + 1, bad);
  }
}

// Shared pmfs (plan.shared_pmf_table, e.g. tied HMM emissions): one CTA per
// pmf builds the pmf's flow histogram over every input that uses it (all
// positions x samples) in shared memory, spreads the missing-sample flow
// over the pmf, and stores the whole row — or, with EM inline (one-process
// lean steps), normalises, blends and stores theta directly (em.py:58-94
// for that group; f_params is then not written).
__global__ void __launch_bounds__(SP_THREADS)
    k_input_flow_shared(int ncat, int B, int ldb, const int32_t* __restrict__ u_pid,
                        const int32_t* __restrict__ u_off, const int32_t* __restrict__ u_slot,
                        const int32_t* __restrict__ u_var, const int32_t* __restrict__ xT,
                        const float* __restrict__ flows, float* __restrict__ theta,
                        float* __restrict__ f_params, int em, float kappa, float step,
                        int32_t* __restrict__ status) {
  pdl_enter();
  extern __shared__ float hist[];
  __shared__ float red[SP_THREADS / 32];
  const int u = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t pid = __ldg(u_pid + u);
#if PCB_SP_FLOW_PREFETCH
  // the inline-EM blend reads the whole theta row after the histogram: have
  // TMA pull its aligned body into L2 now, under the histogram phase (the
  // next CTA's row as well measured slower: the blend already streams)
  if (em && tid == 0) l2_prefetch_row(theta, pid, pid + ncat);
#endif
  for (int c = tid; c < ncat; c += SP_THREADS) hist[c] = 0.f;
  __syncthreads();
  float miss = 0.f;
  const int e0 = __ldg(u_off + u), e1 = __ldg(u_off + u + 1);
  // every (input, sample) pair of the pmf spread over the whole CTA, SP_ITEMS
  // pairs' loads in flight per thread before their shared-memory atomics
  const int n_items = (e1 - e0) * B;
  for (int t0 = tid; t0 < n_items; t0 += SP_ITEMS * SP_THREADS) {
    float f[SP_ITEMS];
    int x[SP_ITEMS];
    // branch-free batch (indices clamped to the last item): every item's
    // loads issue before the first atomic
#pragma unroll
    for (int k = 0; k < SP_ITEMS; ++k) {
      const int t = min(t0 + k * SP_THREADS, n_items - 1);
      const int e = e0 + t / B, b = t - (t / B) * B;
      f[k] = flows[(int64_t)__ldg(u_slot + e) * ldb + b];
      x[k] = __ldg(xT + (int64_t)__ldg(u_var + e) * ldb + b);
    }
#pragma unroll
    for (int k = 0; k < SP_ITEMS; ++k) {
      if (t0 + k * SP_THREADS >= n_items || f[k] == 0.f) continue;
      if (x[k] >= 0)
        atomicAdd(hist + x[k], f[k]);
      else
        miss += f[k];
    }
  }
  auto block_sum = [&](float v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float t = 0.f;
#pragma unroll 8
    for (int w = 0; w < SP_THREADS / 32; ++w) t += red[w];
    return t;
  };
  miss = block_sum(miss);
  float* th = theta + pid;
  if (!em) {
    for (int c = tid; c < ncat; c += SP_THREADS)
      f_params[pid + c] = hist[c] + (miss != 0.f ? miss * __ldg(th + c) : 0.f);
    return;
  }
  // inline EM: F = flows (+ missing spread over theta), total sum(F + kappa)
  float tot = 0.f;
  if (miss != 0.f) {
    for (int c0 = tid; c0 < ncat; c0 += SP_UNROLL * SP_THREADS) {
      float v[SP_UNROLL];
#pragma unroll
      for (int k = 0; k < SP_UNROLL; ++k) {
        const int c = c0 + k * SP_THREADS;
        v[k] = c < ncat ? th[c] : 0.f;
      }
#pragma unroll
      for (int k = 0; k < SP_UNROLL; ++k) {
        const int c = c0 + k * SP_THREADS;
        if (c < ncat) {
          const float F = hist[c] + miss * v[k];
          hist[c] = F;
          tot += F + kappa;
        }
      }
    }
  } else {
    for (int c = tid; c < ncat; c += SP_THREADS) tot += hist[c] + kappa;
  }
  tot = block_sum(tot);
  if (!(tot > 0.f)) return;  // uninformative group keeps theta (em.py:67-80)
  const float inv = 1.f / tot;
  int bad = 0;
  // the blend's theta read and write are the pass's traffic: SP_UNROLL
  // loads in flight per thread
  for (int c0 = tid; c0 < ncat; c0 += SP_UNROLL * SP_THREADS) {
    float v[SP_UNROLL];
#pragma unroll
    for (int k = 0; k < SP_UNROLL; ++k) {
      const int c = c0 + k * SP_THREADS;
      v[k] = (c < ncat && step < 1.f) ? th[c] : 0.f;
    }
#pragma unroll
    for (int k = 0; k < SP_UNROLL; ++k) {
      const int c = c0 + k * SP_THREADS;
      if (c < ncat) {
        const float nv = (hist[c] + kappa) * inv;
        const float t = (step >= 1.f) ? nv : ((1.f - step) * v[k] + step * nv);
        bad += !isfinite(t);
        th[c] = t;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if (tid == 0) atomicAdd(status, 1);
  if (lane == 0 && bad) atomicAdd(status + 1, bad);
}

int launch_input_param_flows(const pcb_plan* p, cudaStream_t s, int B, int ldb,
                             const int32_t* xT, float* theta, const float* flows,
                             const float* flow_scratch, float* f_params, bool alias,
                             const Step* em, bool* inline_done, bool* shared_done) {
  ProfScope prof_(KC_INPUT_FLOW, s);
  *inline_done = false;
  *shared_done = false;
  const Step* em_staged = (em && p->in_inline_ok) ? em : nullptr;
  const InBlocks& ib = p->in_blocks;
  const int32_t* arow = (alias && p->leaf_alias) ? ib.alias_row : nullptr;
  // sorted (atomic-free) kernel when its shared-memory slots fit, else the
  // shared-memory histogram
  const int64_t sorted_bytes = ((int64_t)IS_WARPS * ldb + 2 * (ib.max_ncat + 1) + 1 + B) * 4;
  static const bool hist_only = getenv("PCB_INFLOW_HIST") != nullptr;
  if (ib.n && !hist_only && sorted_bytes <= 160 * 1024) {
    static int attr_s[kMaxDev] = {};
    if (ensure_smem((const void*)k_input_flow_sorted, (int)sorted_bytes, attr_s)) return PCB_CUDA;
    launch_k(k_input_flow_sorted, dim3((unsigned)ib.n), dim3(IS_THREADS), (size_t)sorted_bytes, s, 
        B, ldb, ib.var, ib.ncat, ib.slot0, ib.count, ib.pid_off, ib.pids, xT, theta, flows,
        arow, ib.alias_dir, flow_scratch, f_params, em_staged ? theta : nullptr,
        em_staged ? em_staged->kappa : 0.f, em_staged ? em_staged->step : 1.f,
        em_staged ? em_staged->status : nullptr);
    if (check_launch()) return PCB_CUDA;
    *inline_done = em_staged != nullptr;
  } else if (ib.n) {
    const int bytes = (int)ib.max_elems * 4;
    static int attr[kMaxDev] = {};
    if (ensure_smem((const void*)k_input_flow_block, bytes, attr)) return PCB_CUDA;
    launch_k(k_input_flow_block, dim3((unsigned)ib.n), dim3(IN_THREADS), bytes, s, 
        B, ldb, ib.var, ib.ncat, ib.slot0, ib.count, ib.pid_off, ib.pids, xT, theta, flows,
        arow, ib.alias_dir, flow_scratch, f_params);
    if (check_launch()) return PCB_CUDA;
  }
  const bool em_shared = em && p->n_shared_inline > 0;
  for (auto& c : p->inputs) {
    if (!c.n) continue;
    if (c.n_u) {
      const int bytes = (int)c.ncat * 4;
      static int attr_sp[kMaxDev] = {};
      if (ensure_smem((const void*)k_input_flow_shared, bytes, attr_sp)) return PCB_CUDA;
      launch_k(k_input_flow_shared, dim3((unsigned)c.n_u), dim3(SP_THREADS), bytes, s, 
          (int)c.ncat, B, ldb, c.u_pid, c.u_off, c.u_slot, c.u_var, xT, flows, theta, f_params,
          em_shared ? 1 : 0, em ? em->kappa : 0.f, em ? em->step : 1.f,
          em ? em->status : nullptr);
      if (check_launch()) return PCB_CUDA;
      continue;
    }
    launch_k(k_input_param_flow, dim3(grid_for(c.n * 32, 256)), dim3(256), 0, s, c.n, (int)c.ncat, B, ldb, c.slots,
                                                               c.vars, c.pids, xT, theta, flows,
                                                               f_params);
    if (check_launch()) return PCB_CUDA;
  }
  *shared_done = em_shared;
  return PCB_OK;
}

// ---------------------------------------------------------------- K10 root
__global__ void k_root_fwd(int B, int ldb, int64_t root_slot, int64_t root_vb,
                           const int32_t* __restrict__ rc, const int32_t* __restrict__ rcb,
                           int nrc, const float* __restrict__ values,
                           const float* __restrict__ vbase, float* __restrict__ lroot) {
  pdl_enter();
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  // base + offset in double: |log p| may exceed the fp32 spacing of the parts
  double v;
  if (root_slot >= 0) {
    v = (double)values[root_slot * ldb + b];
    if (root_vb >= 0) v += (double)vbase[root_vb * ldb + b];
  } else {
    v = 0.0;
    for (int q = 0; q < nrc; ++q) {
      v += (double)values[(int64_t)rc[q] * ldb + b];
      if (rcb[q] >= 0) v += (double)vbase[(int64_t)rcb[q] * ldb + b];
    }
  }
  lroot[b] = (float)v;
}

int launch_root_fwd(const pcb_plan* p, cudaStream_t s, int B, int ldb, const float* values,
                    const float* vbase_all, float* lroot) {
  ProfScope prof_(KC_MISC, s);
  launch_k(k_root_fwd, dim3((B + 255) / 256), dim3(256), 0, s, B, ldb, p->root_slot, p->root_vb, p->root_children,
                                              p->root_cb, (int)p->n_root_children, values,
                                              vbase_all, lroot);
  return check_launch();
}

__global__ void k_root_bwd(int B, int ldb, int64_t root_slot, int64_t root_row,
                           const int32_t* __restrict__ rc, int nrc, float* __restrict__ flows,
                           float* __restrict__ pf) {
  pdl_enter();
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  if (root_slot >= 0) {
    flows[root_slot * ldb + b] = 1.f;
  } else {
    if (pf) pf[root_row * ldb + b] = 1.f;
    for (int q = 0; q < nrc; ++q) flows[(int64_t)rc[q] * ldb + b] += 1.f;
  }
}

int launch_root_bwd(const pcb_plan* p, cudaStream_t s, int B, int ldb, float* flows,
                    float* prod_flows) {
  ProfScope prof_(KC_MISC, s);
  launch_k(k_root_bwd, dim3((B + 255) / 256), dim3(256), 0, s, B, ldb, p->root_slot, p->root_row,
                                              p->root_children, (int)p->n_root_children, flows,
                                              prod_flows);
  return check_launch();
}

// ---------------------------------------------------------------- K8 replicas
// f[dst + e] += sum over replicas f[src + e] (engine.py:256-257), grouped by
// destination so the sum is race-free and in the reference's order.
__global__ void k_replica_reduce(int64_t n_dst, const int32_t* __restrict__ dst,
                                 const int32_t* __restrict__ len, const int32_t* __restrict__ soff,
                                 const int32_t* __restrict__ src, float* __restrict__ f) {
  pdl_enter();
  for (int64_t d = blockIdx.x; d < n_dst; d += gridDim.x) {
    const int L = len[d];
    const int a = soff[d], z = soff[d + 1];
    for (int e = threadIdx.x; e < L; e += blockDim.x) {
      float acc = f[(int64_t)dst[d] + e];
      for (int k = a; k < z; ++k) acc += f[(int64_t)src[k] + e];
      f[(int64_t)dst[d] + e] = acc;
    }
  }
}

int launch_replica_reduce(const pcb_plan* p, cudaStream_t s, float* f_params) {
  ProfScope prof_(KC_REPLICA, s);
  if (!p->red_n) return PCB_OK;
  launch_k(k_replica_reduce, dim3(grid_for(p->red_n, 1, 148 * 16)), dim3(256), 0, s, 
      p->red_n, p->red_dst, p->red_len, p->red_src_off, p->red_src, f_params);
  return check_launch();
}

// ---------------------------------------------------------------- K9 EM
// One warp per simplex group (em.py:58-94): counts = F + k; groups with a
// positive total are renormalised and blended with step size; others keep
// theta.  Runs over the groups outside tensor-core tile blocks (k_em_tiles).
__global__ void k_em(int64_t n_list, const int32_t* __restrict__ glist,
                     const int32_t* __restrict__ gstart, const int32_t* __restrict__ gidx,
                     const int32_t* __restrict__ goff, const float* __restrict__ F,
                     float* __restrict__ theta, float kappa, float step, int32_t* status) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int informative = 0, bad = 0;
  for (int64_t gi = warp; gi < n_list; gi += nwarps) {
    const int64_t g = __ldg(glist + gi);
    const int a = goff[g], z = goff[g + 1];
    // contiguous groups index theta directly (no index-table reads)
    const int c0 = __ldg(gstart + gi), shift = c0 - a;
    if (c0 >= 0 && z - a <= 256) {
      // small contiguous group (an input pmf): every flow, then every old
      // theta, in flight together; one reduction; stores
      float v[8], o[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = lane + 32 * u;
        v[u] = k < z - a ? __ldg(F + c0 + k) + kappa : 0.f;
      }
      float tot = 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u) tot += v[u];
      for (int o2 = 16; o2 > 0; o2 >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o2);
      if (!(tot > 0.f)) continue;
      ++informative;
      const float inv = 1.f / tot;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = lane + 32 * u;
        o[u] = (k < z - a && step < 1.f) ? theta[c0 + k] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = lane + 32 * u;
        if (k >= z - a) continue;
        const float nv = v[u] * inv;
        const float th = (step >= 1.f) ? nv : ((1.f - step) * o[u] + step * nv);
        if (!isfinite(th)) ++bad;
        theta[c0 + k] = th;
      }
      continue;
    }
    float tot = 0.f;
    for (int k = a + lane; k < z; k += 32) tot += F[c0 >= 0 ? k + shift : gidx[k]] + kappa;
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (!(tot > 0.f)) continue;
    ++informative;
    const float inv = 1.f / tot;
    for (int k = a + lane; k < z; k += 32) {
      const int q = c0 >= 0 ? k + shift : gidx[k];
      const float nv = (F[q] + kappa) * inv;
      const float th = (step >= 1.f) ? nv : ((1.f - step) * theta[q] + step * nv);
      if (!isfinite(th)) ++bad;
      theta[q] = th;
    }
  }
  if (lane == 0 && informative) atomicAdd(status, informative);
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if (lane == 0 && bad) atomicAdd(status + 1, bad);
}

// Big groups (>= EM_BIG entries): one CTA per group, block-reduced total.
__global__ void __launch_bounds__(256)
    k_em_big(int64_t n_list, const int32_t* __restrict__ glist,
             const int32_t* __restrict__ gstart, const int32_t* __restrict__ gidx,
             const int32_t* __restrict__ goff, const float* __restrict__ F,
             float* __restrict__ theta, float kappa, float step, int32_t* status) {
  pdl_enter();
  __shared__ float red[8];
  __shared__ float tot_s;
  int informative = 0, bad = 0;
  for (int64_t gi = blockIdx.x; gi < n_list; gi += gridDim.x) {
    const int64_t g = __ldg(glist + gi);
    const int a = goff[g], z = goff[g + 1];
    const int c0 = __ldg(gstart + gi), shift = c0 - a;
    float tot = 0.f;
    for (int k = a + threadIdx.x; k < z; k += 256) tot += F[c0 >= 0 ? k + shift : gidx[k]] + kappa;
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = tot;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (int w = 0; w < 8; ++w) t += red[w];
      tot_s = t;
    }
    __syncthreads();
    tot = tot_s;
    __syncthreads();  // red / tot_s are reused by the next group
    if (!(tot > 0.f)) continue;
    if (threadIdx.x == 0) ++informative;
    const float inv = 1.f / tot;
    for (int k = a + threadIdx.x; k < z; k += 256) {
      const int q = c0 >= 0 ? k + shift : gidx[k];
      const float nv = (F[q] + kappa) * inv;
      const float th = (step >= 1.f) ? nv : ((1.f - step) * theta[q] + step * nv);
      if (!isfinite(th)) ++bad;
      theta[q] = th;
    }
  }
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if (threadIdx.x == 0 && informative) atomicAdd(status, informative);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(status + 1, bad);
}

int launch_em(const pcb_plan* p, cudaStream_t s, const float* f_params, float* theta,
              float pseudocount, float step, int32_t* status, bool skip_inline,
              bool skip_shared) {
  ProfScope prof_(KC_EM, s);
  // shared-pmf groups (the last rest groups) were updated by the input pass
  const int64_t nb = p->n_em_rest - p->n_em_small - (skip_shared ? p->n_shared_inline : 0);
  // the staged inputs' pmf groups (last among the small ones) were updated
  // by the input-flow pass (inline EM)
  const int64_t ns = skip_inline ? p->n_em_small_noninl : p->n_em_small;
  if (ns) {
    int blocks = grid_for(ns * 32, 256, 148 * 16);
    launch_k(k_em, dim3(blocks), dim3(256), 0, s, ns, p->em_rest, p->em_rest_start, p->group_idx, p->group_off,
                                f_params, theta, pseudocount, step, status);
    if (check_launch()) return PCB_CUDA;
  }
  if (nb) {
    const int64_t s0 = p->n_em_small;
    launch_k(k_em_big, dim3(grid_for(nb, 1, 148 * 8)), dim3(256), 0, s, nb, p->em_rest + s0, p->em_rest_start + s0,
                                                      p->group_idx, p->group_off, f_params,
                                                      theta, pseudocount, step, status);
    if (check_launch()) return PCB_CUDA;
  }
  return PCB_OK;
}

}  // namespace pcb
