// C ABI: plan parsing and the forward / backward / EM orchestration
// (pcirc/runtime/engine.py:186-259, pcirc/runtime/em.py:58-94).
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <new>

#include "pcb_internal.cuh"

using namespace pcb;

namespace {

constexpr int64_t kMagic = 0x50434232;  // "PCB2"
constexpr int64_t kVersion = 28;

struct Reader {
  const int64_t* p;
  int64_t n, i = 0;
  const int32_t* blob;
  int64_t blob_len;
  bool ok = true;
  int64_t get() {
    if (i >= n) {
      ok = false;
      return 0;
    }
    return p[i++];
  }
  const int32_t* ref(int64_t* count = nullptr) {
    int64_t off = get(), cnt = get();
    if (count) *count = cnt;
    if (off < 0 || cnt < 0 || off + cnt > blob_len) {
      ok = false;
      return nullptr;
    }
    return blob + off;
  }
};

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace

extern "C" {

int pcb_abi_version(void) { return PCB_ABI_VERSION; }

int64_t pcb_launch_count(void) { return (int64_t)g_launches; }

int pcb_plan_create(const int64_t* prog, int64_t prog_len, const int32_t* d_blob,
                    int64_t blob_len, pcb_plan** out) {
  if (!prog || !out) return PCB_USAGE;
  Reader r{prog, prog_len};
  r.blob = d_blob;
  r.blob_len = blob_len;
  if (r.get() != kMagic || r.get() != kVersion) return PCB_USAGE;
  pcb_plan* P = new (std::nothrow) pcb_plan();
  if (!P) return PCB_USAGE;
  P->num_vars = r.get();
  P->num_value_slots = r.get();
  P->scratch_size = r.get();
  P->num_prod_rows = r.get();
  P->theta_size = r.get();
  P->f_params_size = r.get();
  P->reserved = r.get();
  P->root_slot = r.get();
  P->root_row = r.get();
  P->root_children = r.ref(&P->n_root_children);
  P->root_cb = r.ref();
  P->root_vb = r.get();
  P->var_ncat = r.ref();
  P->use_tc = (int)r.get();
  P->n_mma_tiles = r.get();
  P->mma_elems = r.get();
  P->mma_plane = r.get();
  P->mma_theta = r.ref();
  P->mma_slab_f = r.ref();
  P->mma_slab_c = r.ref();
  P->mma_km = r.ref();
  P->mma_kn = r.ref();
  P->scratch_rows = r.get();
  int64_t n_chunks = r.get();
  for (int64_t c = 0; c < n_chunks && r.ok; ++c) {
    InputChunk ch;
    ch.ncat = r.get();
    ch.n = r.get();
    ch.slots = r.ref();
    ch.vars = r.ref();
    ch.pids = r.ref();
    ch.n_u = r.get();
    ch.u_pid = r.ref();
    ch.u_off = r.ref();
    ch.u_slot = r.ref();
    ch.u_var = r.ref();
    P->inputs.push_back(ch);
  }
  P->in_blocks.n = r.get();
  P->in_blocks.var = r.ref();
  P->in_blocks.ncat = r.ref();
  P->in_blocks.slot0 = r.ref();
  P->in_blocks.count = r.ref();
  P->in_blocks.pid_off = r.ref();
  P->in_blocks.pids = r.ref();
  P->in_blocks.max_elems = r.get();
  P->in_blocks.max_ncat = r.get();
  P->in_blocks.max_count = r.get();
  P->in_blocks.alias_row = r.ref();
  P->in_blocks.alias_dir = r.ref();
  P->leaf_alias = (int)r.get();
  P->alias_pad = r.ref(&P->n_alias_pad);
  P->n_zero = r.get();
  P->zero_start = r.ref();
  P->zero_len = r.ref();
  P->prod_rows_written = (int)r.get();
  int64_t n_layers = r.get();
  for (int64_t l = 0; l < n_layers && r.ok; ++l) {
    Layer L;
    L.k_m = r.get();
    L.k_n = r.get();
    L.window = r.get();
    L.n_prod = r.get();
    L.scratch_off = r.get();
    L.flow_lo = r.get();
    L.flow_hi = r.get();
    L.pad_rows = r.ref(&L.n_pad);
    int64_t ne = r.get();
    for (int64_t e = 0; e < ne && r.ok; ++e) {
      Bucket b;
      b.f = r.get();
      b.n = r.get();
      b.idx = r.ref();
      b.children = r.ref();
      L.evals.push_back(b);
    }
    int64_t nf = r.get();
    for (int64_t g = 0; g < nf && r.ok; ++g) {
      FwdGroup G;
      G.rows = r.get();
      G.cap = r.get();
      G.sum_ids = r.ref();
      G.prod_ids = r.ref();
      G.param_ids = r.ref();
      G.flow_ids = r.ref();
      G.param_slab = r.ref();
      G.param_slab_c = r.ref();
      G.exclusive = (int)r.get();
      G.uniform = (int)r.get();
      G.pf_pre = (int)r.get();
      TcRows T, Tp;
      T.count = r.get();
      T.row_off = r.ref();
      T.members = r.ref();
      T.flags = r.ref();
      Tp.count = r.get();
      Tp.row_off = r.ref();
      Tp.members = r.ref();
      Tp.flags = r.ref();
      L.fwd.push_back(G);
      L.fwd_tc.push_back(T);
      L.pf_tc.push_back(Tp);
      if (Tp.count > P->max_tc_rows) P->max_tc_rows = Tp.count;
    }
    int64_t nb = r.get();
    for (int64_t g = 0; g < nb && r.ok; ++g) {
      BwdGroup G;
      G.rows = r.get();
      G.cap = r.get();
      G.ch_ids = r.ref();
      G.par_ids = r.ref();
      G.par_param_ids = r.ref();
      G.par_slab = r.ref();
      G.uniform = (int)r.get();
      TcRows T, Tf;
      T.count = r.get();
      T.row_off = r.ref();
      T.members = r.ref();
      T.flags = r.ref();
      Tf.count = r.get();
      Tf.row_off = r.ref();
      Tf.members = r.ref();
      Tf.flags = r.ref();
      L.bwd.push_back(G);
      L.bwd_tc.push_back(T);
      L.bwd_tc_full.push_back(Tf);
      if (Tf.count > P->max_tc_rows) P->max_tc_rows = Tf.count;
    }
    L.prod_slots = r.ref();
    L.prod_rows = r.ref();
    int64_t np = r.get();
    for (int64_t e = 0; e < np && r.ok; ++e) {
      Bucket b;
      b.f = r.get();
      b.n = r.get();
      b.idx = r.ref();
      b.children = r.ref();
      L.pushes.push_back(b);
    }
    L.prow_off = r.ref();
    L.prow_ch = r.ref();
    L.prow_cb = r.ref();
    L.prod_uniform = (int)r.get();
    L.sb_base = r.get();
    L.n_sb = r.get();
    L.push_flag = r.ref();
    L.push_off = r.ref();
    L.push_ch = r.ref();
    L.n_pblk = r.get();
    L.pb_row = r.ref();
    L.pb_f = r.ref();
    L.pb_qoff = r.ref();
    L.q_blk = r.ref(&L.n_pq);
    L.q_base = r.ref();
    L.q_kind = r.ref();
    L.q_rrow = r.ref();
    L.pre_ratio = (int)r.get();
    L.rmax_off = r.get();
    L.pf_fuse = (int)r.get();
    L.n_pb = L.window / L.k_n;  // including the -inf pad block 0
    for (const FwdGroup& G : L.fwd)
      if (G.pf_pre) P->max_prep_rows = std::max(P->max_prep_rows, pf_prep_rows(L, G));
    L.pb_off = P->n_pb_tot;
    L.vb_off = P->n_sb_tot;
    P->n_pb_tot += L.n_pb;
    P->n_sb_tot += L.n_sb;
    if (L.n_pb > P->max_pb) P->max_pb = L.n_pb;
    if (L.n_sb > P->max_sb) P->max_sb = L.n_sb;
    if (L.n_sb * L.k_m > P->max_sum_rows) P->max_sum_rows = L.n_sb * L.k_m;
    P->layers.push_back(std::move(L));
  }
  // tied-layer parameter-flow fusion groups: rank members by layer index
  for (size_t li = 0; li < P->layers.size(); ++li) {
    Layer& L = P->layers[li];
    if (L.pf_fuse < 0) continue;
    int rank = 0, n = 0;
    for (size_t lj = 0; lj < P->layers.size(); ++lj)
      if (P->layers[lj].pf_fuse == L.pf_fuse) {
        ++n;
        if (lj < li) ++rank;
      }
    L.pf_fuse_rank = rank;
    L.pf_fuse_n = n;
    if (L.fwd.size() == 1)
      P->fuse_prep_rows = std::max(P->fuse_prep_rows, (int64_t)n * pf_prep_rows(L, L.fwd[0]));
  }
  P->red_n = r.get();
  P->red_dst = r.ref();
  P->red_len = r.ref();
  P->red_src_off = r.ref();
  P->red_src = r.ref();
  P->n_groups = r.get();
  P->group_idx = r.ref();
  P->group_off = r.ref();
  P->n_em_blk = r.get();
  P->n_em_tiles = r.get();
  P->em_km = r.ref();
  P->em_kn = r.ref();
  P->em_tile_off = r.ref();
  P->em_goff = r.ref();
  P->em_tile_start = r.ref();
  P->em_tile_slab_f = r.ref();
  P->em_tile_slab_c = r.ref();
  P->n_em_rest = r.get();
  P->n_em_small = r.get();
  P->em_rest = r.ref();
  P->em_rest_start = r.ref();
  P->prod_flows_optional = (int)r.get();
  P->fp_cover = (int)r.get();
  P->n_rmax = r.get();
  P->n_em_small_noninl = r.get();
  P->in_inline_ok = (int)r.get();
  P->n_em_pre = r.get();
  for (auto& L : P->layers) {
    L.em_lo = r.get();
    L.em_hi = r.get();
    L.em_fusable = (int)r.get();
  }
  P->n_shared_inline = r.get();
  P->em_split32 = (int)r.get();  // some tile block takes k_em_tiles32
  P->sp_lo = r.get();            // f_params range stored whole by k_input_flow_shared
  P->sp_hi = r.get();
  if (!r.ok || r.get() != kMagic) {
    delete P;
    return PCB_USAGE;
  }
  // the fused push may pre-compute a layer's flow ratios only if that layer's
  // flow kernels are the persistent tensor-core ones (they read ratio rows,
  // never flows)
  P->push_ratio_ok = P->use_tc == 1 && P->n_rmax > 0;
  for (const Layer& L : P->layers) {
    if (!L.pre_ratio) continue;
    bool ok = tc_bwd_supported(L) && ws_supported((int)L.k_m, (int)L.k_n) && pf_ws_supported(L) &&
              L.k_m <= 64 && (L.k_n == 16 || L.k_n == 32 || L.k_n == 64);
    for (size_t g = 0; g < L.pf_tc.size(); ++g) ok = ok && L.pf_tc[g].count > 0;
    for (size_t g = 0; g < L.bwd_tc.size(); ++g) ok = ok && L.bwd_tc[g].count > 0;
    if (!ok) P->push_ratio_ok = 0;
  }
  *out = P;
  return PCB_OK;
}

pcb_exec::~pcb_exec() {
  if (fork) cudaEventDestroy(fork);
  if (join) cudaEventDestroy(join);
  if (side) cudaStreamDestroy(side);
}

int pcb_exec_create(const pcb_plan* plan, pcb_exec** out) {
  if (!plan || !out) return PCB_USAGE;
  pcb_exec* E = new (std::nothrow) pcb_exec();
  if (!E) return PCB_USAGE;
  if (cudaStreamCreateWithFlags(&E->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&E->fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&E->join, cudaEventDisableTiming) != cudaSuccess) {
    delete E;
    return PCB_CUDA;
  }
  *out = E;
  return PCB_OK;
}

int pcb_exec_set_flow_events(pcb_exec* exec, void* const* events, int n) {
  if (!exec || n < 0 || (n && !events)) return PCB_USAGE;
  exec->flows_done.assign(n, nullptr);
  for (int i = 0; i < n; ++i) exec->flows_done[i] = reinterpret_cast<cudaEvent_t>(events[i]);
  return PCB_OK;
}

int pcb_exec_destroy(pcb_exec* exec) {
  delete exec;
  return PCB_OK;
}

int pcb_plan_destroy(pcb_plan* plan) {
  delete plan;
  return PCB_OK;
}

int pcb_plan_num_layers(const pcb_plan* plan) { return plan ? (int)plan->layers.size() : -1; }

int pcb_plan_set_mma(pcb_plan* plan, void* d_mma, int64_t elems) {
  if (!plan || elems < plan->mma_elems) return PCB_USAGE;
  plan->mma = reinterpret_cast<__nv_bfloat16*>(d_mma);
  return PCB_OK;
}

int pcb_plan_set_theta(pcb_plan* plan, const float* d_theta) {
  if (!plan) return PCB_USAGE;
  plan->theta_bound = d_theta;
  return PCB_OK;
}

int pcb_theta_refresh(const pcb_plan* plan, void* stream, const float* d_theta) {
  if (!plan) return PCB_USAGE;
  return launch_theta_to_mma(plan, as_stream(stream), d_theta);
}

int64_t pcb_plan_scratch_rows(const pcb_plan* plan) { return plan ? plan->scratch_rows : -1; }

}  // extern "C"

namespace {

__global__ void k_check_batch(int64_t nv, int B, int ldb, const int32_t* __restrict__ ncat,
                              const int32_t* __restrict__ xT, int32_t* bad) {
  pdl_enter();
  int64_t total = nv * (int64_t)B;
  int cnt = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t v = t / B;
    int b = (int)(t - v * B);
    int x = xT[v * ldb + b];
    if (x < -1 || x >= ncat[v]) ++cnt;
  }
  if (cnt) atomicAdd(bad, cnt);
}

template <typename T>
__global__ void k_transpose(int64_t nv, int B, int ldb, const T* __restrict__ x,
                            int32_t* __restrict__ xT) {
  pdl_enter();
  __shared__ int32_t tile[32][33];
  const int64_t v0 = (int64_t)blockIdx.x * 32;
  const int b0 = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    int b = b0 + k;
    int64_t v = v0 + threadIdx.x;
    if (b < B && v < nv) tile[k][threadIdx.x] = (int32_t)x[(int64_t)b * nv + v];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    int64_t v = v0 + k;
    int b = b0 + threadIdx.x;
    if (b < B && v < nv) xT[v * ldb + b] = tile[threadIdx.x][k];
  }
}

__global__ void k_axpy(int64_t n, const float* __restrict__ a, float* __restrict__ y) {
  pdl_enter();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    y[t] += a[t];
}

__global__ void k_nonfinite(int64_t n, const float* __restrict__ x, int32_t* cnt) {
  pdl_enter();
  int c = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    c += !isfinite(x[t]);
  if (c) atomicAdd(cnt, c);
}

// spread: split-K slices of the long-K sum kernels may wait for each other
// on the device (spread finish, partial-sum slab), which needs all of a
// launch's CTAs co-resident: only training steps, whose contract is one step
// in flight per device (pcirc_b200.h), enable it; the pure passes, which may
// run on any number of concurrent streams, keep the last-arrival finish.
Work carve(const pcb_plan* P, int ldb, float* d_work, bool spread = false) {
  Work w;
  w.vbase = d_work;
  w.pbase = w.vbase + P->n_sb_tot * (int64_t)ldb;
  w.rmax = w.pbase + P->n_pb_tot * (int64_t)ldb;
  w.ratio = w.rmax + P->max_sb * (int64_t)ldb;
  w.gshift = w.ratio + P->max_sum_rows * (int64_t)ldb;
  w.rmax_all = w.gshift + 2 * P->max_tc_rows * (int64_t)ldb;
  w.prep = w.rmax_all + P->n_rmax * (int64_t)ldb;
  w.fprep = w.prep + P->max_prep_rows * (int64_t)ldb;
  w.part = w.fprep + P->fuse_prep_rows * (int64_t)ldb;
  w.counters = reinterpret_cast<int32_t*>(w.part + ws_part_floats());
  if (!spread) w.part = nullptr;
  return w;
}

// the layer's products alias their inputs in this (lean) pass
bool lean_alias(const pcb_plan* P, const Step& st, const Layer& L) {
  return st.lean && P->leaf_alias && &L == &P->layers[0];
}

// Products of every layer stay resident in their own window of the
// all-layer scratch, so the backward pass reads them instead of recomputing
// (the reference recomputes into one shared window, engine.py:242).
int layer_forward(const pcb_plan* P, const Step& S, const Layer& L, cudaStream_t s, int B,
                  int ldb, const float* theta, float* values, float* scratch_all, const Work& w) {
  float* scratch = scratch_all + L.scratch_off * (int64_t)ldb;
  float* pbase = w.pbase + L.pb_off * (int64_t)ldb;
  float* vbase = w.vbase + L.vb_off * (int64_t)ldb;
  int st;
  if (lean_alias(P, S, L)) {
    // the input pass wrote the product rows and block bases: only the
    // window's padding rows / blocks need -inf
    st = launch_fill(s, L.pad_rows, L.n_pad, B, ldb, scratch, PCB_NEG_INF);
    if (!st) st = launch_fill(s, P->alias_pad, P->n_alias_pad, B, ldb, pbase, PCB_NEG_INF);
  } else {
    st = launch_prod_eval(L, s, B, ldb, values, w.vbase, scratch, pbase);
  }
  if (st) return st;
  for (size_t g = 0; g < L.fwd.size(); ++g) {
    const TcRows& T = L.fwd_tc[g];
    if (P->use_tc && T.count > 0 && tc_supported(L) && ws_supported((int)L.k_n, (int)L.k_m))
      st = launch_sum_fwd_ws(P, L, L.fwd[g], ws_long_k(L.fwd[g].cap) ? L.pf_tc[g] : T, s, B, ldb,
                             scratch, pbase, values, vbase, w.gshift, w.counters,
                             L.fwd.size() == 1, w.part);
    else
      st = launch_sum_fwd_simt(L, L.fwd[g], s, B, ldb, theta, scratch, pbase, values, vbase);
    if (st) return st;
  }
  return PCB_OK;
}

// f_params[0, zero_tile) collects the padding edges' flows (param id 0)
int64_t zero_tile(const pcb_plan* P) {
  int64_t z = 0;
  for (const Layer& L : P->layers) z = std::max(z, L.k_m * L.k_n);
  return z;
}

int child_flows(const pcb_plan* P, const Layer& L, cudaStream_t s, int B, int ldb,
                const float* theta, const float* values, const float* flows, float* scratch,
                float* flow_scratch, const float* ratio, const float* rmax, bool tc,
                const Work& w) {
  const float* pbase = w.pbase + L.pb_off * (int64_t)ldb;
  const float* vbase = w.vbase + L.vb_off * (int64_t)ldb;
  for (size_t g = 0; g < L.bwd.size(); ++g) {
    const TcRows& T = L.bwd_tc[g];
    int st;
    if (tc && T.count > 0 && P->use_tc == 1 && ws_supported((int)L.k_m, (int)L.k_n))
      st = launch_child_flow_ws(P, L, L.bwd[g], ws_long_k(L.bwd[g].cap) ? L.bwd_tc_full[g] : T,
                                s, B, ldb, ratio, scratch, rmax, vbase, pbase, flow_scratch,
                                w.gshift, w.counters, L.bwd.size() == 1, w.part);
    else
      st = launch_child_flow_simt(L, L.bwd[g], s, B, ldb, theta, values, flows, scratch, pbase,
                                  vbase, flow_scratch);
    if (st) return st;
  }
  return PCB_OK;
}

// the layer's parameter flows run on the exec's side stream in this step
static bool pf_side(const pcb_plan* P, const Step& S, const Layer& L) {
  return S.lean && P->push_ratio_ok && L.pre_ratio && S.ex && S.lean != 2;
}

// Tied-layer parameter-flow fusion in this pass: a whole backward pass, no
// per-layer flow hooks (data parallel), and the rank-0 member (launched last)
// on the side stream whenever any member is, so every member's operand
// staging precedes the fused contraction in stream order.
static bool pf_fuse_ok(const pcb_plan* P, const Step& S, const Layer& L, bool tc) {
  if (!tc || !S.pass || !pf_fusable(L) || (S.ex && !S.ex->flows_done.empty())) return false;
  bool any_side = false, zero_side = false;
  for (const Layer& M : P->layers) {
    if (M.pf_fuse != L.pf_fuse) continue;
    if (!pf_fusable(M)) return false;
    const bool sd = pf_side(P, S, M);
    any_side |= sd;
    if (M.pf_fuse_rank == 0) zero_side = sd;
  }
  return zero_side || !any_side;
}

int layer_backward(const pcb_plan* P, Step& S, size_t li, cudaStream_t s, int B, int ldb,
                   float* theta, const float* values, float* flows, float* scratch_all,
                   float* flow_scratch, float* prod_flows, float* f_params, const Work& w) {
  const Layer& L = P->layers[li];
  float* scratch = scratch_all + L.scratch_off * (int64_t)ldb;
  int st = PCB_OK;
  // tensor-core flows: the persistent kernels (K blocks 16 / 32); other
  // block sizes take the SIMT kernels
  const bool tc = P->use_tc == 1 && tc_bwd_supported(L) && ws_supported((int)L.k_m, (int)L.k_n) &&
                  pf_ws_supported(L);
  const bool fused = S.lean && P->push_ratio_ok;
  // pre-ratioed layers (fused push): the flow rows already hold the ratios
  const float* ratio = w.ratio;
  const float* rmax = w.rmax;
  if (fused && L.pre_ratio) {
    ratio = flows + L.sb_base * (int64_t)ldb;
    rmax = w.rmax_all + L.rmax_off * (int64_t)ldb;
  } else if (tc) {
    st = launch_ratio_max(L, s, B, ldb, values, flows, w.rmax, w.ratio);
    if (st) return st;
  }
  // parameter flows: on the side stream when their inputs (ratio rows in the
  // flows buffer, per-layer R rows, the layer's scratch window) stay valid
  // for the rest of the pass, i.e. for pre-ratioed layers of a lean step.
  // EM fused into the parameter-flow epilogue (one-process lean step with
  // EM): the layer's theta tiles and planes are rewritten there, so its
  // parameter flows run after its child flows (which read the planes)
  static const bool em_fuse_off = getenv("PCB_NO_EM_FUSE") != nullptr;  // A/B experiments
  const bool em_fuse = S.em && S.em_done && L.em_fusable && fused && L.pre_ratio && P->mma &&
                       tc && pf_layer_stores(P, L, B) && !em_fuse_off;
  if (em_fuse) {
    st = child_flows(P, L, s, B, ldb, theta, values, flows, scratch, flow_scratch, ratio, rmax,
                     tc, w);
    if (st) return st;
  }
  cudaStream_t sp = s;
  if (fused && L.pre_ratio && S.ex && S.lean != 2) {
    if (cudaEventRecord(S.ex->fork, s) != cudaSuccess ||
        cudaStreamWaitEvent(S.ex->side, S.ex->fork, 0) != cudaSuccess)
      return PCB_CUDA;
    sp = S.ex->side;
  }
  PfEm em{S.kappa, S.step, S.status, P->mma, P->mma_plane, theta};
  // accumulating layers zero their own flow range first (fp_cover plans skip
  // the whole-buffer memset)
  if (P->fp_cover && L.flow_hi > L.flow_lo && !(tc && B > 0 && pf_layer_stores(P, L, B)) &&
      cudaMemsetAsync(f_params + L.flow_lo, 0, sizeof(float) * (L.flow_hi - L.flow_lo), sp) !=
          cudaSuccess)
    return PCB_CUDA;
  const float* pbase = w.pbase + L.pb_off * (int64_t)ldb;
  const float* vbase = w.vbase + L.vb_off * (int64_t)ldb;
  for (size_t g = 0; g < L.fwd.size(); ++g) {
    const TcRows& T = L.pf_tc[g];
    if (tc && T.count > 0) {
      const PfFuse fz{L.pf_fuse_rank, L.pf_fuse_n, w.fprep};
      const bool fuse = !em_fuse && pf_fuse_ok(P, S, L, tc);
      st = launch_param_flow_ws(L, L.fwd[g], T, sp, B, ldb, theta, ratio, rmax, scratch, vbase,
                                pbase, f_params, em_fuse ? &em : nullptr, w.prep,
                                fuse ? &fz : nullptr);
    } else {
      st = launch_param_flow_simt(L, L.fwd[g], sp, B, ldb, theta, values, flows, scratch, pbase,
                                  vbase, f_params);
    }
    if (st) return st;
  }
  if (S.ex && li < S.ex->flows_done.size() && S.ex->flows_done[li] &&
      cudaEventRecord(S.ex->flows_done[li], sp) != cudaSuccess)
    return PCB_CUDA;
  if (em_fuse) {
    (*S.em_done)[li] = 1;
  } else {
    st = child_flows(P, L, s, B, ldb, theta, values, flows, scratch, flow_scratch, ratio, rmax,
                     tc, w);
    if (st) return st;
  }
  // aliased leaf products: the input pass reads their flow rows directly
  if (lean_alias(P, S, L)) return PCB_OK;
  if (fused && L.n_pblk)
    return launch_push_ratio(L, s, B, ldb, flow_scratch, values, flows, w.rmax_all);
  return launch_prod_accum_push(L, s, B, ldb, flow_scratch, prod_flows, flows);
}

int run_forward(const pcb_plan* P, const Step& S, cudaStream_t s, int B, int ldb,
                const int32_t* d_xT, const float* d_theta, float* d_values, float* d_scratch,
                float* d_lroot, float* d_work) {
  const Work w = carve(P, ldb, d_work, S.exclusive);
  // values.fill(-inf) (engine.py:204): every input and sum-block row (padding
  // rows included) is written below, so only the reserved constant rows need it.
  int st = launch_fill_range(s, 0, P->reserved, B, ldb, d_values, PCB_NEG_INF);
  if (st) return st;
  st = launch_input_fwd(P, s, B, ldb, d_xT, d_theta, d_values, d_scratch, w.pbase, S.lean != 0);
  if (st) return st;
  for (auto& L : P->layers) {
    st = layer_forward(P, S, L, s, B, ldb, d_theta, d_values, d_scratch, w);
    if (st) return st;
  }
  return launch_root_fwd(P, s, B, ldb, d_values, w.vbase, d_lroot);
}

int run_backward(const pcb_plan* P, Step& S, cudaStream_t s, int B, int ldb,
                 const int32_t* d_xT, float* d_theta, const float* d_values, float* d_flows,
                 float* d_scratch, float* d_flow_scratch, float* d_prod_flows, float* d_f_params,
                 float* d_work) {
  // prod_flows may be skipped only when no product row accumulates across layers
  if (!d_prod_flows && P->num_prod_rows && !P->prod_flows_optional) return PCB_USAGE;
  const Work w = carve(P, ldb, d_work, S.exclusive);
  {
    ProfScope prof_(KC_MISC, s);
    // replica ranges (past theta_size) are folded onto their master tiles and
    // never written: a lean step, whose EM reads only [0, theta_size), leaves
    // them alone
    const int64_t fp_n = P->fp_cover ? zero_tile(P) : S.lean ? P->theta_size : P->f_params_size;
    // the shared-pmf rows are stored whole by their input-flow kernel (or,
    // with EM inline, not written at all): no zero fill there
    const int64_t sk_lo = std::max(P->sp_lo, zero_tile(P)), sk_hi = std::min(P->sp_hi, fp_n);
    if (B > 0 && sk_lo < sk_hi && getenv("PCB_NO_FP_SKIP") == nullptr) {
      if (cudaMemsetAsync(d_f_params, 0, sizeof(float) * sk_lo, s) != cudaSuccess ||
          cudaMemsetAsync(d_f_params + sk_hi, 0, sizeof(float) * (fp_n - sk_hi), s) !=
              cudaSuccess)
        return PCB_CUDA;
    } else if (cudaMemsetAsync(d_f_params, 0, sizeof(float) * fp_n, s) != cudaSuccess) {
      return PCB_CUDA;
    }
    if (!B) return PCB_OK;
    // only rows that accumulate (several pushes) or receive none need zeros;
    // single-push rows are stored by their push
    if (launch_zero_ranges(s, P->n_zero, P->zero_start, P->zero_len, ldb, d_flows))
      return PCB_CUDA;
    // every product row's first accumulation stores (plan flag): no zeroing
    if (d_prod_flows && P->num_prod_rows && !P->prod_rows_written &&
        cudaMemsetAsync(d_prod_flows, 0, sizeof(float) * P->num_prod_rows * ldb, s) !=
            cudaSuccess)
      return PCB_CUDA;
  }
  const bool side = S.lean && P->push_ratio_ok && S.ex && S.lean != 2;
  S.pass = true;  // every layer's stream placement is this pass's (pf_fuse_ok)
  int st = launch_root_bwd(P, s, B, ldb, d_flows, d_prod_flows);
  if (st) return st;
  for (size_t li = P->layers.size(); li-- > 0;) {
    st = layer_backward(P, S, li, s, B, ldb, d_theta, d_values, d_flows, d_scratch,
                        d_flow_scratch, d_prod_flows, d_f_params, w);
    if (st) return st;
  }
  bool done = false, sdone = false;
  st = launch_input_param_flows(P, s, B, ldb, d_xT, d_theta, d_flows, d_flow_scratch, d_f_params,
                                S.lean != 0, S.em ? &S : nullptr, &done, &sdone);
  if (st) return st;
  S.inputs_done = done;
  S.shared_done = sdone;
  const size_t nl = P->layers.size();
  if (S.ex && nl < S.ex->flows_done.size() && S.ex->flows_done[nl] &&
      cudaEventRecord(S.ex->flows_done[nl], s) != cudaSuccess)
    return PCB_CUDA;
  if (side && (cudaEventRecord(S.ex->join, S.ex->side) != cudaSuccess ||
               cudaStreamWaitEvent(s, S.ex->join, 0) != cudaSuccess))
    return PCB_CUDA;
  return launch_replica_reduce(P, s, d_f_params);
}

// The EM pass over the groups the backward pass did not already update
// (S.em_done layers' tile blocks, the staged inputs when S.inputs_done);
// d_status accumulates (zeroed by the caller).
int run_em(const pcb_plan* P, const Step* S, cudaStream_t s, const float* d_f_params,
           float* d_theta, float kappa, float step, int32_t* d_status) {
  // the plan's own table: the tile-block pass also rewrites the bf16 MMA
  // planes; tensor-core tiles outside tile blocks get the separate refresh
  const bool own = d_theta == P->theta_bound && P->mma;
  int st = PCB_OK;
  if (S && S->em_done) {
    // tile blocks of layers whose EM ran in their parameter-flow epilogue are
    // skipped (blocks are ordered: other layers first, then layer by layer)
    int64_t lo = 0, hi = P->n_em_pre;
    for (size_t li = 0; li < P->layers.size(); ++li) {
      const Layer& L = P->layers[li];
      if (!L.em_fusable || L.em_hi <= L.em_lo) continue;
      const bool done = (*S->em_done)[li] != 0;
      if (!done && L.em_lo == hi) {
        hi = L.em_hi;
        continue;
      }
      if (!done) {
        st = launch_em_tiles(P, s, d_f_params, d_theta, kappa, step, d_status, own, lo, hi);
        if (st) return st;
        lo = L.em_lo;
        hi = L.em_hi;
      }
    }
    st = launch_em_tiles(P, s, d_f_params, d_theta, kappa, step, d_status, own, lo, hi);
  } else {
    st = launch_em_tiles(P, s, d_f_params, d_theta, kappa, step, d_status, own);
  }
  if (st) return st;
  st = launch_em(P, s, d_f_params, d_theta, kappa, step, d_status, S && S->inputs_done,
                 S && S->shared_done);
  if (st) return st;
  if (own && P->n_em_tiles < P->n_mma_tiles) return launch_theta_to_mma(P, s, d_theta);
  return PCB_OK;
}

// the tensor-core kernels read the bf16 planes of the plan's bound table
bool theta_ok(const pcb_plan* P, const float* d_theta) {
  return !P->use_tc || (P->mma && d_theta == P->theta_bound);
}

bool bad_dims(const pcb_plan* p, int B, int ldb) {
  return !p || B < 0 || ldb < B || (ldb % 32) != 0;
}

}  // namespace

extern "C" {

int pcb_check_batch(const pcb_plan* plan, void* stream, int B, int ldb, const int32_t* d_xT,
                    int32_t* d_bad) {
  if (bad_dims(plan, B, ldb)) return PCB_USAGE;
  if (!B) return PCB_OK;
  launch_k(k_check_batch, dim3(grid_for(plan->num_vars * B, 256)), dim3(256), 0, as_stream(stream), 
      plan->num_vars, B, ldb, plan->var_ncat, d_xT, d_bad);
  return check_launch();
}

int pcb_transpose_batch_i64(const pcb_plan* plan, void* stream, int B, int ldb,
                            const int64_t* d_x, int32_t* d_xT) {
  if (bad_dims(plan, B, ldb)) return PCB_USAGE;
  if (!B) return PCB_OK;
  dim3 grid((unsigned)((plan->num_vars + 31) / 32), (unsigned)((B + 31) / 32));
  launch_k((k_transpose<int64_t>), dim3(grid), dim3(dim3(32, 8)), 0, as_stream(stream), plan->num_vars, B, ldb, d_x,
                                                                     d_xT);
  return check_launch();
}

int pcb_transpose_batch_i32(const pcb_plan* plan, void* stream, int B, int ldb,
                            const int32_t* d_x, int32_t* d_xT) {
  if (bad_dims(plan, B, ldb)) return PCB_USAGE;
  if (!B) return PCB_OK;
  dim3 grid((unsigned)((plan->num_vars + 31) / 32), (unsigned)((B + 31) / 32));
  launch_k((k_transpose<int32_t>), dim3(grid), dim3(dim3(32, 8)), 0, as_stream(stream), plan->num_vars, B, ldb, d_x,
                                                                     d_xT);
  return check_launch();
}

int64_t pcb_plan_workspace_floats(const pcb_plan* plan, int ldb) {
  if (!plan || ldb <= 0) return -1;
  // + one split-K arrival counter per (super-row, 128-sample tile)
  return (plan->n_sb_tot + plan->n_pb_tot + plan->max_sb + plan->max_sum_rows +
          2 * plan->max_tc_rows + plan->n_rmax + plan->max_prep_rows + plan->fuse_prep_rows) *
             (int64_t)ldb +
         ws_part_floats() +
         plan->max_tc_rows * (int64_t)((ldb + 127) / 128);
}

int pcb_forward(const pcb_plan* plan, void* stream, int B, int ldb, const int32_t* d_xT,
                const float* d_theta, float* d_values, float* d_scratch, float* d_lroot,
                float* d_work) {
  if (bad_dims(plan, B, ldb) || !d_work || !theta_ok(plan, d_theta)) return PCB_USAGE;
  if (!B) return PCB_OK;
  return run_forward(plan, Step{}, as_stream(stream), B, ldb, d_xT, d_theta, d_values, d_scratch,
                     d_lroot, d_work);
}

int pcb_backward(const pcb_plan* plan, void* stream, int B, int ldb, const int32_t* d_xT,
                 const float* d_theta, const float* d_values, float* d_flows, float* d_scratch,
                 float* d_flow_scratch, float* d_prod_flows, float* d_f_params, float* d_work) {
  if (bad_dims(plan, B, ldb) || !d_work || !theta_ok(plan, d_theta)) return PCB_USAGE;
  Step S;  // no EM: theta is only read
  return run_backward(plan, S, as_stream(stream), B, ldb, d_xT, const_cast<float*>(d_theta),
                      d_values, d_flows, d_scratch, d_flow_scratch, d_prod_flows, d_f_params,
                      d_work);
}

int pcb_train_step(const pcb_plan* plan, const pcb_exec* exec, void* stream, int B, int ldb,
                   const int32_t* d_xT, float* d_theta, float* d_values, float* d_flows,
                   float* d_scratch, float* d_flow_scratch, float* d_prod_flows,
                   float* d_f_params, float* d_lroot, float* d_work, int flags,
                   float pseudocount, float step_size, int32_t* d_status) {
  const bool em = (flags & PCB_STEP_EM) != 0;
  if (bad_dims(plan, B, ldb) || !d_work || !theta_ok(plan, d_theta) ||
      (flags & ~(PCB_STEP_LEAN | PCB_STEP_SERIAL | PCB_STEP_EM)))
    return PCB_USAGE;
  if (em && (!(pseudocount >= 0.f) || !(step_size > 0.f) || step_size > 1.f || !d_status ||
             d_theta != plan->theta_bound))
    return PCB_USAGE;
  cudaStream_t s = as_stream(stream);
  std::vector<char> em_done(plan->layers.size(), 0);
  Step S;
  S.lean = (flags & PCB_STEP_LEAN) ? ((flags & PCB_STEP_SERIAL) || !exec ? 2 : 1) : 0;
  S.ex = exec;
  S.exclusive = true;
  if (em) {
    S.em = S.lean != 0;  // EM inside the backward pass: lean launches only
    S.kappa = pseudocount;
    S.step = step_size;
    S.status = d_status;
    S.em_done = &em_done;
    if (cudaMemsetAsync(d_status, 0, 2 * sizeof(int32_t), s) != cudaSuccess) return PCB_CUDA;
  }
  int st = PCB_OK;
  if (B) {
    st = run_forward(plan, S, s, B, ldb, d_xT, d_theta, d_values, d_scratch, d_lroot, d_work);
    if (st) return st;
  }
  st = run_backward(plan, S, s, B, ldb, d_xT, d_theta, d_values, d_flows, d_scratch,
                    d_flow_scratch, d_prod_flows, d_f_params, d_work);
  if (st || !em) return st;
  return run_em(plan, &S, s, d_f_params, d_theta, pseudocount, step_size, d_status);
}

int pcb_layer_forward(const pcb_plan* plan, int layer, void* stream, int B, int ldb,
                      const float* d_theta, float* d_values, float* d_scratch, float* d_work) {
  if (bad_dims(plan, B, ldb) || !d_work || layer < 0 || layer >= (int)plan->layers.size() ||
      !theta_ok(plan, d_theta))
    return PCB_USAGE;
  if (!B) return PCB_OK;
  return layer_forward(plan, Step{}, plan->layers[layer], as_stream(stream), B, ldb, d_theta,
                       d_values, d_scratch, carve(plan, ldb, d_work));
}

int pcb_layer_backward(const pcb_plan* plan, int layer, void* stream, int B, int ldb,
                       const float* d_theta, const float* d_values, float* d_flows,
                       float* d_scratch, float* d_flow_scratch, float* d_prod_flows,
                       float* d_f_params, float* d_work) {
  if (bad_dims(plan, B, ldb) || !d_work || layer < 0 || layer >= (int)plan->layers.size() ||
      !theta_ok(plan, d_theta) ||
      (!d_prod_flows && plan->num_prod_rows && !plan->prod_flows_optional))
    return PCB_USAGE;
  if (!B) return PCB_OK;
  Step S;
  return layer_backward(plan, S, (size_t)layer, as_stream(stream), B, ldb,
                        const_cast<float*>(d_theta), d_values, d_flows, d_scratch,
                        d_flow_scratch, d_prod_flows, d_f_params, carve(plan, ldb, d_work));
}

int pcb_em_update(const pcb_plan* plan, void* stream, const float* d_f_params, float* d_theta,
                  float pseudocount, float step_size, int32_t* d_status) {
  if (!plan || !d_status || !(pseudocount >= 0.f) || !(step_size > 0.f) || step_size > 1.f)
    return PCB_USAGE;
  cudaStream_t s = as_stream(stream);
  if (cudaMemsetAsync(d_status, 0, 2 * sizeof(int32_t), s) != cudaSuccess) return PCB_CUDA;
  return run_em(plan, nullptr, s, d_f_params, d_theta, pseudocount, step_size, d_status);
}

int pcb_axpy_accumulate(void* stream, int64_t n, const float* d_src, float* d_dst) {
  if (n <= 0) return PCB_OK;
  launch_k(k_axpy, dim3(grid_for(n, 256)), dim3(256), 0, as_stream(stream), n, d_src, d_dst);
  return check_launch();
}

int pcb_count_nonfinite(void* stream, int64_t n, const float* d_x, int32_t* d_count) {
  cudaStream_t s = as_stream(stream);
  if (cudaMemsetAsync(d_count, 0, sizeof(int32_t), s) != cudaSuccess) return PCB_CUDA;
  if (n <= 0) return PCB_OK;
  launch_k(k_nonfinite, dim3(grid_for(n, 256)), dim3(256), 0, s, n, d_x, d_count);
  return check_launch();
}

}  // extern "C"
