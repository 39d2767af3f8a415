// Internal declarations shared by the pcirc_b200 CUDA translation units.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/pcirc_b200.h"

#define PCB_NEG_INF (-__builtin_huge_valf())

namespace pcb {

struct Ref {
  int64_t off = 0;  // element offset into the device int32 blob
  int64_t n = 0;    // element count
};

struct InputChunk {
  int64_t ncat, n;
  const int32_t *slots, *vars, *pids;
  // shared pmfs (plan.shared_pmf_table): per unique pmf (n_u) the CSR of its
  // inputs' value slots and variables; 0 = none
  int64_t n_u = 0;
  const int32_t *u_pid = nullptr, *u_off = nullptr, *u_slot = nullptr, *u_var = nullptr;
};

// Inputs staged per variable in shared memory: block b covers `count`
// consecutive value slots from slot0 on variable var, each with an exclusive
// pmf of ncat entries starting at pids[pid_off + i].
struct InBlocks {
  int64_t n = 0, max_elems = 0, max_ncat = 0, max_count = 0;
  const int32_t *var = nullptr, *ncat = nullptr, *slot0 = nullptr, *count = nullptr,
                *pid_off = nullptr, *pids = nullptr;
  // leaf aliases (plan.leaf_alias): first product row of the block's inputs
  // in the first layer's window (-1: not aliased) and the row step (+1 / -1)
  const int32_t *alias_row = nullptr, *alias_dir = nullptr;
};

struct Bucket {  // product evaluation or push bucket
  int64_t f, n;
  const int32_t* idx;       // out scratch rows (eval) or prod-flow rows (push)
  const int32_t* children;  // [n x f] value slots
};

struct FwdGroup {
  int64_t rows, cap;
  const int32_t *sum_ids, *prod_ids, *param_ids, *flow_ids;
  const int32_t* param_slab;  // bf16 MMA-tile offset per (row, col), -1 for padding
  const int32_t* param_slab_c;  // product-major plane offset per (row, col) (fused EM)
  int exclusive = 0;          // every flow tile of the group has no other writer in the pass
  int uniform = 0;            // every row has the same child blocks (dense layer)
  int pf_pre = 0;             // parameter-flow operands converted once per layer (pf_pre_ok)
};

struct BwdGroup {
  int64_t rows, cap;
  const int32_t *ch_ids, *par_ids, *par_param_ids;
  const int32_t* par_slab;
  int uniform = 0;  // every row has the same parent blocks (dense layer)
};

// Tensor-core work list for one forward / backward group: "super-rows" stack
// sum blocks (or product blocks) that share an identical child (parent) row.
struct TcRows {
  int64_t count = 0;           // number of super-rows
  const int32_t* row_off = 0;  // [count+1] offsets into members (block rows of the group)
  const int32_t* members = 0;  // group-row indices, stacked in order
  // bit 0: contiguous sum rows, bit 1: contiguous children (param-flow stacks);
  // bit 2: the stacked theta tiles of every column are one run per plane
  const int32_t* flags = 0;
};

struct Layer {
  int64_t k_m, k_n, window, n_prod;
  // parameter-flow fusion over tied layers (plan pf fusion id >= 0): this
  // layer's rank among the n members (rank 0 = lowest index = last in the
  // backward pass, which launches the one fused contraction)
  int pf_fuse = -1, pf_fuse_rank = 0, pf_fuse_n = 0;
  int64_t flow_lo = 0, flow_hi = 0;  // the layer's f_params flow range (disjoint when fp_cover)
  int64_t scratch_off;  // first row of this layer's window in the all-layer scratch
  const int32_t* pad_rows;
  int64_t n_pad;
  std::vector<Bucket> evals;
  std::vector<FwdGroup> fwd;
  std::vector<BwdGroup> bwd;
  std::vector<TcRows> fwd_tc;   // aligned with fwd (count 0 = no TC plan)
  std::vector<TcRows> pf_tc;    // aligned with fwd: full stacks for the param-flow kernel
  std::vector<TcRows> bwd_tc;   // aligned with bwd
  std::vector<TcRows> bwd_tc_full;  // aligned with bwd: full stacks (persistent kernels)
  const int32_t *prod_slots, *prod_rows;
  std::vector<Bucket> pushes;
  // derived tables (plan v3)
  const int32_t *prow_off, *prow_ch;  // per scratch row: product children CSR
  const int32_t* prow_cb;             // per CSR child: its value block's vbase row, -1 = base 0
  int prod_uniform = 0;               // every block's rows share one child-base list (row 0's)
  int64_t sb_base, n_sb;              // sum blocks of the layer: slots [sb_base, +n_sb*k_m)
  int64_t n_pb;                       // product blocks in the window incl. pad block 0
  int64_t pb_off = 0, vb_off = 0;     // first pbase / vbase row of the layer
  // fused accumulate + push, product order: flag bit0 push, bit1 first
  // accumulation (store); push_ch = slot * 2 + (single push into the slot)
  const int32_t *push_flag, *push_off, *push_ch;
  // fused push + flow ratio (lean steps, plan.push_ratio_tables): blocks of
  // k products (flow-scratch rows pb_row..+k, fan-in pb_f); per fan-in slot q
  // (pb_qoff..): child base slot, kind (0: flow store, 1: ratio of a
  // pre-ratioed sum block, its R row at q_rrow)
  int64_t n_pblk = 0, n_pq = 0;  // push blocks, fan-in slots
  const int32_t *pb_row = nullptr, *pb_f = nullptr, *pb_qoff = nullptr, *q_blk = nullptr,
                *q_base = nullptr, *q_kind = nullptr, *q_rrow = nullptr;
  int pre_ratio = 0;     // every sum block's ratio comes from a fused push
  // EM fused into this layer's parameter-flow epilogue (plan.em_fused_order):
  // its tile blocks are [em_lo, em_hi)
  int em_fusable = 0;
  int64_t em_lo = 0, em_hi = 0;
  int64_t rmax_off = -1;  // its R rows in the all-layer rmax region
};

// Log values are stored as (integer base, fp32 offset) pairs: every value
// row of a block holds l - base, the base is one integer-valued fp32 per
// (block, sample).  Bases add exactly (|base| < 2^24), so differences of
// log values of any magnitude (|log p| ~ 1.7e4 at 3072 variables, where the
// fp32 spacing is 2^-9) are formed from small offsets and exact integer
// base differences: flows keep full fp32 relative precision.
//   inputs                      base 0 (log-pmf rows)
//   sum block (vbase row)       G = max of its child blocks' bases (the
//                               sum kernels' shift), offsets ln D
//   product block (pbase row)   floor(max_j (sum of its children's bases +
//                               offsets)), -inf for an all -inf block
// Workspace carved from the caller's d_work buffer (pcb_plan_workspace_floats):
//   vbase [n_sb_tot x ldb]  per sum block (all layers) and sample
//   pbase [n_pb_tot x ldb]  per product block (all layers' windows, pad
//                           block 0 included) and sample
//   rmax [max_sb x ldb]  per sum block and sample: max lg2(flow) - offset*log2(e)
//   ratio [max_sum_rows x ldb] per sum row of the layer: log2 flow ratio minus
//                               its block's rmax (k_ratio)
//   gshift [2 max_tc_rows x ldb] per-(super-row, sample) shifts of long-K
//                               layers (child flows: g rows, then base rows)
//   prep [max_prep_rows x ldb]  pre-converted bf16 hi/lo parameter-flow
//                               operand images of one pf_pre layer (+ its shift row)
//   fprep [fuse_prep_rows x ldb] the same for every member of a tied-layer
//                               fusion group, laid end to end along K
//   counters [max_tc_rows x ldb/128] split-K arrivals (self-resetting, zeroed at allocation)
struct Work {
  float* vbase;
  float* pbase;
  float* rmax;
  float* ratio;
  float* gshift;
  float* rmax_all;  // [n_rmax x ldb] R rows of the pre-ratioed layers
  float* prep;
  float* fprep;
  float* part;  // split-K partial sums of co-resident slices (one tile per CTA)
  int32_t* counters;
};

}  // namespace pcb

struct pcb_plan {
  int64_t num_vars, num_value_slots, scratch_size, num_prod_rows, theta_size,
      f_params_size, reserved;
  int64_t root_slot, root_row;
  const int32_t* root_children;
  const int32_t* root_cb;  // vbase row per root child (-1: base 0)
  int64_t n_root_children;
  int64_t root_vb = -1;    // vbase row of a sum root's block
  const int32_t* var_ncat;
  std::vector<pcb::InputChunk> inputs;  // generic (gather / atomic) inputs
  pcb::InBlocks in_blocks;              // shared-memory staged inputs
  std::vector<pcb::Layer> layers;
  // replica reductions grouped by destination tile
  int64_t red_n;
  const int32_t *red_dst, *red_len, *red_src_off, *red_src;
  // simplex groups
  int64_t n_groups;
  const int32_t *group_idx, *group_off;
  // EM tile blocks: k_m groups that exactly tile k_m x k_n tensor-core tiles
  // (updated tile by tile, bf16 planes written in the same pass); the other
  // groups (em_rest) take the generic per-group pass
  int64_t n_em_blk = 0, n_em_tiles = 0, n_em_rest = 0, n_em_small = 0;  // rest: small first
  int em_split32 = 0;  // some tile block takes k_em_tiles32 (pcb_tc.cu)
  int64_t sp_lo = 0, sp_hi = 0;  // f_params range of the shared pmfs (contiguous) or empty
  const int32_t *em_km = nullptr, *em_kn = nullptr, *em_tile_off = nullptr, *em_goff = nullptr,
                *em_tile_start = nullptr, *em_tile_slab_f = nullptr, *em_tile_slab_c = nullptr,
                *em_rest = nullptr,
                *em_rest_start = nullptr;  // first theta index of a contiguous rest group, else -1
  const float* theta_bound = nullptr;  // the plan's own theta (pcb_plan_set_theta)
  int use_tc;  // 0: SIMT; 1: tensor cores (warp-specialised where supported)
  int64_t max_pb = 1, max_sb = 1, max_sum_rows = 1, max_tc_rows = 1;
  int64_t n_pb_tot = 0, n_sb_tot = 0;  // all layers' product / sum blocks (base rows)
  int64_t max_prep_rows = 0;  // pre-converted parameter-flow operand rows (pf_pre groups)
  int64_t fuse_prep_rows = 0;  // ... of the largest tied-layer fusion group
  // bf16 tensor-core copies of theta tiles (plan v4)
  // bf16 planes: regions of mma_plane elements: [F hi][F lo][C hi][C lo];
  // tile t's sum-major planes at slab_f[t] (+ plane), its product-major
  // planes at 2 * plane + slab_c[t] (+ plane)
  int64_t n_mma_tiles = 0, mma_elems = 0, mma_plane = 0;
  const int32_t *mma_theta = nullptr, *mma_slab_f = nullptr, *mma_slab_c = nullptr,
                *mma_km = nullptr, *mma_kn = nullptr;
  __nv_bfloat16* mma = nullptr;  // bound by pcb_plan_set_mma
  int64_t scratch_rows = 1;      // all-layer scratch rows (sum of layer windows)
  int prod_rows_written = 0;     // every prod-flow row is stored by its first accumulation
  int prod_flows_optional = 0;   // every product row is accumulated + pushed in one layer
  // f_params[:theta_size] is the zero tile, the stored pmf ranges of the
  // staged inputs and disjoint per-layer flow ranges: the backward pass zeroes
  // only the ranges of layers that accumulate (no whole-buffer memset)
  int fp_cover = 0;
  // the first layer's products alias their staged inputs (pcb_plan_set_lean)
  int leaf_alias = 0;
  // fused push + ratio usable (every pre-ratioed layer runs the persistent
  // tensor-core flow kernels, which read ratio rows only)
  int push_ratio_ok = 0;
  int64_t n_rmax = 0;
  int64_t n_alias_pad = 0;
  const int32_t* alias_pad = nullptr;  // pad blocks of the first layer's window
  // inline input EM (pcb_train_step with EM): the input-flow pass of a lean
  // backward applies the EM update to the staged inputs' pmf groups (the
  // last small rest groups, [n_em_small_noninl, n_em_small)) directly
  int64_t n_em_small_noninl = 0;
  int in_inline_ok = 0;  // every staged input pmf is such a group (ncat <= 256)
  int64_t n_em_pre = 0;  // tile blocks of layers without fused EM (first in order)
  int64_t n_shared_inline = 0;  // shared-pmf groups (last rest groups) updated by the input pass
  int64_t n_zero = 0;            // flow-row ranges zeroed before the backward pass
  const int32_t *zero_start = nullptr, *zero_len = nullptr;
};

// Per-stream execution state of pcb_train_step (the plan itself is immutable):
// lean steps run the parameter flows of pre-ratioed layers on a side stream,
// forked per layer and joined at the end of the backward pass.
struct pcb_exec {
  ~pcb_exec();
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  // optional, caller-owned: recorded when each layer's parameter flows are
  // issued (index = layer) and after the input flows (index = num layers), so
  // a data-parallel caller can all-reduce finished f_params ranges while the
  // rest of the backward pass runs
  std::vector<cudaEvent_t> flows_done;
};

namespace pcb {

extern unsigned long long g_launches;

// Options of one pass (a plain forward / backward is Step{}); the per-call
// state of a training step lives here, never in the plan.
struct Step {
  int lean = 0;              // 0 full, 1 lean, 2 lean without side-stream overlap
  bool em = false;           // EM inside the backward pass where exact (one-process steps)
  float kappa = 0.f, step = 1.f;
  int32_t* status = nullptr;
  const pcb_exec* ex = nullptr;
  std::vector<char>* em_done = nullptr;  // per layer: EM fused into its parameter flows
  bool inputs_done = false;              // the input-flow pass updated the staged pmfs
  bool shared_done = false;              // ... and the shared pmfs
  bool pass = false;                     // a whole backward pass (stream placement known)
  bool exclusive = false;                // pcb_train_step: one step in flight per device
};

// kernel classes for the live per-class timing used by bench.py
enum KClass {
  KC_INPUT_FWD = 0,
  KC_PROD_EVAL,
  KC_SUM_FWD_TC,
  KC_SUM_FWD_SIMT,
  KC_PARAM_FLOW,
  KC_CHILD_FLOW,
  KC_ACCUM_PUSH,
  KC_INPUT_FLOW,
  KC_REPLICA,
  KC_EM,
  KC_MISC,
  KC_COUNT
};

// Records a CUDA event pair around every launch wrapper of one class when
// profiling is enabled (pcb_profile_enable); otherwise a no-op.
struct ProfScope {
  int cls;
  cudaStream_t s;
  unsigned long long l0;
  int slot;
  ProfScope(int c, cudaStream_t st);
  ~ProfScope();
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: cache the
// largest size set for each device ordinal (cache[kMaxDev] per kernel)
constexpr int kMaxDev = 64;
inline int ensure_smem(const void* fn, int bytes, int* cache) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return PCB_CUDA;
  if (dev >= 0 && dev < kMaxDev && bytes <= cache[dev]) return PCB_OK;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    return PCB_CUDA;
  if (dev >= 0 && dev < kMaxDev) cache[dev] = bytes;
  return PCB_OK;
}

inline int grid_for(int64_t n, int threads, int max_blocks = 148 * 32) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

int check_launch();

// Programmatic dependent launch (PDL).  Every kernel of the library is
// launched through launch_k with cudaLaunchAttributeProgrammaticStream-
// Serialization, and begins with pdl_enter(): griddepcontrol.wait (the
// previous kernel in the stream has completed and its writes are visible --
// no global access happens before it).  No kernel triggers its dependents
// early (the implicit trigger is each CTA's exit): the launch of the next
// kernel is processed ahead and released as this one drains, instead of
// after it (inside CUDA graphs: a programmatic edge).  An early
// griddepcontrol.launch_dependents at kernel entry was measured slower
// (HCLT-256 61.8k vs 62.9k samples/s, HMM-4096 34.4k vs 37.5k): dependent
// CTAs parked on the SMs beside the running kernel cost it issue slots.
// PCB_NO_PDL=1 launches without the attribute (plain stream order; the
// wait is then a no-op).
__device__ __forceinline__ void pdl_enter() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<Args&&>(args)...);
}

// SIMT kernels (pcb_simt.cu).  Base rows: `pbase` / `vbase` point at the
// layer's first product / sum block row (Layer::pb_off / vb_off), except
// where noted.
int launch_input_fwd(const pcb_plan* p, cudaStream_t s, int B, int ldb, const int32_t* xT,
                     const float* theta, float* values, float* scratch_all, float* pbase_all,
                     bool alias);
int launch_prod_eval(const Layer& L, cudaStream_t s, int B, int ldb, const float* values,
                     const float* vbase_all, float* scratch, float* pbase);
int launch_ratio_max(const Layer& L, cudaStream_t s, int B, int ldb, const float* values,
                     const float* flows, float* rmax, float* ratio);
int launch_push_ratio(const Layer& L, cudaStream_t s, int B, int ldb, const float* flow_scratch,
                      const float* values, float* flows, float* rmax_all);
int launch_sum_fwd_simt(const Layer& L, const FwdGroup& g, cudaStream_t s, int B, int ldb,
                        const float* theta, const float* scratch, const float* pbase,
                        float* values, float* vbase);
int launch_param_flow_simt(const Layer& L, const FwdGroup& g, cudaStream_t s, int B, int ldb,
                           const float* theta, const float* values, const float* flows,
                           const float* scratch, const float* pbase, const float* vbase,
                           float* f_params);
int launch_child_flow_simt(const Layer& L, const BwdGroup& g, cudaStream_t s, int B, int ldb,
                           const float* theta, const float* values, const float* flows,
                           const float* scratch, const float* pbase, const float* vbase,
                           float* flow_scratch);
int launch_prod_accum_push(const Layer& L, cudaStream_t s, int B, int ldb,
                           const float* flow_scratch, float* prod_flows, float* flows);
// em: apply EM to the staged inputs' pmfs in this pass (theta updated in place)
int launch_input_param_flows(const pcb_plan* p, cudaStream_t s, int B, int ldb,
                             const int32_t* xT, float* theta, const float* flows,
                             const float* flow_scratch, float* f_params, bool alias,
                             const Step* em, bool* inline_done, bool* shared_done);
// vbase_all: the whole vbase region (root_vb / root_cb are global rows)
int launch_root_fwd(const pcb_plan* p, cudaStream_t s, int B, int ldb, const float* values,
                    const float* vbase_all, float* lroot);
int launch_root_bwd(const pcb_plan* p, cudaStream_t s, int B, int ldb, float* flows,
                    float* prod_flows);
int launch_replica_reduce(const pcb_plan* p, cudaStream_t s, float* f_params);
int launch_em(const pcb_plan* p, cudaStream_t s, const float* f_params, float* theta,
              float pseudocount, float step, int32_t* status, bool skip_inline,
              bool skip_shared = false);
int launch_em_tiles(const pcb_plan* p, cudaStream_t s, const float* f_params, float* theta,
                    float pseudocount, float step, int32_t* status, bool planes,
                    int64_t blk0 = 0, int64_t blk1 = -1);
// EM fused into the parameter-flow epilogue (one-process lean steps)
// a tied-layer parameter-flow fusion member (launch_param_flow_ws)
struct PfFuse {
  int rank, n;   // segment of this layer, members
  float* prep;   // the group's operand images (n shift rows, n x A, n x B)
};

struct PfEm {
  float kappa, step;
  int32_t* status;
  __nv_bfloat16* mma;
  int64_t plane;
  float* theta;  // updated in place
};
int launch_fill_range(cudaStream_t s, int64_t row0, int64_t n, int B, int ldb, float* buf,
                      float v);
int launch_fill(cudaStream_t s, const int32_t* rows, int64_t n, int B, int ldb, float* buf,
                float v);
int launch_zero_ranges(cudaStream_t s, int64_t n, const int32_t* start, const int32_t* len,
                       int ldb, float* buf);

// streaming multiprocessors of the current device (grid sizing)
inline int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

// tensor-core support (pcb_tc.cu)
bool tc_supported(const Layer& L);
bool tc_bwd_supported(const Layer& L);
int launch_theta_to_mma(const pcb_plan* p, cudaStream_t s, const float* theta);
// EM tile block handled by the split kernel k_em_tiles32
bool em_split32_block(int km, int kn, int ntiles);
// warp-specialised persistent tensor-core kernels (pcb_tc_ws.cu), K block 16 / 32
bool ws_supported(int kc, int nb);
// long contractions (>= 32 K blocks, e.g. HMM's 4096-wide layers) use full
// 256-wide stacks and split K across CTAs; short ones keep more, narrower
// super-rows and no split
inline bool ws_long_k(int64_t cap) { return cap >= 32; }
// split_ok: the group owns its layer's output rows, so K may be split
// across CTAs (partial sums reduced in place, finished by the last arrival)
int launch_sum_fwd_ws(const pcb_plan* P, const Layer& L, const FwdGroup& g, const TcRows& tc,
                      cudaStream_t s, int B, int ldb, const float* scratch, const float* pbase,
                      float* values, float* vbase, float* gshift, int32_t* counters,
                      bool split_ok, float* part = nullptr);
int launch_child_flow_ws(const pcb_plan* P, const Layer& L, const BwdGroup& g, const TcRows& tc,
                         cudaStream_t s, int B, int ldb, const float* ratio, const float* scratch,
                         const float* rmax, const float* vbase, const float* pbase,
                         float* flow_scratch, float* gshift, int32_t* counters, bool split_ok,
                         float* part = nullptr);
// floats of the split-K partial-sum slab (one 128 x 256 tile per SM)
int64_t ws_part_floats();
bool pf_ws_supported(const Layer& L);
bool pf_layer_stores(const pcb_plan* P, const Layer& L, int B);
int launch_param_flow_ws(const Layer& L, const FwdGroup& g, const TcRows& tc, cudaStream_t s,
                         int B, int ldb, const float* theta, const float* ratio, const float* rmax,
                         const float* scratch, const float* vbase, const float* pbase,
                         float* f_params, const PfEm* em = nullptr, float* prep = nullptr,
                         const PfFuse* fuse = nullptr);
// the layer may join its tied-layer parameter-flow fusion group
bool pf_fusable(const Layer& L);
// pf_pre groups: image rows of the pre-converted operands
int64_t pf_prep_rows(const Layer& L, const FwdGroup& g);

}  // namespace pcb
