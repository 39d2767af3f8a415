/*
 * pcirc_b200.h — C ABI of the B200-native block-sparse probabilistic-circuit
 * hot path (forward / backward / EM of arXiv 2406.00766, PyJuice).
 *
 * Plain pointers and sizes only; no torch types.  Every pointer named d_* is
 * device memory on the current CUDA device; `stream` is a cudaStream_t cast to
 * void* (0 = legacy default stream).  All launches are asynchronous on that
 * stream; nothing allocates except pcb_plan_create.  Functions return a status:
 *
 *   PCB_OK 0, PCB_USAGE 1 (UsageError), PCB_FORMAT 2 (FormatError),
 *   PCB_NUMERIC 3 (NumericError), PCB_CUDA 4 (launch / runtime failure)
 *
 * mapped by the Python shim onto the reference's exception classes
 * (pcirc/errors.py:8-40).
 *
 * The reference has no native boundary: its hot path is Python/numpy
 * (pcirc/runtime/engine.py, pcirc/runtime/em.py).  Each entry point below
 * replaces the reference function cited beside it; a maintainer binds them
 * with ctypes.
 *
 * Buffer layout (the reference's, pcirc/runtime/buffers.py:18-57): node-major,
 * batch-contiguous fp32 matrices with row stride `ldb` (>= B, multiple of 32):
 *   values, flows        [num_value_slots x ldb]
 *   scratch, flow_scratch [scratch_size   x ldb]
 *   prod_flows           [num_prod_rows   x ldb]
 *   f_params             [f_params_size]        (theta_size prefix + replicas)
 *   theta                [theta_size]
 *   xT                   [num_vars x ldb] int32, category or -1 (missing)
 * Sample columns b >= B are padding and never contribute to parameter flows.
 *
 * Log values are stored as (integer block base, fp32 offset) pairs: d_values
 * and d_scratch hold offsets, d_work holds one integer-valued fp32 base per
 * (sum block | product block, sample) (its first rows: the sum-block bases of
 * all layers in layer order, see pcb_plan_workspace_floats).  A node's log
 * value is offset + base; bases add exactly, so log-value differences (flow
 * ratios) keep fp32 relative precision at any |log p|.
 *
 * Ownership and threading: the plan is immutable after pcb_plan_set_theta /
 * pcb_plan_set_mma and may be shared by any number of streams; every call
 * that runs on a stream takes its mutable state from its arguments (caller-
 * owned buffers and, for pcb_train_step, a per-stream pcb_exec).  The
 * tensor-core kernels read the bf16 planes of the plan's own theta, so
 * passes over tensor-core layers require d_theta == the table bound with
 * pcb_plan_set_theta (PCB_USAGE otherwise).
 */
#ifndef PCIRC_B200_H
#define PCIRC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCB_OK 0
#define PCB_USAGE 1
#define PCB_FORMAT 2
#define PCB_NUMERIC 3
#define PCB_CUDA 4

#define PCB_ABI_VERSION 3

typedef struct pcb_plan pcb_plan;
typedef struct pcb_exec pcb_exec;

/* pcb_train_step flags */
#define PCB_STEP_LEAN 1   /* lean launches (nothing downstream reads node values / flows) */
#define PCB_STEP_SERIAL 2 /* no side-stream overlap (per-kernel-class profiling) */
#define PCB_STEP_EM 4     /* apply the mini-batch EM update inside the call */

/* ABI version of the loaded library. */
int pcb_abi_version(void);

/* Build an immutable execution plan.
 *   prog/prog_len : host int64 program (layer / group records with offsets into
 *                   d_blob), written by paper_2406_00766_b200/runtime/plan.py.
 *   d_blob        : device int32 index tables (compiled layout narrowed to int32).
 * Replaces: pcirc/compiler/ir.py:131-200 (CompiledCircuit consumed by engine.py). */
int pcb_plan_create(const int64_t* prog, int64_t prog_len, const int32_t* d_blob,
                    int64_t blob_len, pcb_plan** out);
int pcb_plan_destroy(pcb_plan* plan);

/* Number of sum layers in the plan. */
int pcb_plan_num_layers(const pcb_plan* plan);

/* Rows of the all-layer product scratch (sum of layer windows): every layer's
 * products stay resident between forward and backward. */
int64_t pcb_plan_scratch_rows(const pcb_plan* plan);

/* Bind the device buffer (>= the plan's MMA-tile element count, bf16) that holds
 * the tensor-core copies of theta, and (re)derive them from d_theta: every
 * tile of a tensor-core layer as bf16 hi + lo planes in UMMA core-matrix
 * order.  Call pcb_theta_refresh after every change of theta. */
int pcb_plan_set_mma(pcb_plan* plan, void* d_mma, int64_t elems);
int pcb_theta_refresh(const pcb_plan* plan, void* stream, const float* d_theta);

/* Bind the plan's own theta table: pcb_em_update on exactly this table also
 * rewrites the bf16 tensor-core planes (no separate pcb_theta_refresh). */
int pcb_plan_set_theta(pcb_plan* plan, const float* d_theta);

/* Validate a device batch (xT, [num_vars x ldb]) against the category counts:
 * writes the number of bad entries to *d_bad (device int32).
 * Replaces: pcirc/runtime/engine.py:36-52 (_validate_batch) for device batches. */
int pcb_check_batch(const pcb_plan* plan, void* stream, int B, int ldb,
                    const int32_t* d_xT, int32_t* d_bad);

/* Transpose a row-major [B x num_vars] int64/int32 batch into xT [num_vars x ldb]. */
int pcb_transpose_batch_i64(const pcb_plan* plan, void* stream, int B, int ldb,
                            const int64_t* d_x, int32_t* d_xT);
int pcb_transpose_batch_i32(const pcb_plan* plan, void* stream, int B, int ldb,
                            const int32_t* d_x, int32_t* d_xT);

/* Floats of device workspace (d_work) the passes below need at row stride ldb:
 * the sum-block bases of all layers [first n_sum_blocks x ldb floats], the
 * product-block bases, per-(sum block, sample) flow-ratio maxima, per-(sum,
 * sample) shifted log2 flow ratios of one layer, long-K shifts and split-K
 * counters.  Derived state, not part of the reference's buffers. */
int64_t pcb_plan_workspace_floats(const pcb_plan* plan, int ldb);

/* Full forward pass: values, scratch, lroot[B].
 * Replaces: pcirc/runtime/engine.py:186-217 (forward). */
int pcb_forward(const pcb_plan* plan, void* stream, int B, int ldb,
                const int32_t* d_xT, const float* d_theta, float* d_values,
                float* d_scratch, float* d_lroot, float* d_work);

/* Full backward pass (flows, prod_flows, f_params incl. replica reduction).
 * d_prod_flows may be NULL when every product row is accumulated and pushed
 * in a single layer (then nothing reads it; PCB_USAGE otherwise).
 * Replaces: pcirc/runtime/engine.py:220-259 (backward). */
int pcb_backward(const pcb_plan* plan, void* stream, int B, int ldb,
                 const int32_t* d_xT, const float* d_theta, const float* d_values,
                 float* d_flows, float* d_scratch, float* d_flow_scratch,
                 float* d_prod_flows, float* d_f_params, float* d_work);

/* Per-layer operator API (the reference's private kernels that
 * pcirc/bench.py:22-27 imports): product evaluation + sum forward of layer
 * `layer` (engine.py:68-102), and its backward (engine.py:105-165 + :249-254). */
int pcb_layer_forward(const pcb_plan* plan, int layer, void* stream, int B, int ldb,
                      const float* d_theta, float* d_values, float* d_scratch, float* d_work);
int pcb_layer_backward(const pcb_plan* plan, int layer, void* stream, int B, int ldb,
                       const float* d_theta, const float* d_values, float* d_flows,
                       float* d_scratch, float* d_flow_scratch, float* d_prod_flows,
                       float* d_f_params, float* d_work);

/* Per-stream execution state of pcb_train_step: a side stream and two
 * events (the parameter flows of pre-ratioed layers overlap the child-flow
 * chain on the side stream).  One per stream that runs training steps. */
int pcb_exec_create(const pcb_plan* plan, pcb_exec** out);
int pcb_exec_destroy(pcb_exec* exec);

/* Optional data-parallel overlap: n caller-owned cudaEvent_t handles.  A
 * step's backward pass records events[l] once sum layer l's parameter flows
 * are issued (on the stream that ran them) and events[num_layers] after the
 * input flows, so the caller can start the all-reduce of each finished
 * f_params range on another stream while the rest of the backward pass runs
 * (the reference's fixed-order merge, pcirc/train.py:100-101, bucketed). */
int pcb_exec_set_flow_events(pcb_exec* exec, void* const* events, int n);

/* One training step on a batch: forward + backward (+ EM with PCB_STEP_EM),
 * the reference's _accumulate_batch + em_step_full + em_step_mini +
 * apply_theta (pcirc/train.py:84-101, :133-142) in one call.
 *   PCB_STEP_LEAN: lean launches.  When the first layer's products are
 *     single-child aliases of exclusively owned staged inputs (plan-
 *     detected), forward writes those inputs' log values straight into the
 *     product rows and backward reads their flows from the product-flow rows
 *     (that layer's product evaluation and push are skipped; those rows of
 *     d_values / d_flows / d_prod_flows are not written); fused push + flow
 *     ratio (the ratio rows of pre-ratioed layers overwrite their d_flows
 *     rows); parameter flows of pre-ratioed layers on exec's side stream.
 *   PCB_STEP_EM (requires d_theta == the plan's bound table): the update
 *     theta <- (1 - step) theta + step normalise(F + pseudocount) of
 *     pcb_em_update is applied in this call.  With PCB_STEP_LEAN, EM runs
 *     inside the backward pass where the plan proves it exact (staged input
 *     pmfs in the input-flow pass; tile blocks of eligible layers in the
 *     parameter-flow epilogue): those parts of d_f_params are not written.
 *     d_status (device int32[2]) is zeroed and receives [informative groups,
 *     non-finite results].  Without PCB_STEP_EM d_theta is read-only and
 *     d_f_params[:theta_size] holds the step's parameter flows (data-parallel
 *     steps all-reduce them, then call pcb_em_update).
 * d_prod_flows may be NULL as for pcb_backward; exec may be NULL (serial).
 * Concurrency: unlike the pure passes, at most one training step may be in
 * flight per device at a time (a second one on another stream or under MPS
 * must be ordered after it): the split-K slices of its long contractions
 * wait for each other on the device and assume their launch owns the SMs it
 * was granted.  Steps of different processes are time-sliced and safe. */
int pcb_train_step(const pcb_plan* plan, const pcb_exec* exec, void* stream, int B, int ldb,
                   const int32_t* d_xT, float* d_theta, float* d_values, float* d_flows,
                   float* d_scratch, float* d_flow_scratch, float* d_prod_flows,
                   float* d_f_params, float* d_lroot, float* d_work, int flags,
                   float pseudocount, float step_size, int32_t* d_status);

/* EM over the simplex groups, in place on d_theta:
 *   theta[g] <- (1 - step) * theta[g] + step * (F[g] + k) / sum(F[g] + k)
 * for every group whose total is > 0 (others keep theta).  step = 1 gives the
 * full-batch renormalisation.  d_status (device int32[2]) receives
 * [informative group count, non-finite result count].  On the table bound by
 * pcb_plan_set_theta the tensor-core planes are refreshed in the same pass.
 * Replaces: pcirc/runtime/em.py:58-94 (em_step_full, em_step_mini, apply_theta). */
int pcb_em_update(const pcb_plan* plan, void* stream, const float* d_f_params,
                  float* d_theta, float pseudocount, float step_size, int32_t* d_status);

/* f[i] += g[i] over n floats (EMAccumulator merge, pcirc/runtime/em.py:48-55). */
int pcb_axpy_accumulate(void* stream, int64_t n, const float* d_src, float* d_dst);

/* Non-finite count of a float vector into *d_count (device int32).
 * Replaces the theta check of pcirc/runtime/engine.py:197-198. */
int pcb_count_nonfinite(void* stream, int64_t n, const float* d_x, int32_t* d_count);

/* Total kernel launches issued by this library (for the bench's gpu_launches claim). */
int64_t pcb_launch_count(void);

/* Live per-kernel-class timing with CUDA events on the launching stream.
 * Classes: 0 input_fwd, 1 prod_eval, 2 sum_fwd_tc, 3 sum_fwd_simt,
 * 4 param_flow, 5 child_flow, 6 accum_push, 7 input_flow, 8 replica, 9 em, 10 misc.
 * pcb_profile_read fills per-class milliseconds, wrapper-scope counts and kernel
 * launch counts accumulated since the previous read (it synchronises). */
int pcb_profile_enable(int on);
int pcb_profile_read(double* ms, int64_t* scopes, int64_t* launches, int n);

/* tcgen05 self-test: D[128 x n] = A[128 x k] . B[n x k]^T in bf16 with fp32
 * accumulation on one CTA (n in {16..256, step 16}, k multiple of 16 <= 256).
 * Used by tests to pin the UMMA descriptor encoding. */
int pcb_tc_selftest(void* stream, int n, int k, const uint16_t* d_a, const uint16_t* d_b,
                    float* d_d);

/* Same with B given as [k x n] row-major and read through an MN-major UMMA
 * descriptor from the theta-tile layout (variant selects the LBO/SBO roles). */
int pcb_tc_selftest_mn(void* stream, int n, int k, int variant, const uint16_t* d_a,
                       const uint16_t* d_b, float* d_d);

#ifdef __cplusplus
}
#endif

#endif /* PCIRC_B200_H */
