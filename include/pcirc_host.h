/*
 * pcirc_host.h -- C ABI of the native host-compiler core
 * (paper_2406_00766_b200/_lib/libpcirc_host.so, csrc/host/pcc_compile.cpp).
 *
 * Host-only (no CUDA): the passes of compile_circuit that are proportional
 * to the edge count, restating pcirc/compiler/build.py:183-631 and
 * blocks.py:73-148 with the reference's orderings.  The Python compiler
 * (compiler/build.py, compiler/_native.py) drives them; a reference-side
 * binding would call them in the same order.  All arrays
 * are caller-owned, C-contiguous int64 unless noted; pointer tables
 * (`const int64_t* const*`) hold one row-major matrix per segment.
 * Results never depend on the worker count.
 */
#ifndef PCIRC_HOST_H
#define PCIRC_HOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int pcc_version(void);
void pcc_set_threads(int n); /* 0 = hardware concurrency */
int pcc_threads(void);

/* build.py:195-222 -- one sum layer's per-edge arrays (sum id, child id,
 * child key = id for products / -2 - id for inputs, slot) from its
 * segments; ch_stride[s] = row stride of segment s's children (0: one row
 * shared by every sum of the segment). */
void pcc_gather_layer(int nseg, const int64_t* const* children, const int64_t* ch_stride,
                      const int64_t* const* slots, const int64_t* fan,
                      const int64_t* const* rows, const int64_t* nrows, const int64_t* starts,
                      const int8_t* kinds, int8_t product_kind, int64_t vkey_base,
                      int64_t* e_sum, int64_t* e_child, int64_t* e_key, int64_t* e_slot);

/* blocks.py:73-148 -- a layer handle over (sum ids, child keys CSR); the
 * arrays must outlive the handle.  pcc_blocks returns 0, or 3 when the key
 * range exceeds int32.  meta = km, kn, demoted, n_sb, n_pb, n_prod_keys,
 * n_cb; pads = sum / product pad fractions. */
void* pcc_layer_new(int64_t n, const int64_t* sids, int64_t E, const int64_t* key,
                    const int64_t* off);
void pcc_layer_free(void* h);
int pcc_blocks(void* h, int64_t k, int64_t k_n, double demote);
void pcc_blocks_meta(void* h, int64_t* meta, double* pads);
void pcc_blocks_get(void* h, int64_t* smat, int64_t* pmat, int64_t* cb_flat, int64_t* cb_off,
                    int64_t* sum_keys, int64_t* sum_blk, int64_t* sum_off, int64_t* prod_keys,
                    int64_t* prod_blk, int64_t* prod_off);

/* build.py:251-339 -- theta layout.  pcc_slot_uses marks rep slots used by
 * sum edges (seen / multi bitsets); pcc_tiles lays out one blocked layer's
 * tiles (returns 0, 1 = parallel edge, 2 = misaligned tying, 4 = theta
 * capacity); the tile table carries tied patterns and writer counts across
 * layers. */
void pcc_slot_uses(int64_t E, const int64_t* slots, const int64_t* rep, uint64_t* seen,
                   uint64_t* multi);
void* pcc_tiles_new(void);
void pcc_tiles_free(void* t);
int64_t pcc_tiles_count(void* t);
void pcc_tiles_get(void* t, int64_t* starts, int64_t* writers);
int pcc_tiles(void* h, void* table, const int64_t* slots, const int64_t* rep,
              const uint64_t* multi, const double* params, double* theta, int64_t theta_cap,
              int64_t* theta_size, int64_t* slot_phys, int64_t* ref, int64_t* pair_theta);
void pcc_release(void); /* frees the scratch kept across one compile's layers */

/* input pmf ranges (build.py:251-290): theta copies, slot_phys + tying claims */
void pcc_fill_i64(int64_t* p, int64_t n, int64_t v);
void pcc_copy_ranges(int64_t n, const int64_t* src_start, const int64_t* len,
                     const int64_t* dst_start, const double* src, double* dst);
void pcc_iota_ranges(int64_t n, const int64_t* dst_off, const int64_t* start,
                     const int64_t* len, int64_t* out);
int pcc_assign_ranges(int64_t n, const int64_t* slot_start, const int64_t* len,
                      const int64_t* phys_start, int ordered, int64_t* slot_phys,
                      const int64_t* rep, int64_t* ref);
int pcc_claim_ranges(int64_t n, const int64_t* start, const int64_t* len, uint64_t* bits);

/* build.py:535-567 -- simplex groups: disjoint fast path (returns 1 on a
 * shared position) and the general path's exact row grouping + claims. */
int pcc_sum_groups_multi(int64_t nseg, const int64_t* counts, const int64_t* fans,
                         const int64_t* const* slot_ptrs, const int64_t* slot_phys,
                         uint64_t* bits, const int64_t* dst, int64_t* group_idx);
void* pcc_rows_new(void);
void pcc_rows_free(void* h);
void pcc_rows_add_multi(void* h, int64_t nseg, const int64_t* counts, int64_t fan,
                        const int64_t* const* slot_ptrs, const int64_t* id0s,
                        const int64_t* slot_phys, int64_t* contig_start);
int64_t pcc_rows_count(void* h, int64_t* n_members);
void pcc_rows_get(void* h, int64_t* first_id, int64_t* off, int64_t* members);
int pcc_claim_groups(int64_t ngroups, const int64_t* group_off, const int64_t* group_idx,
                     int64_t* claim);

/* build.py:103-110 depths; build.py:634-657 graph-hash records */
void pcc_depths(int64_t nseg, const int64_t* starts, const int64_t* counts, const int64_t* fans,
                const int8_t* kinds, const int64_t* const* child_ptrs, const int64_t* strides,
                int64_t* depth);
void pcc_hash_records_multi(int64_t nseg, const int8_t* kinds, const int64_t* counts,
                            const int64_t* fans, const int64_t* const* a,
                            const int64_t* a_stride, const int64_t* const* b,
                            const int64_t* b_stride, const int64_t* const* c, uint8_t* out);

/* device-plan table helpers (runtime/plan.py) */
void pcc_group_runs(int64_t ngroups, const int64_t* go, const int64_t* gi, int64_t* run_off,
                    int64_t* rs, int64_t* rl);
void pcc_minmax(const int64_t* a, int64_t n, int64_t* out);
void pcc_narrow_i32(const int64_t* src, int64_t n, int32_t* dst);

#ifdef __cplusplus
}
#endif

#endif /* PCIRC_HOST_H */
