/*
 * epsgraph_b200.h -- C ABI of the B200-native eps-graph build path.
 *
 * The reference (`epsgraph` 0.1.0) is a pure-Python package whose hot loops
 * are numba @njit kernels; it has no FFI layer of its own.  Each entry point
 * below replaces one reference function (cited file:line, relative to
 * /root/reference/pkg/src/epsgraph/), and the Python package
 * `paper_0904_3151_b200` binds them through ctypes exactly where the
 * reference calls its numba kernels.
 *
 * Conventions
 *  - Every pointer argument named d_* is DEVICE memory owned by the caller;
 *    h_* pointers are host memory.  The library never allocates or frees
 *    caller memory; scratch comes from a caller-provided workspace whose size
 *    is returned by the matching *_workspace() query.
 *  - `stream` is a cudaStream_t passed as void*; all work is enqueued on it.
 *    Functions that must return a count synchronise that stream once.
 *  - Row indices are < 2^32.  Pair keys are uint64 (i << 32) | j with i < j,
 *    so sorting keys sorts pairs lexicographically by (i, j).
 *  - Return value: EG_OK or one of the EG_ERR_* codes; eg_last_error()
 *    returns a message for the last failure on the calling thread.
 */
#ifndef EPSGRAPH_B200_H
#define EPSGRAPH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EG_OK 0
#define EG_ERR_ARG 1          /* invalid argument (-> ValueError)            */
#define EG_ERR_CUDA 2         /* CUDA runtime failure (-> RuntimeError)      */
#define EG_ERR_CAPACITY 3     /* output capacity too small; count returned   */
#define EG_ERR_WORKSPACE 4    /* workspace smaller than *_workspace() says   */
#define EG_ERR_UNSUPPORTED 5  /* shape outside the kernels' limits           */

#define EG_METRIC_COSINE 0
#define EG_METRIC_EUCLIDEAN 1

/* Largest string length / block count the enumeration kernels support. */
#define EG_MAX_LENGTH 256
#define EG_MAX_BLOCKS 64
/* replicates a pair tag can name (d_out_rep is uint16)                   */
#define EG_MAX_REPLICATES 65535

const char *eg_last_error(void);

/* Path overrides for tests and tuning (the product never reads the       */
/* environment).  Names: "project_path" (0 auto, 1 SIMT, 2 kind::tf32,    */
/* 3 unfused norms, 4 non-TMA tensor-core kernel), "fixup_force_seq",     */
/* "fixup_cap" (> 0 caps the band-entry list: overflow path),            */
/* "msm_blocks" (> 0 forces the block count or a design's plan code      */
/* 10000 + 100 v + m, -1 keeps the reference's), "msm_designs" (0: the    */
/* plan considers complete designs only), "msm_batches" (> 0: launch      */
/* batches per eg_msm_pairs call), "plan_debug" (1: eg_msm_plan prints    */
/* its candidates to stderr), "msm_streams" (1 or 2), "verify_wide",      */
/* "sort_path" (-1 auto, 0 onesweep, 1 classic).  EG_ERR_ARG for an       */
/* unknown name or value.                                                 */
/* Process-wide; not synchronised with calls in flight.                   */
int eg_set_option(const char *name, long long value);
void eg_reset_options(void);
int eg_version(void);
/* Number of SMs of the current device (for host-side sizing). */
int eg_device_sm_count(void);

/* Instrumentation (bench.py): number of kernels this library has launched,
 * and optional per-kernel-class CUDA-event timing.  eg_profile_read
 * synchronises the recorded events, fills ms/count per class (class names
 * from eg_profile_class_name) and clears the record; returns #classes. */
long long eg_launch_count(void);
void eg_profile_enable(int on);
const char *eg_profile_class_name(int cls);
int eg_profile_read(double *ms_out, long long *count_out, int max_classes);

/* --------------------------------------------------------------------- */
/* Row statistics.  Replaces the validation in VectorDataset.__init__     */
/* (lsh.py:48-57), _check_norms (lsh.py:121-125) and the norm pass of     */
/* filter_exact (pipeline.py:203).                                        */
/* d_x: n x dim row-major, float32 (x_is_f64 = 0) or float64 (= 1).       */
/* d_norms[n] = sqrt(sum_q x_q^2) in fp64, squares added by fma in        */
/* ascending q (one fixed order on every path).  d_bad (device uint64[2]):*/
/* [0] = first row with a non-finite entry, [1] = first zero-norm row,    */
/* UINT64_MAX when none.  Asynchronous (no host synchronisation), so the  */
/* build can check the flags once at its end.                             */
/* --------------------------------------------------------------------- */
int eg_row_stats(const void *d_x, int x_is_f64, int64_t n, int32_t dim,
                 double *d_norms, uint64_t *d_bad, void *stream);

/* --------------------------------------------------------------------- */
/* Projection + sign packing.  Replaces _sign_bits (lsh.py:96-113),       */
/* _project_words (lsh.py:128-147) and BitStringPool.from_bits            */
/* (bitpool.py:125-141) for `replicates` replicates at once.              */
/* d_r: (replicates*length) x dim fp64 directions, replicate-major (the   */
/* host draws them with numpy exactly as lsh.py:116-118,145 does).        */
/* d_rnorm[replicates*length]: fp64 Euclidean norms of those rows.        */
/* d_codes: replicates x n x W uint64, W = ceil(length/64); bit t of a    */
/* row is word t/64, position t%64; padding bits are zero.                */
/* Signs are bit-identical to the reference's sequential fp64 sum: a fast */
/* pass decides every entry whose |dot| exceeds a certified error band;   */
/* the rest are recomputed with separately rounded fp64 mul/add (if the   */
/* band list overflows, every entry is recomputed exactly, on device).    */
/* d_fixups (optional, device uint64) receives the number of band         */
/* entries.  Asynchronous.                                                */
/* --------------------------------------------------------------------- */
size_t eg_project_workspace(int64_t n, int32_t dim, int32_t length, int32_t replicates);
int eg_project(const void *d_x, int x_is_f64, int64_t n, int32_t dim,
               const double *d_norms, const double *d_r, const double *d_rnorm,
               int32_t length, int32_t replicates, uint64_t *d_codes,
               void *d_workspace, size_t workspace_bytes, uint64_t *d_fixups,
               void *stream);

/* eg_row_stats + eg_project in one call: d_norms / d_bad are OUTPUTS (as  */
/* eg_row_stats).  On the tensor-core path the norms are accumulated by    */
/* the projection kernel itself, so the rows cross HBM once; elsewhere the */
/* two kernels run back to back.  Same results as the separate calls.      */
/* Workspace: eg_project_workspace.  Asynchronous.                         */
int eg_project_rows(const void *d_x, int x_is_f64, int64_t n, int32_t dim,
                    double *d_norms, uint64_t *d_bad, const double *d_r,
                    const double *d_rnorm, int32_t length, int32_t replicates,
                    uint64_t *d_codes, void *d_workspace, size_t workspace_bytes,
                    uint64_t *d_fixups, void *stream);

/* Test hook: when d_buf is non-null, the tensor-core projection path also */
/* writes its raw fp32 accumulator (n x replicates*length) to d_buf, so the */
/* tests can measure the worst error against the exact fp64 product.       */
void eg_debug_set_tc_dump(float *d_buf);
/* Debug: MSM counters (zero unless built with -DEG_MSM_STATS=1):          */
/* [0..5] buckets, rows, filter candidates, groups, grouped rows, pair    */
/* visits of the hash-table tiers; [8..15] reserved (zero).               */
int eg_debug_msm_stats(unsigned long long *out16, int reset);

/* --------------------------------------------------------------------- */
/* Multiple-sorting-method enumeration over (replicate, mask) units.      */
/* Replaces, per unit, masked_key_table (bitpool.py:224-253),             */
/* _counting_pass/_sort_grouped (hamming_join.py:52-82, 252-272),         */
/* _group_bounds (:85-101), _emit_group_pairs (:104-149), and the         */
/* cross-replicate first-witness fold (pipeline.py:286-314).              */
/* d_codes: replicates x n x W (as produced by eg_project, or a pool).    */
/* h_block_bounds[k+1]: block offsets (bitpool.py:44-69).                 */
/* h_unit_rep[n_units], h_unit_mask[n_units]: replicate index and block   */
/* bitmask (bit b set = block b masked) of each unit; |mask| == d.        */
/* A pair (i<j) is emitted by unit (h, B) iff popcount(c_i^c_j) <= d in   */
/* replicate h, B is the lexicographically first d-subset containing the  */
/* blocks where they differ (== the reference's first-witness mask rule), */
/* and popcount > d in every replicate g < h.                             */
/* d_out_keys[capacity]: emitted pair keys, in no particular order.       */
/* d_out_rep (optional, replicates > 1): when given, the cross-replicate  */
/* rule is NOT applied here; every raw pair is emitted with its replicate */
/* index in d_out_rep[slot] and eg_xrep_filter applies the rule later.    */
/* h_counts (2*replicates + 2 int64): [0] total emitted (may exceed       */
/* capacity -> EG_ERR_CAPACITY), [1] largest equal-key group seen,        */
/* [2+h] raw pairs of replicate h (before the cross-replicate rule),      */
/* [2+replicates+h] new pairs of replicate h (0 when deferred).           */
/* --------------------------------------------------------------------- */
size_t eg_msm_workspace(int64_t n, int32_t length, int32_t replicates);

/* --------------------------------------------------------------------- */
/* Block-count plan for eg_msm_pairs.  The pair set the units emit is     */
/* {(i,j): popcount(c_i^c_j) <= d}, independent of the block count        */
/* (hamming_join.py:300-375), so the count is a cost knob:    */
/* C(k',d) units of n rows each vs. the in-group pairs visited.  Samples  */
/* up to 8192 rows of d_codes (replicate 0, n x W), counts sum C(g,2)     */
/* and the largest group for probe masks of every k' in (d, min(L,64)],   */
/* and returns in *h_k_out the k' minimising the modelled cost (k itself  */
/* unless another is >= 5% cheaper).  k is always returned when the       */
/* reference's oversized-group warning (largest group > fraction * n,     */
/* hamming_join.py:341-348) could fire on the reference blocks, when      */
/* n < 65536, or when C(k,d) > 4096.  Blocks of every k' follow the       */
/* reference partition (first L % k' blocks one bit wider).  Synchronous. */
/* h_cost (optional, 2 doubles): modelled ms of the chosen and of k.      */
/* Option "msm_blocks" (eg_set_option): >0 forces that k', -1 forces k.    */
/*                                                                       */
/* Covering designs.  The complete family of C(k',d) masks is one way to  */
/* make every pair within d share a masked key in some unit; any family   */
/* of masked block sets that contains every d-subset of the blocks does   */
/* (each member masks m >= d blocks), with far fewer units at the same    */
/* key width (48 bits, d = 3: 20 units of 26 kept bits from C(11,5,3)     */
/* instead of 35 units of 27 bits from k' = 7).  The plan also probes the */
/* built-in table (eg_msm_design) and returns the plan code               */
/* 10000 + 100 v + m for the design (v blocks, m masked per unit) when it */
/* is the cheapest; such units run through eg_msm_pairs_design.  Option   */
/* "msm_designs" = 0 restricts the plan to complete designs; "msm_blocks" */
/* also accepts a plan code.                                              */
/* --------------------------------------------------------------------- */
size_t eg_msm_plan_workspace(int32_t length, int32_t k, int32_t d);
int eg_msm_plan(const uint64_t *d_codes, int64_t n, int32_t length, int32_t k,
                int32_t d, double oversized_fraction, int32_t *h_k_out,
                double *h_cost, void *d_workspace, size_t workspace_bytes,
                void *stream);
/* Built-in covering design C(v, m, t): writes min(count, capacity) block */
/* masks (bit b = block b masked) to h_masks (may be null) and returns    */
/* the member count, 0 when the table has no such design.                 */
int eg_msm_design(int32_t v, int32_t m, int32_t t, uint64_t *h_masks, int32_t capacity);
/* Output-size estimate for eg_msm_pairs' capacity: pairs with Hamming    */
/* <= d among a strided sample of min(n, 8192) rows of (up to 4 of) the   */
/* replicates, scaled by n(n-1)/(S(S-1)) and replicates/probed.            */
/* h_estimate[0] = point estimate of the raw pairs (all replicates),      */
/* h_estimate[1] = ~4-sigma upper bound (+10 %).  Workspace >= 256 bytes. */
/* Synchronous.                                                           */
int eg_msm_estimate_pairs(const uint64_t *d_codes, int64_t n, int32_t W,
                          int32_t replicates, int32_t d, double *h_estimate,
                          void *d_workspace, size_t workspace_bytes, void *stream);
int eg_msm_pairs(const uint64_t *d_codes, int64_t n, int32_t length,
                 int32_t replicates, const int32_t *h_block_bounds, int32_t k,
                 int32_t d, const int32_t *h_unit_rep, const uint64_t *h_unit_mask,
                 int64_t n_units, uint64_t *d_out_keys, uint16_t *d_out_rep,
                 int64_t capacity, int64_t *h_counts, void *d_workspace,
                 size_t workspace_bytes, void *stream);

/* eg_msm_pairs for the units of a covering design: h_design[n_design]     */
/* (<= 64) is the ordered family of masked block sets every replicate     */
/* runs (each >= d blocks; every d-subset of the k blocks inside a member, */
/* checked); every h_unit_mask must be a member (any subset of the units: */
/* sharding).  A pair is emitted by the FIRST member under which it is    */
/* grouped (the role of the reference's earlier-mask search,              */
/* hamming_join.py:130-141), so the emitted set is again exactly          */
/* {(i,j): popcount(c_i^c_j) <= d}.  n_design = 0: eg_msm_pairs.          */
int eg_msm_pairs_design(const uint64_t *d_codes, int64_t n, int32_t length,
                        int32_t replicates, const int32_t *h_block_bounds, int32_t k,
                        int32_t d, const int32_t *h_unit_rep, const uint64_t *h_unit_mask,
                        int64_t n_units, const uint64_t *h_design, int32_t n_design,
                        uint64_t *d_out_keys, uint16_t *d_out_rep, int64_t capacity,
                        int64_t *h_counts, void *d_workspace, size_t workspace_bytes,
                        void *stream);

/* Deferred cross-replicate first-witness rule (pipeline.py:286-314) over  */
/* pairs emitted by eg_msm_pairs with d_out_rep: d_keep[p] = 1 iff the     */
/* pair's Hamming distance exceeds d in every replicate before its own.   */
/* h_new_counts[replicates] receives the survivors per replicate.         */
int eg_xrep_filter(const uint64_t *d_keys, const uint16_t *d_reps, int64_t m,
                   const uint64_t *d_codes, int64_t n, int32_t W, int32_t d,
                   int32_t replicates, uint8_t *d_keep, int64_t *h_new_counts,
                   void *stream);
/* Same, without synchronising: the survivor counts go to device memory   */
/* d_new_counts[replicates] (valid once the stream reaches this point).   */
/* d_keep may be null: the keys of dropped pairs are then overwritten     */
/* with ~0 in place (d_keys must be writable), so that one sort of the    */
/* whole array leaves the sum(d_new_counts) survivors in front -- the     */
/* build's path when few pairs can be dropped (no compaction pass).       */
int eg_xrep_filter_async(const uint64_t *d_keys, const uint16_t *d_reps, int64_t m,
                         const uint64_t *d_codes, int64_t n, int32_t W, int32_t d,
                         int32_t replicates, uint8_t *d_keep, uint64_t *d_new_counts,
                         void *stream);

/* Full-code Hamming filter for pairs enumerated on a code prefix         */
/* (lengths above EG_MAX_LENGTH: the MSM runs on the first 256 bits, a    */
/* superset of the answer): d_keep[p] = popcount over all W words of the  */
/* pair's replicate codes <= d (replicate from d_reps, or 0 when null);   */
/* d_raw_counts[replicates] (device) counts the survivors per replicate.  */
/* Asynchronous.                                                          */
int eg_hamming_filter_async(const uint64_t *d_keys, const uint16_t *d_reps, int64_t m,
                            const uint64_t *d_codes, int64_t n, int32_t W, int32_t d,
                            int32_t replicates, uint8_t *d_keep, uint64_t *d_raw_counts,
                            void *stream);

/* --------------------------------------------------------------------- */
/* Grouped sort of one mask.  Replaces grouped_radix_sort                 */
/* (hamming_join.py:275-297) with the reference's exact permutation: the  */
/* kept bits are chunked chunk_bits wide MSB first (masked_key_table,     */
/* bitpool.py:224-253) and applied last chunk first as stable counting    */
/* passes with buckets in first-seen order (_counting_pass, :52-82).      */
/* d_perm[n] receives the permutation, d_bounds[0..groups] the run        */
/* offsets (groups+1 values), *h_groups the group count.  Synchronous.    */
/* --------------------------------------------------------------------- */
size_t eg_grouped_sort_workspace(int64_t n, int32_t chunk_bits);
int eg_grouped_sort(const uint64_t *d_codes, int64_t n, int32_t length,
                    const int32_t *h_block_bounds, int32_t k, uint64_t mask_bits,
                    int32_t chunk_bits, uint32_t *d_perm, int64_t *d_bounds,
                    int64_t *h_groups, void *d_workspace, size_t workspace_bytes,
                    void *stream);

/* --------------------------------------------------------------------- */
/* Cross-replicate first witness for externally supplied pair sets.       */
/* Replaces dedup_across_replicates' inner loop (pipeline.py:104-146):    */
/* d_keep[m] = 1 iff popcount over every pool g in d_pools[0..n_pools)    */
/* exceeds d.  d_pools is a device array of device pointers.              */
/* --------------------------------------------------------------------- */
int eg_first_witness(const uint64_t *d_keys, int64_t m,
                     const uint64_t *const *d_pools, int32_t n_pools, int32_t W,
                     int32_t d, uint8_t *d_keep, void *stream);

/* --------------------------------------------------------------------- */
/* Radix sort of uint64 keys (optionally carrying uint32 values).         */
/* Replaces the final np.lexsort of enumerate_pairs (hamming_join.py:     */
/* 369-375) and filter_exact (pipeline.py:222).  Sorts the low key_bits   */
/* bits; result lands back in d_keys/d_vals.                              */
/* --------------------------------------------------------------------- */
size_t eg_sort_workspace(int64_t m, int with_values);
int eg_sort_keys(uint64_t *d_keys, uint32_t *d_vals, int64_t m, int32_t key_bits,
                 void *d_workspace, size_t workspace_bytes, void *stream);
/* Pair keys (i << 32 | j) with i, j < n: only the populated digits of both
 * halves are sorted.  Workspace: eg_sort_workspace(m, 0). */
int eg_sort_pair_keys(uint64_t *d_keys, int64_t m, int64_t n, void *d_workspace,
                      size_t workspace_bytes, void *stream);

/* --------------------------------------------------------------------- */
/* Stable compaction of keys by a byte flag (keeps input order).          */
/* --------------------------------------------------------------------- */
/* Merge of sorted runs (the ranks' sorted edge lists in the multi-GPU    */
/* build): d_keys[h_offsets[0] .. h_offsets[runs]) holds `runs` ascending */
/* runs (run r = [h_offsets[r], h_offsets[r+1])) with optional 64-bit     */
/* payloads d_vals (distance bits); on return the whole range is sorted,  */
/* stably (merge path, log2(runs) rounds).  Asynchronous.                 */
/* --------------------------------------------------------------------- */
size_t eg_merge_runs_workspace(int64_t m, int with_values);
int eg_merge_runs(uint64_t *d_keys, uint64_t *d_vals, const int64_t *h_offsets,
                  int32_t runs, void *d_workspace, size_t workspace_bytes, void *stream);

/* --------------------------------------------------------------------- */
size_t eg_compact_workspace(int64_t m);
int eg_compact_keys(const uint64_t *d_keys, const uint8_t *d_flags, int64_t m,
                    uint64_t *d_out, int64_t *h_count, void *d_workspace,
                    size_t workspace_bytes, void *stream);

/* --------------------------------------------------------------------- */
/* Exact verification.  Replaces filter_exact (pipeline.py:183-223).      */
/* Cosine: dist = clip(1 - dot/(n_i n_j), 0, 2); Euclidean: ||x_i-x_j||.  */
/* fp64 accumulation in a fixed order per pair (per-pair deterministic).  */
/* Keeps dist <= eps; output keeps the input order (stable), so sorted    */
/* candidate keys give sorted edges.  h_count receives the edge count.    */
/* Keys must satisfy i, j < n (checked; EG_ERR_ARG on violation).         */
/* --------------------------------------------------------------------- */
size_t eg_verify_workspace(int64_t m);
int eg_verify(const void *d_x, int x_is_f64, int64_t n, int32_t dim,
              const double *d_norms, const uint64_t *d_keys, int64_t m,
              int32_t metric, double eps, uint64_t *d_out_keys, double *d_out_dist,
              int64_t *h_count, void *d_workspace, size_t workspace_bytes,
              void *stream);

/* --------------------------------------------------------------------- */
/* Exhaustive oracle on the GPU.                   */
/* eg_bf_cosine_candidates replaces the all-pairs product of              */
/* exact.brute_force_cosine (exact.py:57-95): every pair i < j whose      */
/* cosine distance can be <= eps (fp16 tensor-core screen with a          */
/* certified margin) as keys (i << 32) | j, unordered.  The exact fp64    */
/* decision and distance come from eg_verify on the sorted keys.          */
/* h_count receives the candidate count; when it exceeds cap only cap     */
/* keys were written (call again with a larger buffer).  dim <= 512.      */
/* eg_bf_hamming replaces exact.brute_force_hamming (exact.py:98-121):    */
/* all pairs i < j with popcount(c_i ^ c_j) <= d (words <= 4), unordered, */
/* same capacity contract.  Both synchronise the stream before return.    */
/* --------------------------------------------------------------------- */
size_t eg_bf_cosine_workspace(int64_t n, int32_t dim);
int eg_bf_cosine_candidates(const void *d_x, int x_is_f64, int64_t n, int32_t dim,
                            const double *d_norms, double eps, uint64_t *d_keys,
                            int64_t cap, int64_t *h_count, void *d_workspace,
                            size_t workspace_bytes, void *stream);
size_t eg_bf_hamming_workspace(void);
int eg_bf_hamming(const uint64_t *d_codes, int64_t n, int32_t words, int32_t d,
                  uint64_t *d_keys, int64_t cap, int64_t *h_count, void *d_workspace,
                  size_t workspace_bytes, void *stream);

/* --------------------------------------------------------------------- */
/* Edge-list text.  Replaces the formatting loop of */
/* io.write_edges (io.py:145-158): for m <= EG_FORMAT_MAX_EDGES edges      */
/* (keys (i << 32) | j, fp64 distances) writes "i j d.ddddddddd\n" lines   */
/* (%.9f, round-half-even on the exact binary value, as Python's float     */
/* formatting) back to back into d_out; *h_bytes = total bytes.  Returns   */
/* EG_ERR_CAPACITY (with *h_bytes set, nothing written) if out_cap is too  */
/* small, EG_ERR_UNSUPPORTED if |dist| * 1e9 >= 2^63.  Synchronises.       */
/* --------------------------------------------------------------------- */
#define EG_FORMAT_MAX_EDGES (1ll << 26)
size_t eg_format_edges_workspace(int64_t m);
int eg_format_edges(const uint64_t *d_keys, const double *d_dist, int64_t m, char *d_out,
                    int64_t out_cap, int64_t *h_bytes, void *d_workspace,
                    size_t workspace_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* EPSGRAPH_B200_H */
