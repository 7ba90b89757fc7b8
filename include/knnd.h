/*
 * knnd.h — C ABI of the B200 local-join hot path of comparator K-NN descent
 * (arXiv 2202.00517; reference package `rankdescent`, pure Python/numpy).
 *
 * One shared object, libknnd.so, built for sm_100a.  Every entry point takes
 * plain device pointers, sizes and a CUDA stream (passed as void*), is
 * stream-ordered, allocates no device memory and keeps no state apart from a
 * per-thread last-error string, a launch counter and a memo of launch
 * configurations (per device and kernel: the dynamic-shared-memory limit set
 * and the occupancy at a block shape — host data only, so repeated calls make
 * no attribute or occupancy API calls): streams are the caller's, and the
 * only CUDA objects the library creates are the two fork / join events of one
 * *_local_join_peers call with a side stream, destroyed before that call
 * returns.  The caller (the Python host in
 * paper_2202_00517_b200/, using PyTorch for device buffers) owns all memory.
 * Environment variables read per call (diagnostics / A-B only; results never
 * depend on them): KNND_PLAN, KNND_WLIM, KNND_SIDE_CLASSES, KNND_CLASS_TIMING.
 *
 * Return value: KNND_OK (0) or a negative KNND_E* code; knnd_last_error()
 * then describes the failure.  Errors never fall back to a CPU path.
 *
 * Ids are int32 (n < 2^31, n*K < 2^31).  Tables are row-major.
 *
 * The reference interface each entry replaces is cited as file:line relative
 * to /root/reference/pkg/src/rankdescent/.
 */
#ifndef KNND_H
#define KNND_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KNND_ABI_VERSION 3

enum {
  KNND_OK = 0,
  KNND_EINVAL = -1,       /* bad argument (null pointer, size out of range) */
  KNND_ECUDA = -2,        /* CUDA runtime error (launch / memcpy)           */
  KNND_EWORKSPACE = -3,   /* workspace smaller than *_workspace_bytes()     */
  KNND_EUNSUPPORTED = -4, /* K > 64 or other unsupported shape              */
  KNND_EDEVICE = -5       /* a kernel flagged malformed input (e.g. |U|<K)  */
};

int knnd_abi_version(void);
const char *knnd_last_error(void);
/* Number of kernels this library has launched in this process (all threads). */
unsigned long long knnd_launch_count(void);
/* Checked build only (libknnd_checked.so, compiled with -DKNND_CHECKED): the
 * number of device-side bounds checks that failed since the last call, and
 * the first failure's location (file id * 100000 + line); both are cleared.
 * The product build returns KNND_EUNSUPPORTED (its checks are compiled out).
 * Synchronises with the device. */
int knnd_check_failures(unsigned long long *count, unsigned long long *first);

/*
 * KlRankingSystem.__init__ precompute (similarity.py:87-95):
 *   log64[i,j] = log(points[i,j])                (fp64, n x d)
 *   log32[i,j] = (float)log64[i,j], j < d; 0 for d <= j < ld32   (n x ld32)
 *   xlogx[i]   = sum_j points[i,j] * log64[i,j]  (fp64)
 * ld32 must be a multiple of 4 and >= d (16-byte aligned rows for float4).
 */
int knnd_kl_prepare(const double *points, int64_t n, int32_t d, int32_t ld32,
                    float *log32, double *log64, double *xlogx, void *stream);

/*
 * Exact fp64 scores of `ids` against anchor x — the plugin operator
 * ScoredRankingSystem.batch_scores / KlRankingSystem.batch_scores
 * (core.py:97-103, similarity.py:101-106):
 *   out[i] = xlogx[x] - sum_j log64[ids[i], j] * points[x, j]
 * Each value depends only on (x, ids[i]) (batch independent).
 */
int knnd_batch_scores(const double *points, const double *log64, const double *xlogx,
                      int64_t n, int32_t d, int64_t x, const int32_t *ids, int64_t m,
                      double *out, void *stream);

/*
 * Co-friend CSR for the targets owned by this rank — _transpose_csr
 * (descent.py:151-160), restricted to targets in [row_lo, row_hi):
 *   cofriends(t) = indices[indptr[t-row_lo] : indptr[t-row_lo+1]]
 *               = { s : t in friends[s, :] }     (order within a segment is
 *                                                 unspecified; descent.py
 *                                                 re-sorts via np.unique)
 * indptr has (row_hi-row_lo+1) int64 entries, indices has room for n*k.
 * max_indeg (device int32, may be NULL) receives max segment length.
 */
size_t knnd_csr_workspace_bytes(int64_t n, int32_t k, int64_t row_lo, int64_t row_hi);
int knnd_csr_build(const int32_t *friends, int64_t n, int32_t k, int64_t row_lo,
                   int64_t row_hi, int64_t *indptr, int32_t *indices, int32_t *max_indeg,
                   void *ws, size_t ws_bytes, void *stream);
/* knnd_csr_build that also records counted_event (a cudaEvent_t of the stream's device, nullable)
 * on the stream once *max_indeg is final — after the counting pass, before the scan and the
 * fill: the round driver reads its per-round statistics (descent.py:305-313) behind that event
 * while the rest of the build runs. */
int knnd_csr_build_ev(const int32_t *friends, int64_t n, int32_t k, int64_t row_lo, int64_t row_hi,
                      int64_t *indptr, int32_t *indices, int32_t *max_indeg, void *ws,
                      size_t ws_bytes, void *stream, void *counted_event);

/*
 * The local join for anchors x in [row_lo, row_hi) — _propose_scored
 * (descent.py:230-242) as driven by _propose_block / run_round
 * (descent.py:262-314):
 *   U_x = unique(F(x) + C(x) + F(F(x)) + F(C(x))) minus {x}
 *   out_ids[x-row_lo, :] = the K members of U_x with the smallest
 *                          (score, id), best first, score = batch_scores
 * with fp64-exact ordering (fp32 screening pass + fp64 rescoring of every
 * candidate the screening cannot exclude).
 *   out_kl    (nullable) fp64 scores of out_ids
 *   out_ucount(nullable) |U_x| per anchor
 *   tally[0] += sum |U_x|  (RoundStats.comparisons, descent.py:275)
 *   tally[1] += #rows that differ from friends[x] (order-sensitive,
 *               RoundStats.changed_friend_sets, descent.py:276-277)
 *   tally[2] += #anchors with |U_x| < K (malformed input; must stay 0)
 *   tally[3] += #rows whose order the screen could not certify (ranked in fp64)
 *   (tally is 4 x uint64, device memory, accumulated — the caller zeroes it)
 * max_indeg must be >= the longest CSR segment (from knnd_csr_build).
 * bound_in / bound_out (nullable, row_hi-row_lo floats): a per-row bound kept
 * between rounds — bound_out[x] receives the largest screened (fp32) value
 * among the row written for x; passing it back as bound_in with the table
 * built from those rows lets the next round skip the threshold selection.
 * Use NaN (or NULL) when unknown; a bound from any other table is invalid.
 * flags: KNND_JOIN_NONPOS_LOG when every coordinate of every point is <= 1
 * (all logs <= 0, e.g. simplex data): the screen's error scale
 * sum |x log y| then equals -sum x log y and is not accumulated separately.
 * Results do not depend on flags (only the work does).
 */
#define KNND_JOIN_NONPOS_LOG 1u
#define KNND_MAX_PEERS 15
size_t knnd_local_join_workspace_bytes(int64_t n, int32_t d, int32_t k, int64_t row_lo,
                                       int64_t row_hi, int32_t max_indeg);
int knnd_local_join(const double *points, const float *log32, const double *log64,
                    const double *xlogx, int64_t n, int32_t d, int32_t ld32,
                    const int32_t *friends, int32_t k, const int64_t *indptr,
                    const int32_t *indices, int64_t row_lo, int64_t row_hi,
                    int32_t max_indeg, int32_t *out_ids, double *out_kl,
                    int32_t *out_ucount, unsigned long long *tally, const float *bound_in,
                    float *bound_out, void *ws, size_t ws_bytes, uint32_t flags, void *stream);

/*
 * The local join fused with the table exchange of a row-sharded round
 * (run_round's snapshot semantics, descent.py:282-314, over P ranks; the
 * reference has one process, so this replaces the all-gather the sharded
 * engine would otherwise need after every join).  Identical to
 * knnd_local_join, plus: each row written to out_ids (row x - row_lo of this
 * rank's slice) is also stored at row x of every table in peer_tables[0..npeers)
 * — host array of device pointers to row 0 of the other ranks' (n, k) next
 * tables, mapped into this device's address space (CUDA IPC / symmetric
 * memory over NVLink).  The stores overlap the join; before any rank reads the
 * gathered table, the caller runs a cross-rank barrier on the stream (the
 * kernels end with a system-scope fence).  npeers in 0..KNND_MAX_PEERS.
 * qrows / q_h / q_ld (nullable qrows): screen with the 23-bit fixed-point copy
 * of the log table (knnd_kl_q23_prepare: q_ld = 16, 32, 48, 64 or 160 bytes per row,
 * >= 3 d; K <= 32) instead of log32 — the random row gather sets the join's
 * rate and smaller rows move faster (64-byte rows at d = 20: two aligned
 * sectors in one 128-byte line, against three sectors over 1.5 lines); the
 * error bound is as tight as the fp32 screen's and the fp64 decision is
 * unchanged, so results do not depend on it.
 * side_stream (nullable, a stream of the same device other than `stream`):
 * the few long anchors of the big-table size classes run there, concurrently
 * with the bulk classes on `stream`; the call forks to it and joins back, so
 * all of its work is ordered before later work on `stream`.  NULL runs every
 * class on `stream` (knnd_local_join does that).  Results do not depend on it.
 */
int knnd_local_join_peers(const double *points, const float *log32, const double *log64,
                          const double *xlogx, int64_t n, int32_t d, int32_t ld32,
                          const int32_t *friends, int32_t k, const int64_t *indptr,
                          const int32_t *indices, int64_t row_lo, int64_t row_hi,
                          int32_t max_indeg, int32_t *out_ids, double *out_kl,
                          int32_t *out_ucount, unsigned long long *tally,
                          const float *bound_in, float *bound_out, void *ws, size_t ws_bytes,
                          uint32_t flags, int32_t *const *peer_tables, int32_t npeers,
                          const void *qrows, const float *q_h, int32_t q_ld, void *stream,
                          void *side_stream);

/*
 * The 23-bit fixed-point copy of the log table for the join's q23 screen:
 * per column j, h_j = (max log - min log) / (2^23 - 1) (0 for a constant
 * column), q = round((max log - log64) / h_j) in 0..2^23-1, stored in 3 bytes
 * (little endian) at byte 3 j of a row of row_bytes bytes (a multiple of 16,
 * >= 3 d; padding 0); qh[j] = (float)h_j (row_bytes / 3 floats, 0 past d).
 * |(max log - h_j q) - log| <= h_j / 2.  A table with a non-finite log yields
 * non-finite qh entries: the caller must then keep the fp32 screen.
 * Workspace: knnd_kl_q23_workspace_bytes(d).
 */
size_t knnd_kl_q23_workspace_bytes(int32_t d);
int knnd_kl_q23_prepare(const double *log64, int64_t n, int32_t d, int32_t row_bytes, uint8_t *q23,
                        float *qh, void *ws, size_t ws_bytes, void *stream);

/*
 * Friend clustering rate count — friend_clustering_rate (descent.py:317-338)
 * with the sample (xs, i, j) drawn on the host by the reference's own RNG
 * stream (derive_rng(seed, 3, round), descent.py:330-333, j already shifted):
 *   *out_count = #{ s : y in F(z) or z in F(y) },  y = F[xs,i], z = F[xs,j]
 * out_count is overwritten.  rate = count / s_count.
 */
int knnd_fcc(const int32_t *friends, int64_t n, int32_t k, const int32_t *xs,
             const int32_t *is, const int32_t *js, int32_t s_count, int32_t *out_count,
             void *stream);

/*
 * Initial row ordering — _sort_rows_by_anchor (descent.py:163-174): each row
 * of `draws` (rows row_lo..row_hi-1 of the random K-out table) sorted by
 * (fp64 score, draw position), i.e. a stable argsort on scores.
 * out_kl (nullable) receives the sorted scores.
 */
int knnd_sort_rows(const double *points, const double *log64, const double *xlogx,
                   int64_t n, int32_t d, int32_t k, int64_t row_lo, int64_t row_hi,
                   const int32_t *draws, int32_t *out_ids, double *out_kl, void *stream);

/*
 * The initial random K-out draws on the device, bit-identical to numpy —
 * init_random_kout's first draw (descent.py:194-197):
 *   draws = Generator(PCG64).integers(0, n - 1, size=(n, k), dtype=int64)
 *   draws += draws >= row
 * (state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger) is the PCG64
 * state numpy reports in `bit_generator.state` before the call.
 *   out       int32 (n, k): the draws
 *   consumed  (device uint64) number of 32-bit values taken from the stream
 *             (counting a buffered half), so the caller can advance its numpy
 *             generator and continue the rejection loop (descent.py:198-205)
 *   bad/nbad  (device) rows containing a repeated id, unordered, and their count
 * Requires n - 1 <= 2^32 - 1 and n*k < 2^31.
 */
size_t knnd_random_kout_workspace_bytes(int64_t n, int32_t k);
int knnd_random_kout(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                     int32_t has_uint32, uint32_t uinteger, int64_t n, int32_t k, int32_t *out,
                     uint64_t *consumed, int32_t *bad, int32_t *nbad, void *ws, size_t ws_bytes,
                     void *stream);

/*
 * Exact K nearest neighbours of a set of queries by brute force: row a holds
 * the K smallest (fp64 score, id) over every point y != queries[a] —
 * evaluation.py:83-90 (exact_knn's per-anchor body: s = batch_scores(x);
 * s[x] = inf; _smallest_k(s, K), evaluation.py:53-71).  An fp32 screen of all
 * n candidates keeps those within the rigorous error band of the K-th, which
 * are rescored in fp64.  out_count[a] (device int32 per query) receives the
 * number of candidates kept; a value > cap means row a was NOT written and
 * must be recomputed with cap >= out_count[a].  out_scores (nullable) gets
 * the fp64 scores.  flags: KNND_JOIN_NONPOS_LOG as for the local join.
 * The screen runs on the tensor cores (tcgen05.mma kind::tf32, band widened to
 * the tf32 error); ld32 <= 96 here.
 * Workspace: knnd_exact_knn_workspace_bytes(n, ld32, nq, cap) (the candidate
 * lists and a re-tiled copy of the candidate table).  K in 1..64.
 */
size_t knnd_exact_knn_workspace_bytes(int64_t n, int32_t ld32, int64_t nq, int32_t cap);
int knnd_exact_knn(const double *points, const float *log32, const double *log64,
                   const double *xlogx, int64_t n, int32_t d, int32_t ld32,
                   const int32_t *queries, int64_t nq, int32_t k, int32_t cap,
                   int32_t *out_ids, double *out_scores, int32_t *out_count, void *ws,
                   size_t ws_bytes, uint32_t flags, void *stream);

/*
 * Squared-Euclidean scorer (EuclideanRankingSystem, similarity.py:119-140):
 *   d2(x, y) = max(sq[x] + sq[y] - 2 * sum_j y_j x_j, 0),  sq = einsum("ij,ij->i").
 * Tables (knnd_l2_prepare, from the fp64 vectors, their host-computed squared
 * norms sq64 and a center mu, e.g. the column means):
 *   rows64   (n, d+1) fp64  the vector, then sq
 *   cand32   (n, ld32) fp32 [v - mu, |v - mu|^2, 0 ...]      ld32 >= d+1, % 4 == 0
 *   anchor32 (n, ld32) fp32 [2 (v - mu), -1, 0 ...]
 * The screen -sum anchor32[x] * cand32[y] equals d2(x, y) minus a per-anchor
 * constant, so the same fused join / exact K-NN kernels run both metrics.
 * maxnorm = max_y sqrt(sq[y]) bounds the fp64 rounding of d2 for the screen.
 * Workspace of the L2 join: knnd_local_join_workspace_bytes(n, d + 1, ...).
 */
int knnd_l2_prepare(const double *vectors, const double *sq64, int64_t n, int32_t d, int32_t ld32,
                    const double *center, float *cand32, float *anchor32, double *rows64, void *stream);
int knnd_l2_batch_scores(const double *rows64, const double *sq64, int64_t n, int32_t d, int64_t x,
                         const int32_t *ids, int64_t m, double *out, void *stream);
int knnd_l2_sort_rows(const double *rows64, const double *sq64, int64_t n, int32_t d, int32_t k,
                      int64_t row_lo, int64_t row_hi, const int32_t *draws, int32_t *out_ids,
                      double *out_d2, void *stream);
int knnd_l2_local_join(const float *anchor32, const float *cand32, const double *rows64,
                       const double *sq64, int64_t n, int32_t d, int32_t ld32, double maxnorm,
                       const int32_t *friends, int32_t k, const int64_t *indptr,
                       const int32_t *indices, int64_t row_lo, int64_t row_hi, int32_t max_indeg,
                       int32_t *out_ids, double *out_d2, int32_t *out_ucount,
                       unsigned long long *tally, const float *bound_in, float *bound_out, void *ws,
                       size_t ws_bytes, void *stream);
/* knnd_l2_local_join with the fused table exchange (and side stream) of knnd_local_join_peers.
 * qrows / q_h / q_ld (nullable qrows): the 23-bit fixed-point screen rows, as for the KL join —
 * knnd_kl_q23_prepare run on the n x (d + 1) fp64 table of the cand32 columns (v - mu, |v - mu|^2),
 * q_ld = 32, 48 or 64 >= 3 (d + 1), K <= 32.  The weights 2 (x - mu)_j h_j 2^126 must stay inside fp32's normal
 * range (the caller checks the data's scale). */
int knnd_l2_local_join_peers(const float *anchor32, const float *cand32, const double *rows64,
                             const double *sq64, int64_t n, int32_t d, int32_t ld32,
                             double maxnorm, const int32_t *friends, int32_t k,
                             const int64_t *indptr, const int32_t *indices, int64_t row_lo,
                             int64_t row_hi, int32_t max_indeg, int32_t *out_ids, double *out_d2,
                             int32_t *out_ucount, unsigned long long *tally,
                             const float *bound_in, float *bound_out, void *ws, size_t ws_bytes,
                             int32_t *const *peer_tables, int32_t npeers, const void *qrows,
                             const float *q_h, int32_t q_ld, void *stream, void *side_stream);
int knnd_l2_exact_knn(const float *anchor32, const float *cand32, const double *rows64,
                      const double *sq64, int64_t n, int32_t d, int32_t ld32, double maxnorm,
                      const int32_t *queries, int64_t nq, int32_t k, int32_t cap, int32_t *out_ids,
                      double *out_d2, int32_t *out_count, void *ws, size_t ws_bytes, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* KNND_H */
