// The local join's host side (plan, class launches, the C entries) and the fp32, K <= 32
// kernel family; the kernels themselves are in join_impl.cuh (see its header comment).
#include "join_impl.cuh"

namespace knnd {

int join_dispatch_f32k1(const Plan &P, int i, const JoinParams &p, const int32_t *lists, const int32_t *counts,
                        int64_t m, int32_t *slabs, cudaStream_t st) {
  return dispatch_class_family<FAM_F32K1>(P, i, p, lists, counts, m, slabs, st);
}

static int dispatch_class(const Plan &P, int i, const JoinParams &p, const int32_t *lists, const int32_t *counts,
                          int64_t m, int32_t *slabs, cudaStream_t st) {
  if (p.scr != SCR_F32) return join_dispatch_q23(P, i, p, lists, counts, m, slabs, st);
  return P.kpl == 1 ? join_dispatch_f32k1(P, i, p, lists, counts, m, slabs, st)
                    : join_dispatch_f32k2(P, i, p, lists, counts, m, slabs, st);
}

}  // namespace knnd

using namespace knnd;

extern "C" {

size_t knnd_local_join_workspace_bytes(int64_t n, int32_t d, int32_t k, int64_t row_lo, int64_t row_hi,
                                       int32_t max_indeg) {
  if (k < 2 || k > 64 || d < 1 || row_hi < row_lo || max_indeg < 0 || n < 1) return 0;
  return make_plan(n, row_hi - row_lo, d, k, max_indeg).total;
}

}  // extern "C"

// shared by the KL and L2 entries: validation that does not depend on the
// metric, the plan, and the class launches
static int join_run(const char *who, JoinParams &p, int64_t n, int32_t dplan, int32_t k, int64_t row_lo,
                    int64_t row_hi, int32_t max_indeg, void *ws, size_t ws_bytes, void *stream,
                    void *side_stream) {
  const int32_t d = p.d, ld32 = p.ld;
  KNND_CHECK_ARG(p.F && p.indptr && p.indices && p.out_ids && p.tally, "%s: null pointer", who);
  KNND_CHECK_ARG(n >= 2 && d >= 1, "%s: bad shape n=%lld d=%d", who, (long long)n, d);
  KNND_CHECK_ARG(ld32 >= dplan && ld32 % 4 == 0, "%s: ld32=%d must be >= %d and a multiple of 4", who, ld32, dplan);
  KNND_CHECK_ARG(0 <= row_lo && row_lo <= row_hi && row_hi <= n, "%s: bad row range", who);
  KNND_CHECK_ARG(n * (int64_t)k < ((int64_t)1 << 31), "%s: n*K must be < 2^31", who);
  KNND_CHECK_ARG(max_indeg >= 0 && max_indeg <= n, "%s: bad max_indeg %d", who, max_indeg);
  if (k < 2 || k > 64) {
    set_error("%s: K=%d unsupported (2..64)", who, k);
    return KNND_EUNSUPPORTED;
  }
  const int64_t m = row_hi - row_lo;
  if (m == 0) return KNND_OK;
  if (((int64_t)k + max_indeg) * (k + 1) > ((int64_t)1 << 29)) {
    set_error("%s: pre-dedup bound (K+%d)(K+1) too large", who, max_indeg);
    return KNND_EUNSUPPORTED;
  }
  const Plan P = make_plan(n, m, dplan, k, max_indeg);
  if (ws_bytes < P.total || !ws) {
    set_error("%s: workspace %zu < %zu bytes", who, ws_bytes, P.total);
    return KNND_EWORKSPACE;
  }
  cudaStream_t st = as_stream(stream);
  char *w = static_cast<char *>(ws);
  int32_t *lists = reinterpret_cast<int32_t *>(w + P.lists_off);
  int32_t *counts = reinterpret_cast<int32_t *>(w + P.counts_off);
  int32_t *slabs = reinterpret_cast<int32_t *>(w + P.slab_off);
  const int64_t *indptr = p.indptr;
  unsigned long long *tally = p.tally;
  p.lo = row_lo;
  p.n = n;
  p.m = m;
  p.K = k;
  // rigorous bound on |fp32 screen - fp64| relative to sum |x*log y| (+ margin)
  p.band = (float)((ld32 + 8) * 0x1p-24);
  // Q23: three roundings in a weight (x, h, their product), a chain of ceil(NQ / 4)
  // FMAs and two adds per entry — (1 + u)^(ceil(NQ / 4) + 5) - 1, one more u of margin
  if (p.scr != SCR_F32) p.band = (float)((((16 * p.nvq) / 3 + 3) / 4 + 6) * 0x1p-24);

  KNND_CUDA(cudaMemsetAsync(counts, 0, 64, st));
  {
    Lims lims;
    lims.n = P.ncls;
    for (int i = 0; i < P.ncls; ++i) lims.v[i] = P.c[i].lim;
    int64_t blocks = (m + 255) / 256;
    if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
    classify_kernel<<<(unsigned)blocks, 256, 0, st>>>(indptr, m, row_lo, k, lims, lists, counts);
    KNND_LAUNCHED(1);
  }
  // diagnostics: KNND_CLASS_TIMING=1 times each class (synchronising) and prints
  // anchors / comparisons / ms per class to stderr
  const bool timing = getenv("KNND_CLASS_TIMING") != nullptr;
  // The big-table classes (>= 2^14 slots and the hubs) run on the caller's
  // side stream (when one is given), concurrently with the rest: they hold few
  // anchors, each long and latency bound, and serialised their tails left most
  // SMs idle — ~0.1-0.3 ms per round, a 10-15% loss once a rank holds 1/8 of
  // the anchors.  Persistent blocks that find no anchor exit at once, so the
  // other classes fill the machine around the busy ones.  Measured (C3): P = 1
  // +0.5%, the 8-rank projection's join -5.5%; C4 -0.7%.  KNND_SIDE_CLASSES=k
  // overrides (the k biggest classes; 0 = all serial).  The fork / join events
  // live for this call only (destroyed here; CUDA releases them once they
  // complete), so the library keeps no stream or event state.
  const char *nside_s = getenv("KNND_SIDE_CLASSES");
  const int nside_env = nside_s ? atoi(nside_s) : -1;
  int ig = P.ncls;  // classes [ig, ncls) go to the side stream
  if (nside_env >= 0) {
    ig = P.ncls - nside_env;
  } else {
    while (ig - 1 > 0 && (P.c[ig - 1].kind == KIND_GLOBAL || P.c[ig - 1].logH >= 14)) --ig;
  }
  cudaStream_t sst = as_stream(side_stream);
  const bool side = sst != nullptr && sst != st && !timing && ig > 0 && ig < P.ncls;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  if (side) {
    KNND_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    if (cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming) != cudaSuccess) {
      cudaEventDestroy(ev_fork);
      set_error("%s: cudaEventCreate failed", who);
      return KNND_ECUDA;
    }
    int rc = KNND_OK;
    if (cudaEventRecord(ev_fork, st) != cudaSuccess || cudaStreamWaitEvent(sst, ev_fork, 0) != cudaSuccess) {
      set_error("%s: fork to the side stream failed", who);
      rc = KNND_ECUDA;
    }
    for (int i = P.ncls - 1; i >= ig && rc == KNND_OK; --i)
      if (P.c[i].need) rc = dispatch_class(P, i, p, lists, counts, m, slabs, sst);
    if (rc == KNND_OK && cudaEventRecord(ev_join, sst) != cudaSuccess) {
      set_error("%s: join of the side stream failed", who);
      rc = KNND_ECUDA;
    }
    cudaEventDestroy(ev_fork);
    if (rc != KNND_OK) {
      cudaEventDestroy(ev_join);
      return rc;
    }
  }
  // biggest tables first: the few long hub anchors start early
  for (int i = P.ncls - 1; i >= 0; --i) {
    if (!P.c[i].need || (side && i >= ig)) continue;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    unsigned long long t0[4] = {0, 0, 0, 0};
    if (timing) {
      KNND_CUDA(cudaStreamSynchronize(st));
      KNND_CUDA(cudaMemcpy(t0, tally, sizeof(t0), cudaMemcpyDeviceToHost));
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, st);
    }
    const int rc = dispatch_class(P, i, p, lists, counts, m, slabs, st);
    if (rc) {
      if (side) cudaEventDestroy(ev_join);
      return rc;
    }
    if (timing) {
      cudaEventRecord(e1, st);
      KNND_CUDA(cudaStreamSynchronize(st));
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long t1[4];
      int cnt[MAXCLS + 1];
      KNND_CUDA(cudaMemcpy(t1, tally, sizeof(t1), cudaMemcpyDeviceToHost));
      KNND_CUDA(cudaMemcpy(cnt, counts, sizeof(int) * P.ncls, cudaMemcpyDeviceToHost));
      const unsigned long long u = t1[0] - t0[0];
      fprintf(stderr, "knnd class %d kind %d logH %d: %d anchors, %llu comparisons, %.3f ms, %.3e/s, %llu rows ranked in fp64\n",
              i, P.c[i].kind, P.c[i].logH, cnt[i], u, ms, ms > 0 ? u / (ms * 1e-3) : 0.0, t1[3] - t0[3]);
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
  }
  if (side) {  // the hub rows are part of this call's output
    const cudaError_t e = cudaStreamWaitEvent(st, ev_join, 0);
    cudaEventDestroy(ev_join);
    KNND_CUDA(e);
  }
  return KNND_OK;
}

// peer tables of the fused exchange (host array of device pointers)
static int set_peers(JoinParams &p, const char *who, int32_t *const *peer_tables, int32_t npeers) {
  KNND_CHECK_ARG(npeers >= 0 && npeers <= KNND_MAX_PEERS, "%s: npeers=%d outside 0..%d", who, npeers,
                 KNND_MAX_PEERS);
  KNND_CHECK_ARG(npeers == 0 || peer_tables, "%s: null peer_tables", who);
  p.npeers = npeers;
  for (int q = 0; q < npeers; ++q) {
    KNND_CHECK_ARG(peer_tables[q], "%s: null peer table %d", who, q);
    p.peers[q] = peer_tables[q];
  }
  return KNND_OK;
}

extern "C" {

int knnd_local_join_peers(const double *points, const float *log32, const double *log64, const double *xlogx,
                          int64_t n, int32_t d, int32_t ld32, const int32_t *friends, int32_t k,
                          const int64_t *indptr, const int32_t *indices, int64_t row_lo, int64_t row_hi,
                          int32_t max_indeg, int32_t *out_ids, double *out_kl, int32_t *out_ucount,
                          unsigned long long *tally, const float *bound_in, float *bound_out, void *ws,
                          size_t ws_bytes, uint32_t flags, int32_t *const *peer_tables, int32_t npeers,
                          const void *qrows, const float *q_h, int32_t q_ld, void *stream, void *side_stream) {
  KNND_CHECK_ARG(points && log32 && log64 && xlogx, "knnd_local_join: null pointer");
  JoinParams p{};
  p.points = points;
  p.log32 = log32;
  p.log64 = log64;
  p.xlogx = xlogx;
  p.F = friends;
  p.indptr = indptr;
  p.indices = indices;
  p.out_ids = out_ids;
  p.out_kl = out_kl;
  p.out_ucount = out_ucount;
  p.tally = tally;
  p.d = d;
  p.ld = ld32;
  p.nonpos = (flags & KNND_JOIN_NONPOS_LOG) ? 1 : 0;
  p.bound_in = bound_in;
  p.bound_out = bound_out;
  p.metric = METRIC_KL;
  p.d64 = d;
  p.pstride = d;
  p.aside32 = nullptr;
  if (qrows) {  // the 23-bit fixed-point screen (knnd_kl_q23_prepare)
    KNND_CHECK_ARG(q_h && (q_ld == 16 || q_ld == 32 || q_ld == 48 || q_ld == 64 || q_ld == 160) && q_ld >= 3 * d &&
                       k <= 32,
                   "knnd_local_join: the q23 screen needs q_h, rows of 16, 32, 48, 64 or 160 bytes (>= 3 d) and K <= 32 "
                   "(q_ld=%d d=%d K=%d)",
                   q_ld, d, k);
    p.log32 = reinterpret_cast<const float *>(qrows);
    p.qh = q_h;
    p.nvq = q_ld / 16;
    p.scr = SCR_Q23;
  }
  if (int rc = set_peers(p, "knnd_local_join", peer_tables, npeers)) return rc;
  return join_run("knnd_local_join", p, n, d, k, row_lo, row_hi, max_indeg, ws, ws_bytes, stream, side_stream);
}

int knnd_local_join(const double *points, const float *log32, const double *log64, const double *xlogx, int64_t n,
                    int32_t d, int32_t ld32, const int32_t *friends, int32_t k, const int64_t *indptr,
                    const int32_t *indices, int64_t row_lo, int64_t row_hi, int32_t max_indeg, int32_t *out_ids,
                    double *out_kl, int32_t *out_ucount, unsigned long long *tally, const float *bound_in,
                    float *bound_out, void *ws, size_t ws_bytes, uint32_t flags, void *stream) {
  return knnd_local_join_peers(points, log32, log64, xlogx, n, d, ld32, friends, k, indptr, indices, row_lo, row_hi,
                               max_indeg, out_ids, out_kl, out_ucount, tally, bound_in, bound_out, ws, ws_bytes, flags,
                               nullptr, 0, nullptr, nullptr, 0, stream, nullptr);
}

int knnd_l2_local_join_peers(const float *anchor32, const float *cand32, const double *rows64, const double *sq64,
                             int64_t n, int32_t d, int32_t ld32, double maxnorm, const int32_t *friends, int32_t k,
                             const int64_t *indptr, const int32_t *indices, int64_t row_lo, int64_t row_hi,
                             int32_t max_indeg, int32_t *out_ids, double *out_d2, int32_t *out_ucount,
                             unsigned long long *tally, const float *bound_in, float *bound_out, void *ws,
                             size_t ws_bytes, int32_t *const *peer_tables, int32_t npeers, const void *qrows,
                             const float *q_h, int32_t q_ld, void *stream, void *side_stream) {
  KNND_CHECK_ARG(anchor32 && cand32 && rows64 && sq64, "knnd_l2_local_join: null pointer");
  JoinParams p{};
  p.points = rows64;  // the anchor's fp64 coordinates: the first d entries of its row
  p.log32 = cand32;
  p.log64 = rows64;
  p.xlogx = sq64;
  p.F = friends;
  p.indptr = indptr;
  p.indices = indices;
  p.out_ids = out_ids;
  p.out_kl = out_d2;
  p.out_ucount = out_ucount;
  p.tally = tally;
  p.d = d;
  p.ld = ld32;
  p.nonpos = 0;
  p.bound_in = bound_in;
  p.bound_out = bound_out;
  p.metric = METRIC_L2;
  p.d64 = d + 1;
  p.pstride = d + 1;
  p.aside32 = anchor32;
  p.slack = (float)((d + 4) * 0x1p-53 * 4.0 * maxnorm * maxnorm);
  if (qrows) {  // the 23-bit fixed-point screen over (v - mu, |v - mu|^2) (knnd_kl_q23_prepare on those columns)
    KNND_CHECK_ARG(q_h && (q_ld == 32 || q_ld == 48 || q_ld == 64) && q_ld >= 3 * (d + 1) && k <= 32,
                   "knnd_l2_local_join: the q23 screen needs q_h, rows of 32, 48 or 64 bytes (>= 3 (d + 1)) "
                   "and K <= 32 (q_ld=%d d=%d K=%d)",
                   q_ld, d, k);
    p.log32 = reinterpret_cast<const float *>(qrows);
    p.qh = q_h;
    p.nvq = q_ld / 16;
    p.scr = SCR_Q23L2;
  }
  if (int rc = set_peers(p, "knnd_l2_local_join", peer_tables, npeers)) return rc;
  return join_run("knnd_l2_local_join", p, n, d + 1, k, row_lo, row_hi, max_indeg, ws, ws_bytes, stream,
                  side_stream);
}

int knnd_l2_local_join(const float *anchor32, const float *cand32, const double *rows64, const double *sq64,
                       int64_t n, int32_t d, int32_t ld32, double maxnorm, const int32_t *friends, int32_t k,
                       const int64_t *indptr, const int32_t *indices, int64_t row_lo, int64_t row_hi,
                       int32_t max_indeg, int32_t *out_ids, double *out_d2, int32_t *out_ucount,
                       unsigned long long *tally, const float *bound_in, float *bound_out, void *ws, size_t ws_bytes,
                       void *stream) {
  return knnd_l2_local_join_peers(anchor32, cand32, rows64, sq64, n, d, ld32, maxnorm, friends, k, indptr, indices,
                                  row_lo, row_hi, max_indeg, out_ids, out_d2, out_ucount, tally, bound_in, bound_out,
                                  ws, ws_bytes, nullptr, 0, nullptr, nullptr, 0, stream, nullptr);
}

}  // extern "C"

KNND_CHECK_READER(join, 1)
