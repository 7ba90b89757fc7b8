// K2+K3+K4 — the fused local join (descent.py:230-242 driven by 262-314).
//
// Per anchor x:
//   phase 0  stage S = F(x) ++ C(x) and the anchor row (x32, x64) in smem
//   phase 1  enumerate the (K+c)(K+1) pre-dedup ids  S ++ F(S)  and insert
//            every id != x into an open-addressing hash table in shared
//            memory; the first inserter of an id appends it to the unique
//            list U.  |U| is the reference's `comparisons` (descent.py:275).
//   phase 2  screen: gather the fp32 log row of every y in U into shared
//            memory (cp.async, row-contiguous chunks) and compute
//            ce = -sum x32*log32, ab = sum |x32*log32| (FP32 FFMA).  The fp64
//            cross entropy CE lies within c*ab of ce, c = (ld+8)*2^-24
//            (rigorous: all products of one sign, one rounding of x and of
//            log per term plus the FMA chain).
//   phase 2b T >= the K-th smallest ce.  Then K candidates have CE <= T + c*am
//            (am = max ab), so every exact top-K member has ce <= T + 2*c*am.
//   phase 3  R = { y : ce(y) <= T + 2*c*am }   (|R| >= K, typically K..K+2)
//   phase 4  gather the fp64 log rows of R (cp.async), rescore exactly and
//            keep the K smallest (score, id) — the reference's stable-argsort
//            order — then write the row, |U| and the order-sensitive change flag.
//
// So the output equals ranking all of U by exact fp64 scores, at the gather
// cost of one fp32 row per comparison plus one fp64 row per member of R.
//
// Rows are gathered into shared memory in row-contiguous chunks: a warp
// instruction then touches a few 128 B lines instead of 32 scattered ones —
// with one lane per row the gather is bound by L1TEX wavefronts, not DRAM.
//
// Anchors are binned by their pre-dedup bound P = (K+c)(K+1):
//   W1, W2  one warp per anchor, private smem slab (table of H1 / 2*H1 slots)
//   B       one 256-thread block per anchor, table of up to 2^15 slots in smem
//   L       one 512-thread block per anchor, table in a global-memory slab
#pragma once
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "score.cuh"

namespace knnd {

constexpr int EMPTY = -1;
// the screen's row format (template parameter SCR of the join kernels)
constexpr int SCR_F32 = 0;  // fp32 log rows
constexpr int SCR_Q23 = 1;  // 23-bit fixed point in 3 bytes per entry (knnd_kl_q23_prepare)
constexpr int SCR_Q23L2 = 2;  // the same rows for the Euclidean scorer (signed weights: its own instantiations,
                              // so the KL kernels carry none of its branches — they had cost W1 0.8%)
constexpr int UNR1 = 4;  // pre-dedup ids loaded per thread before inserting

struct JoinParams {
  const double *__restrict__ points;
  const float *__restrict__ log32;
  const double *__restrict__ log64;
  const double *__restrict__ xlogx;
  const int32_t *__restrict__ F;
  const int64_t *__restrict__ indptr;
  const int32_t *__restrict__ indices;
  int32_t *__restrict__ out_ids;
  double *__restrict__ out_kl;
  int32_t *__restrict__ out_ucount;
  unsigned long long *tally;
  int64_t lo;
  int64_t n, m;  // items, own rows (checked build: id and row ranges)
  int d, ld, K;
  float band;
  int nonpos;  // every log coordinate <= 0: sum |x log y| == -sum x log y exactly
  const float *__restrict__ qh;  // Q23 screen: per-column steps h_j (log32 then points at the quantised rows)
  int nvq;                       // Q23: 16-byte chunks per quantised row
  int scr;                       // the screen's row format: SCR_F32 / SCR_Q23
  const float *__restrict__ bound_in;  // per own row: max screened value of the current row (or NaN)
  float *__restrict__ bound_out;       // the same for the row written this round
  // metric (score.cuh): KL, or squared Euclidean (EuclideanRankingSystem, similarity.py:119-140)
  int metric;
  int d64;                               // fp64 row length of log64 (d; d+1 for L2: the vector, then |v|^2)
  int pstride;                           // row stride of `points` (the anchor's fp64 coordinates)
  const float *__restrict__ aside32;     // L2: anchor-side fp32 rows (2(x-mu), -1); KL: null (from points)
  // absolute error bound of the exact fp64 values (0 for KL, whose error is
  // relative and inside `band`; L2: (d+4) 2^-53 (2 maxnorm)^2 >= |fl(d2) - d2|);
  // the screen band of an anchor is 2 (band * am + slack)
  float slack;
  // fused table exchange (knnd_local_join_peers): every written row is also
  // stored at row x of each peer's next table (NVLink peer memory), so the
  // rows reach the other ranks while the join runs — no all-gather afterwards
  int npeers;
  int32_t *peers[KNND_MAX_PEERS];
};

// the row's K ids to every peer table (row x, absolute) — lane i stores id i
__device__ __forceinline__ void store_peers(const JoinParams &p, int64_t x, int i, int id) {
  for (int q = 0; q < p.npeers; ++q) p.peers[q][x * p.K + i] = id;
}

__host__ __device__ inline size_t al16(size_t v) { return (v + 15) & ~(size_t)15; }

// ---------------------------------------------------------------------------
// shared device pieces

__device__ __forceinline__ unsigned hash_slot(int y, unsigned shift) { return ((unsigned)y * 0x9E3779B1u) >> shift; }

// Insert into 4-slot buckets (one int4 read finds a duplicate without atomics;
// a new id CAS-es the first empty slot).  Buckets fill left to right — a CAS
// only ever targets the first slot its reader saw empty, and slots are never
// freed — so the first empty slot is the number of occupied ones (ids >= 0,
// EMPTY = -1: count the sign bits) and a bucket is full iff its last slot is.
__device__ __forceinline__ bool hash_insert_cas(int32_t *table, int y, unsigned shift, unsigned mask) {
  const unsigned bmask = mask >> 2;
  unsigned b = hash_slot(y, shift + 2);
  while (true) {
    asm volatile("" ::: "memory");  // re-read the bucket every pass (other warps insert concurrently)
    const int4 v = reinterpret_cast<const int4 *>(table)[b];
    if ((v.x == y) | (v.y == y) | (v.z == y) | (v.w == y)) return false;
    if (v.w == EMPTY) {
      const int occ = 4 + (v.x >> 31) + (v.y >> 31) + (v.z >> 31) + (v.w >> 31);
      KNND_DCHECK(b * 4 + occ <= mask && occ >= 0 && occ < 4);
      const int prev = atomicCAS(table + b * 4 + occ, EMPTY, y);
      if (prev == EMPTY) return true;
      if (prev == y) return false;
      continue;  // lost the slot to another id: re-read the bucket
    }
    b = (b + 1) & bmask;
  }
}

// UNR1 inserts of one lane with their first probes issued together: the
// bucket reads, then the CAS of every id that saw its bucket without it and
// with a free slot, all predicated (no per-id branches); an id whose CAS lost
// (another id took the slot) or whose bucket was full takes the probing loop.
// Same outcome as UNR1 calls of hash_insert_cas: an id is new exactly once.
__device__ __forceinline__ void hash_insert4(int32_t *table, const int (&id)[UNR1], int x, unsigned shift,
                                             unsigned mask, bool (&nw)[UNR1]) {
  unsigned b[UNR1];
  int4 v[UNR1];
  bool valid[UNR1];
#pragma unroll
  for (int u = 0; u < UNR1; ++u) {
    valid[u] = id[u] >= 0 && id[u] != x;
    b[u] = hash_slot(id[u], shift + 2);
    v[u] = valid[u] ? reinterpret_cast<const int4 *>(table)[b[u]] : make_int4(0, 0, 0, 0);
  }
  int prev[UNR1];
  bool retry[UNR1];
#pragma unroll
  for (int u = 0; u < UNR1; ++u) {
    const int y = id[u];
    const bool found = (v[u].x == y) | (v[u].y == y) | (v[u].z == y) | (v[u].w == y);
    const bool can = valid[u] && !found && v[u].w == EMPTY;
    const int occ = 4 + (v[u].x >> 31) + (v[u].y >> 31) + (v[u].z >> 31) + (v[u].w >> 31);
    KNND_DCHECK(!can || (b[u] * 4 + occ <= mask && occ >= 0 && occ < 4));
    prev[u] = can ? atomicCAS(table + b[u] * 4 + occ, EMPTY, y) : EMPTY;  // EMPTY: no CAS made
    nw[u] = can && prev[u] == EMPTY;
    retry[u] = valid[u] && !found && !nw[u] && prev[u] != y;
  }
  // the retries of a lane run one after the other inside ONE divergent region
  // (lanes with no retry skip it), not as UNR1 regions one after the other: in
  // a pass of 32 x UNR1 ids some lane nearly always loses a slot to another
  // id of the same bucket, and the warp then pays for the longest lane, not
  // for the sum over u of the longest lanes
  unsigned pend = 0;
#pragma unroll
  for (int u = 0; u < UNR1; ++u) pend |= retry[u] ? 1u << u : 0u;
  while (pend) {
    const int u = __ffs(pend) - 1;
    pend &= pend - 1;
    int y = id[0];
#pragma unroll
    for (int q = 1; q < UNR1; ++q) y = u == q ? id[q] : y;
    const bool isnew = hash_insert_cas(table, y, shift, mask);
#pragma unroll
    for (int q = 0; q < UNR1; ++q) nw[q] = u == q ? isnew : nw[q];
  }
}

// warp-aggregated append of `val` (where `take`) to list[*counter ...]
__device__ __forceinline__ void warp_append(bool take, int val, int *counter, int32_t *list, int lane) {
  const unsigned m = __ballot_sync(FULL, take);
  if (m) {
    const int leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(counter, __popc(m));
    base = __shfl_sync(FULL, base, leader);
    if (take) list[base + __popc(m & lanemask_lt())] = val;
  }
}

// issue cp.async copies of the fp32 log rows of ids[0..nrow) into stage
// (row stride ld floats) in 16 B chunks: lane l copies chunk l % nv4 of rows
// l / nv4, l / nv4 + 32 / nv4, ... so each warp instruction covers
// floor(32 / nv4) whole rows (a few 128 B lines)
template <int NV4>
__device__ __forceinline__ void stage_rows_f32(float *stage, const float *__restrict__ log32, const int32_t *ids,
                                               int nrow, int ld_rt, int lane) {
  const int ld = NV4 > 0 ? NV4 * 4 : ld_rt;
  const int nv4 = ld >> 2;
  if (nv4 <= 32) {
    const int rpi = 32 / nv4;
    const int r0 = lane / nv4, part = lane - r0 * nv4;
    if (r0 < rpi) {
      unsigned dst = smem_u32(stage) + (unsigned)(r0 * ld + part * 4) * 4u;
      const unsigned dstep = (unsigned)(rpi * ld) * 4u;
      const float *src = log32 + part * 4;
      for (int r = r0; r < nrow; r += rpi, dst += dstep)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src + (int64_t)ids[r] * ld)
                     : "memory");
    }
  } else {
    for (int r = 0; r < nrow; ++r)
      for (int part = lane; part < nv4; part += 32)
        cp_async16(stage + r * ld + part * 4, log32 + (int64_t)ids[r] * ld + part * 4);
  }
}

// same, with the row ids held in registers: lane r holds ids of row r of the
// batch (nrow <= 32), rows are fetched with a shuffle
template <int NV4, int SLD = NV4 * 4>
__device__ __forceinline__ void stage_rows_f32_reg(float *stage, const float *__restrict__ log32, int idreg,
                                                   int nrow, int lane) {
  constexpr int ld = NV4 * 4;  // source row (floats); SLD: staged row stride
  constexpr int rpi = 32 / NV4;
  const int r0 = lane / NV4, part = lane - r0 * NV4;
  unsigned dst = smem_u32(stage) + (unsigned)(r0 * SLD + part * 4) * 4u;
  const float *src = log32 + part * 4;
  const int iters = (nrow + rpi - 1) / rpi;
  for (int t = 0; t < iters; ++t, dst += rpi * SLD * 4u) {
    const int r = r0 + t * rpi;
    const int y = __shfl_sync(FULL, idreg, r & 31);
    if (r0 < rpi && r < nrow)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src + (int64_t)y * ld) : "memory");
  }
}

// the warp kernel's variant of stage_rows_f32_reg: every lane executes every
// shuffle, the copies are predicated, fixed unrolled iterations (the block
// kernels measured slower with it)
template <int NV4, int SLD = NV4 * 4>
__device__ __forceinline__ void stage_rows_f32_reg_full(float *stage, const float *__restrict__ log32, int idreg,
                                                        int nrow, int lane) {
  constexpr int ld = NV4 * 4;  // source row (floats); SLD: staged row stride
  constexpr int rpi = 32 / NV4;
  constexpr int ITERS = (32 + rpi - 1) / rpi;  // nrow <= 32: a fixed, fully unrolled count
  const int r0 = lane / NV4, part = lane - r0 * NV4;
  const unsigned dst = smem_u32(stage) + (unsigned)(r0 * SLD + part * 4) * 4u;
  const float *src = log32 + part * 4;
  const bool lane_on = r0 < rpi;
#pragma unroll
  for (int t = 0; t < ITERS; ++t) {
    const int r = r0 + t * rpi;
    const int y = __shfl_sync(FULL, idreg, r & 31);
    if (t * rpi < nrow && lane_on && r < nrow)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + (unsigned)(t * rpi * SLD * 4)),
                   "l"(src + (int64_t)y * ld)
                   : "memory");
  }
}

// ce = -sum x*l and ab = sum |x*l| of one staged row (left to right).  With
// nonpos (all logs <= 0) every term of ab equals the term of ce, so ab == ce
// bit for bit and only one accumulator is needed.
template <int NV4>
__device__ __forceinline__ void screen_row(const float *row, const float *x32, int ld, int nonpos, float &ce,
                                           float &ab) {
  const float4 *r4 = reinterpret_cast<const float4 *>(row);
  const float4 *x4 = reinterpret_cast<const float4 *>(x32);
  const int nv4 = NV4 > 0 ? NV4 : (ld >> 2);
  float a = 0.f, b = 0.f;
  if (nonpos) {
#pragma unroll
    for (int q = 0; q < (NV4 > 0 ? NV4 : 64); ++q) {
      if (NV4 == 0 && q >= nv4) break;
      const float4 xv = x4[q];
      const float4 l = r4[q];
      a = fmaf(-xv.x, l.x, a);
      a = fmaf(-xv.y, l.y, a);
      a = fmaf(-xv.z, l.z, a);
      a = fmaf(-xv.w, l.w, a);
    }
    ce = a;
    ab = a;
    return;
  }
#pragma unroll
  for (int q = 0; q < (NV4 > 0 ? NV4 : 64); ++q) {
    if (NV4 == 0 && q >= nv4) break;
    const float4 xv = x4[q];
    const float4 l = r4[q];
    a = fmaf(-xv.x, l.x, a);
    a = fmaf(-xv.y, l.y, a);
    a = fmaf(-xv.z, l.z, a);
    a = fmaf(-xv.w, l.w, a);
    b = fmaf(fabsf(xv.x), fabsf(l.x), b);
    b = fmaf(fabsf(xv.y), fabsf(l.y), b);
    b = fmaf(fabsf(xv.z), fabsf(l.z), b);
    b = fmaf(fabsf(xv.w), fabsf(l.w), b);
  }
  ce = a;
  ab = b;
}

// same with the anchor row held in registers (warp kernel, compile-time width)
template <int NV4>
__device__ __forceinline__ void screen_row_reg(const float *row, const float4 (&xr)[NV4], int nonpos, float &ce,
                                               float &ab) {
  const float4 *r4 = reinterpret_cast<const float4 *>(row);
  float a = 0.f, b = 0.f;
  if (nonpos) {
    // four independent chains (the error bound holds for any order of same-sign terms)
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
    for (int q = 0; q < NV4; ++q) {
      const float4 l = r4[q];
      a0 = fmaf(-xr[q].x, l.x, a0);
      a1 = fmaf(-xr[q].y, l.y, a1);
      a2 = fmaf(-xr[q].z, l.z, a2);
      a3 = fmaf(-xr[q].w, l.w, a3);
    }
    a = (a0 + a1) + (a2 + a3);
    ce = a;
    ab = a;
    return;
  }
#pragma unroll
  for (int q = 0; q < NV4; ++q) {
    const float4 l = r4[q];
    a = fmaf(-xr[q].x, l.x, a);
    a = fmaf(-xr[q].y, l.y, a);
    a = fmaf(-xr[q].z, l.z, a);
    a = fmaf(-xr[q].w, l.w, a);
    b = fmaf(fabsf(xr[q].x), fabsf(l.x), b);
    b = fmaf(fabsf(xr[q].y), fabsf(l.y), b);
    b = fmaf(fabsf(xr[q].z), fabsf(l.z), b);
    b = fmaf(fabsf(xr[q].w), fabsf(l.w), b);
  }
  ce = a;
  ab = b;
}

// ---------------------------------------------------------------------------
// The 23-bit fixed-point screen (Q23: rows of 3 bytes per entry, 16 * NCH bytes
// per row — 64 B at d = 20 instead of 80: two aligned sectors and one 128-B
// line per row instead of three sectors over 1.5 lines; the random row gather
// sets the join's rate, tools/row_probe.cu).  knnd_kl_q23_prepare stores, per
// column j, q = round((Lmax_j - log y_j) / h_j) < 2^23, h_j = range_j / (2^23 - 1),
// little endian.  One byte permute per entry builds the float whose bit
// pattern is q (top byte 0 by replicating the sign of q's high byte, which is
// 0): the denormal F_j = q_j 2^-149.  With w_j = x_j h_j 2^126 the screened
// value v = sum_j w_j F_j = 2^-23 sum_j x_j h_j q_j equals
// 2^-23 (ce + sum_j x_j Lmax_j) up to
//   quantisation            2^-23 A1 / 2,  A1 = sum_j x_j h_j   (|q - exact| <= 1/2)
//   fp32 weights and FMAs   (ceil(NQ / 4) + 6) 2^-24 v           (every term >= 0: x_j > 0)
// — the fp32 screen's error model (relative band on max v, plus an absolute
// slack), so the threshold / certification rules are shared with it and the
// fp64 ranking is the only second tier.
template <int NCH>
struct Q23 {
  static constexpr int NQ = (16 * NCH) / 3;  // entries a row of NCH chunks holds
};

// the anchor's weights; returns the absolute (quantisation) part of its error bound
template <int NCH>
__device__ __forceinline__ float q23_weights(const double *x64, const float *__restrict__ qh, int d,
                                             float (&w)[Q23<NCH>::NQ]) {
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < Q23<NCH>::NQ; ++j) {
    const float x = j < d ? (float)x64[j] : 0.f;
    const float h = j < d ? __ldg(qh + j) : 0.f;
    w[j] = (x * h) * 0x1p126f;
    s = fmaf(fabsf(w[j]), 0x1p-75f, s);
  }
  return s * 0x1p-75f * (1.f + 0x1p-9f) + 1e-36f;  // sum_j w_j 2^-150 = 2^-23 A1 / 2
}

// The Euclidean scorer's weights, from its anchor-side fp32 row xs32 = (2 (x - mu), -1)
// over dq = d + 1 columns.  They are signed, so the relative part of the bound cannot
// use a candidate's own value: abq = sum_j |w_j| F_max bounds sum_j |w_j F_j| of every
// candidate (2^-23 sum_j |a_j| range_j).  (A separate function: selecting the source
// per entry inside q23_weights cost the KL kernels 6%.)
template <int NCH>
__device__ __forceinline__ float q23_weights_signed(const float *xs32, const float *__restrict__ qh, int dq,
                                                    float (&w)[Q23<NCH>::NQ], float &abq) {
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < Q23<NCH>::NQ; ++j) {
    const float x = j < dq ? xs32[j] : 0.f;
    const float h = j < dq ? __ldg(qh + j) : 0.f;
    w[j] = (x * h) * 0x1p126f;
    s = fmaf(fabsf(w[j]), 0x1p-75f, s);
  }
  abq = s * 0x1p-51f * (1.f + 0x1p-9f);            // sum_j |w_j| 2^-126
  return s * 0x1p-75f * (1.f + 0x1p-9f) + 1e-36f;  // sum_j |w_j| 2^-150 = 2^-23 A1 / 2
}

// entries [J0, J0 + NJ) of a row from the CW words at word offset W0 (48 bytes
// hold 16 entries exactly, so 3-chunk groups are self-contained)
template <int W0, int CW, int J0, int NJ, int NQ>
__device__ __forceinline__ void q23_group(const float *row, const float (&w)[NQ], float (&a)[4]) {
  const uint4 *r4 = reinterpret_cast<const uint4 *>(row) + W0 / 4;
  unsigned W[CW];
#pragma unroll
  for (int q = 0; q < CW / 4; ++q) {
    const uint4 u = r4[q];
    W[4 * q + 0] = u.x;
    W[4 * q + 1] = u.y;
    W[4 * q + 2] = u.z;
    W[4 * q + 3] = u.w;
  }
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int k = (3 * j) >> 2, o = (3 * j) & 3;
    const unsigned sel = o == 0 ? 0xA210u : o == 1 ? 0xB321u : o == 2 ? 0xC432u : 0xD543u;
    unsigned bits;  // (prmt's sign-replication selector bit is outside __byte_perm's documented range)
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(bits) : "r"(W[k]), "r"(W[k + 1 < CW ? k + 1 : k]), "r"(sel));
    a[(J0 + j) & 3] = fmaf(w[J0 + j], __uint_as_float(bits), a[(J0 + j) & 3]);
  }
}

template <int NCH>
__device__ __forceinline__ float screen_row_q23(const float *row, const float (&w)[Q23<NCH>::NQ]) {
  constexpr int NQ = Q23<NCH>::NQ;
  float a[4] = {0.f, 0.f, 0.f, 0.f};
  if constexpr (NCH <= 4) {
    q23_group<0, 4 * NCH, 0, NQ, NQ>(row, w, a);  // the whole row's words in registers
  } else {
    // wide rows: 48-byte groups of 16 entries (12 words live at a time), then the rest
    static_assert(NCH == 10, "wide q23 rows are built for 10 chunks (d <= 53)");
    q23_group<0, 12, 0, 16, NQ>(row, w, a);
    q23_group<12, 12, 16, 16, NQ>(row, w, a);
    q23_group<24, 12, 32, 16, NQ>(row, w, a);
    q23_group<36, 4, 48, NQ - 48, NQ>(row, w, a);
  }
  return (a[0] + a[1]) + (a[2] + a[3]);
}

// issue cp.async copies of the fp64 log rows of ids[0..nrow) into stage
// (row stride sd doubles, sd odd to spread banks), 8 B chunks
__device__ __forceinline__ void stage_rows_f64(double *stage, int sd, const double *__restrict__ log64,
                                               const int32_t *ids, int nrow, int d, int lane) {
  const int nchunk = nrow * d;
  const int rq = 32 / d, rr = 32 - rq * d;
  int r = lane / d, j = lane - r * d;
  for (int c = lane; c < nchunk; c += 32) {
    cp_async8(stage + r * sd + j, log64 + (int64_t)ids[r] * d + j);
    r += rq;
    j += rr;
    if (j >= d) {
      j -= d;
      ++r;
    }
  }
}

// exact fp64 score from a staged row: same left-to-right FMA order as exact_score
__device__ __forceinline__ double exact_from_row(const double *row, const double *x64, int d, double xl, int metric) {
  double acc = 0.0;
  for (int j = 0; j < d; ++j) acc = fma(x64[j], row[j], acc);
  return finish_score(metric, xl, metric == METRIC_L2 ? row[d] : 0.0, acc);
}

// emit the sorted row (lanes hold the exact top-K), return the change flag
template <int KPL>
__device__ __forceinline__ bool emit_row(const JoinParams &p, const WarpTopK<KeyD, KPL> &ex, int x, int64_t xr,
                                         int lane) {
  const int K = p.K;
  bool diff = false;
#pragma unroll
  for (int q = 0; q < KPL; ++q) {
    const int i = q * 32 + lane;
    if (i < K) {
      const KeyD kq = ex.b[q];
      p.out_ids[xr * K + i] = kq.id;
      store_peers(p, x, i, kq.id);
      if (p.out_kl) p.out_kl[xr * K + i] = kq.s;
      diff |= kq.id != __ldg(p.F + (int64_t)x * K + i);
    }
  }
  return __any_sync(FULL, diff);
}

// phase 4 for one warp: exact rescoring of R = ids[0..nR) through stage64
template <int KPL>
__device__ __forceinline__ void exact_rank(const JoinParams &p, WarpTopK<KeyD, KPL> &ex, const int32_t *ids, int nR,
                                           double *stage64, int rcap, const double *x64, double xl, int lane) {
  const int d = p.d64, sd = d | 1;
  ex.init();
  for (int b = 0; b < nR; b += rcap) {
    const int nrow = min(rcap, nR - b);
    {  // row ids of this batch in registers, fetched once per lane
      const int idreg = lane < nrow ? ids[b + lane] : 0;
      const int nchunk = nrow * d;
      const int rq = 32 / d, rr = 32 - rq * d;
      int r = lane / d, j = lane - (lane / d) * d;
      for (int c0 = 0; c0 < nchunk; c0 += 32) {
        const int y = __shfl_sync(FULL, idreg, r & 31);
        if (c0 + lane < nchunk) cp_async8(stage64 + r * sd + j, p.log64 + (int64_t)y * d + j);
        r += rq;
        j += rr;
        if (j >= d) {
          j -= d;
          ++r;
        }
      }
    }
    cp_async_wait_all();
    __syncwarp();
    KeyD key = KeyD::inf();
    if (lane < nrow) {
      key.s = exact_from_row(stage64 + lane * sd, x64, p.d, xl, p.metric);
      key.id = ids[b + lane];
    }
    __syncwarp();
    if (b == 0)
      ex.first(key, lane);
    else
      ex.insert(key, p.K, lane);
  }
}

// The fp64 fallback of phase 4: rescore R, write the row, return the change
// flag.  (Kept inline: an out-of-line call measured slower — the call saves
// and restores the live registers.)
template <int KPL>
__device__ __forceinline__ bool exact_row(const JoinParams &p, const int32_t *ids, int nR, double *stage64, int rcap,
                                       const double *x64, int x, int64_t xr, int lane) {
  WarpTopK<KeyD, KPL> ex;
  exact_rank<KPL>(p, ex, ids, nR, stage64, rcap, x64, __ldg(p.xlogx + x), lane);
  return emit_row<KPL>(p, ex, x, xr, lane);
}

// Phase 4 without fp64 when the screen already decides the row: sort R (<= 32)
// by (screened value, id); if each of the first K screened values is below the
// next one by more than the error band 2c*am (+ margin), the exact order of the
// top K+1 — hence the row — is the screened order (exact ties are impossible
// at that distance).  Returns false (nothing written) when a gap is too small.
__device__ __forceinline__ bool certify_row(const JoinParams &p, const int32_t *ids, const float *vals, int nR,
                                            float band, int x, int64_t xr, int lane, bool &diff, float &kth) {
  const int K = p.K;
  KeyU key = KeyU::inf();
  if (lane < nR) key = KeyU::make(vals[lane], ids[lane]);
  key = warp_sort32(key, lane);
  const float kv = key.v();
  const float nextv = __shfl_down_sync(FULL, kv, 1);
  const float gap_need = band + fabsf(kv) * 2.5e-7f + 1e-30f;  // (the margin: ~4 ulp for the gap arithmetic)
  const bool need_check = lane < K && lane + 1 < nR;  // nR == K: the set is R itself
  const bool ok = !need_check || (nextv - kv > gap_need);
  if (!__all_sync(FULL, ok)) return false;
  kth = __shfl_sync(FULL, kv, K - 1);
  bool d = false;
  if (lane < K) {
    p.out_ids[xr * K + lane] = key.id();
    store_peers(p, x, lane, key.id());
    d = key.id() != __ldg(p.F + (int64_t)x * K + lane);
  }
  diff = __any_sync(FULL, d);
  return true;
}

// ---------------------------------------------------------------------------
// block-per-anchor kernel (classes B and L)

// R = {k : scores[k] <= theta} (ids, and the screened values of the first 32)
// appended block-wide through the counter *nr
__device__ __forceinline__ void collect_r(const float *scores, const int32_t *list, int U, float theta, int32_t *R,
                                          float *rval, int *nr, int tid, int lane, int G) {
  const int iters = (U + G - 1) / G;
  for (int it = 0; it < iters; ++it) {
    const int k = it * G + tid;
    const float v = k < U ? scores[k] : 0.f;
    const bool take = k < U && v <= theta;
    const unsigned m = __ballot_sync(FULL, take);
    if (m) {
      const int leader = __ffs(m) - 1;
      int b0 = 0;
      if (lane == leader) b0 = atomicAdd(nr, __popc(m));
      b0 = __shfl_sync(FULL, b0, leader);
      if (take) {
        const int r = b0 + __popc(m & lanemask_lt());
        KNND_DCHECK(r < U);  // R (table + H/2) holds up to H/2 >= U ids
        R[r] = list[k];
        if (r < 32) rval[r] = v;
      }
    }
  }
}

struct SmemLayout {
  size_t x32, x64, S, pre, red, hist, rval, stage, table, list, total;  // (x32, x64[, S]) twice, `pre` apart
};

constexpr int NBIN = 256;        // histogram-select buckets per pass
constexpr int LSTAGE_FLOATS = 1536;  // per-warp staging (6 KB, two buffers) in the global-table class
// per-warp staging floats of the global-table class: 6 KB, and at least 2 x 8 rows
__host__ __device__ inline int lstage_floats(int ld) { return LSTAGE_FLOATS > 16 * ld ? LSTAGE_FLOATS : 16 * ld; }

__host__ __device__ inline SmemLayout smem_layout(int G, bool gtab, int d, int ld, int H, int SW, int XT = 0) {
  SmemLayout L;
  size_t o = 64;  // header ints: [0] |U| [1] |R| [2] b1 [3] before1 [4] b2, [8..12] next anchor
  L.x32 = o;
  o = al16(o + (size_t)ld * 4);
  L.x64 = o;
  o = al16(o + (size_t)d * 8);
  L.S = 0;
  if (!gtab) {
    L.S = o;
    o = al16(o + (size_t)SW * 4);
  }
  L.pre = o - L.x32;  // one anchor's inputs; the next anchor's are prefetched into the second copy
  o += L.pre;
  L.red = o;
  o = al16(o + (size_t)(G / 32) * 4 * 4);
  L.hist = o;
  o = al16(o + (size_t)2 * NBIN * 4);
  L.rval = o;  // screened values of the first 32 members of R
  o = al16(o + 32 * 4);
  if (!gtab) {
    L.stage = 0;  // staging uses the (dead) table
    L.table = o;
    o = al16(o + (size_t)(H + XT) * 4);  // XT: extra staging ints past the hash table (launch_join)
    L.list = o;
    o = al16(o + (size_t)(H / 2) * 4);
  } else {
    size_t st = (size_t)(G / 32) * lstage_floats(ld) * 4;
    const size_t st64 = (size_t)32 * ((d + 1) | 1) * 8;  // fp64 rows of d (KL) or d+1 (L2) doubles
    if (st < st64) st = st64;
    L.stage = o;
    o = al16(o + st);
    L.table = L.list = 0;
  }
  L.total = o;
  return L;
}

// warp 0: the bucket holding the target-th smallest (1-based) of hist[0..NBIN)
// -> hdr[slot] = bucket, hdr[slot+1] = count strictly below it
__device__ __forceinline__ void hist_find(const int *hist, int target, int *hdr, int slot, int lane) {
  constexpr int PER = NBIN / 32;
  int c[PER], tot = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    c[i] = hist[lane * PER + i];
    tot += c[i];
  }
  int inc = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += u;
  }
  const unsigned m = __ballot_sync(FULL, inc >= target);
  const int first = m ? __ffs(m) - 1 : 31;
  if (lane == first) {
    int run = inc - tot, b = PER - 1;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      if (run + c[i] >= target) {
        b = i;
        break;
      }
      run += c[i];
    }
    hdr[slot] = lane * PER + b;
    hdr[slot + 1] = run;
  }
}

template <int G, int NV4, int KPL, bool GTAB, bool PF, int SCR>
__global__ void __launch_bounds__(G) join_kernel(JoinParams p, const int32_t *__restrict__ alist,
                                                 const int32_t *__restrict__ acount, int logH, int SW,
                                                 int32_t *__restrict__ gslab, int64_t slab_ints, int XT) {
  constexpr int W = G / 32;
  constexpr bool Q23S = SCR != SCR_F32, Q23SIGNED = SCR == SCR_Q23L2;
  extern __shared__ __align__(16) unsigned char sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int H = 1 << logH;
  const unsigned shift = 32u - (unsigned)logH;
  const SmemLayout L = smem_layout(G, GTAB, p.d, p.ld, H, SW, XT);
  int *hdr = reinterpret_cast<int *>(sm);
  float *red = reinterpret_cast<float *>(sm + L.red);
  int *hist = reinterpret_cast<int *>(sm + L.hist);
  int *hist2 = hist + NBIN;
  float *rval = reinterpret_cast<float *>(sm + L.rval);
  int32_t *slabS = nullptr, *table, *list;
  float *wstage;  // this warp's fp32 staging rows
  double *stage64;
  int wrows, rcap64;
  if constexpr (GTAB) {
    int32_t *slab = gslab + (int64_t)blockIdx.x * slab_ints;
    slabS = slab;
    table = slab + SW;
    list = table + H;
    wrows = min(32, lstage_floats(p.ld) / (2 * (Q23S ? (NV4 | 1) * 4 : p.ld)));  // rows per buffer, two buffers per warp
    wstage = reinterpret_cast<float *>(sm + L.stage) + (size_t)warp * lstage_floats(p.ld);
    stage64 = reinterpret_cast<double *>(sm + L.stage);
    rcap64 = 32;
  } else {
    table = reinterpret_cast<int32_t *>(sm + L.table);
    list = reinterpret_cast<int32_t *>(sm + L.list);
    wrows = 0;  // set per anchor (the staging area follows the scores)
    wstage = nullptr;
    stage64 = reinterpret_cast<double *>(table);  // lower half, free in phase 4
    rcap64 = min(32, (2 * H) / ((p.d64 | 1) * 8));
  }
  const int K = p.K, K1 = K + 1;
  const int d = p.d;
  // staged row stride (floats): the Q23 rows are 16 * NV4 bytes, staged an odd
  // number of 16-byte units apart (64-byte rows 64 bytes apart would make the
  // screen's LDS.128 reads 4-way bank conflicts)
  constexpr int SLD = Q23S ? (NV4 | 1) * 4 : NV4 * 4;
  const int ld = Q23S ? SLD : p.ld;
  const int Gq = G / K1, Gr = G % K1;
  const int s_init = tid / K1, j_init = tid % K1;
  unsigned long long acc_comp = 0, acc_changed = 0, acc_bad = 0, acc_exact = 0;
  const int count = *acount;
  int *cursor = const_cast<int *>(acount) + 8;  // dynamic anchor fetch (zeroed with the counts)
  // The next anchor is fetched one anchor ahead: thread 0 takes its index at the
  // top, loads its id during phase 0 and its CSR range during the dedup, and
  // publishes them in hdr[8..12] after the screen; every thread then cp.asyncs
  // its inputs (S, rows) into the other input buffer while this anchor finishes.
  int64_t *hdr64 = reinterpret_cast<int64_t *>(hdr + 10);
  auto inputs = [&](int b, int32_t *&S, float *&x32, double *&x64) {
    unsigned char *ib = sm + (size_t)b * L.pre;
    x32 = reinterpret_cast<float *>(ib + L.x32);
    x64 = reinterpret_cast<double *>(ib + L.x64);
    S = GTAB ? slabS : reinterpret_cast<int32_t *>(ib + L.S);
  };
  auto prefetch = [&](int b, int xp, int64_t cp0, int cp) {
    int32_t *S;
    float *x32;
    double *x64;
    inputs(b, S, x32, x64);
    if constexpr (!GTAB) {
#pragma unroll 1
      for (int i = tid; i < K + cp; i += G)
        cp_async4(S + i, i < K ? p.F + (int64_t)xp * K + i : p.indices + cp0 + (i - K));
    }
#pragma unroll 1
    for (int i = tid; i < d; i += G) cp_async8(x64 + i, p.points + (int64_t)xp * p.pstride + i);
    if (p.aside32)
#pragma unroll 1
      for (int i = tid; i < p.ld / 4; i += G) cp_async16(x32 + 4 * i, p.aside32 + (int64_t)xp * p.ld + 4 * i);
    cp_async_commit();
  };
  if (tid == 0) {
    const int a0 = atomicAdd(cursor, 1);
    hdr[8] = a0;
    if (a0 < count) {
      const int x0 = alist[a0];
      hdr[9] = x0;
      hdr64[0] = p.indptr[(int64_t)x0 - p.lo];
      hdr[12] = (int)(p.indptr[(int64_t)x0 - p.lo + 1] - hdr64[0]);
    }
  }
  __syncthreads();
  if (hdr[8] < count) prefetch(0, hdr[9], hdr64[0], hdr[12]);
  cp_async_wait_all();
  __syncthreads();  // the first anchor's inputs are in buffer 0
  int pb = 0;

  for (int a = hdr[8]; a < count; a = hdr[8]) {
    const int x = hdr[9];
    const int64_t xr = (int64_t)x - p.lo;
    const int64_t c0 = hdr64[0];
    const int c = hdr[12];
    const int nS = K + c;
    const int total = nS * K1;
    int32_t *S;
    float *x32;
    double *x64;
    inputs(pb, S, x32, x64);
    int an = 0, xn = -1;
    int64_t nc0 = 0, nc1 = 0;
    if (tid == 0) an = atomicAdd(cursor, 1);  // used after phase 0 (latency off the path)
    // global-memory tables are sized per anchor (>= 2P slots, at least 2^15): the
    // slab fits the largest hub, but clearing and probing only what this anchor
    // needs keeps the hub class from sweeping megabytes per anchor
    int Ha = H;
    unsigned sha = shift;
    if constexpr (GTAB) {
      // (a class table below 2^15 slots arises when small K hands the 2^15 shared-memory
      // class to this one: then the whole table, which holds 2 Pmax >= 2 total)
      int la = logH < 15 ? logH : 15;
      while (la < logH && (1 << la) < 2 * total) ++la;
      Ha = 1 << la;
      sha = 32u - (unsigned)la;
      KNND_DCHECK((int64_t)SW + Ha + Ha / 2 <= slab_ints && 2 * total <= Ha);
    }
    KNND_DCHECK(nS <= SW && xr >= 0 && xr < p.m && x >= 0 && x < p.n);
    // (this anchor's inputs are in buffer pb: the end of the previous anchor
    // waited for them before its barrier; hdr[8..12] is rewritten only after
    // the phase-0 barrier below)

    // ---- phase 0: clear table + histograms (S and the anchor rows were prefetched)
    {
      int4 *t4 = reinterpret_cast<int4 *>(table);
      for (int i = tid; i < (Ha >> 2); i += G) t4[i] = make_int4(EMPTY, EMPTY, EMPTY, EMPTY);
    }
    for (int i = tid; i < 2 * NBIN; i += G) hist[i] = 0;
    if constexpr (GTAB)
      for (int i = tid; i < nS; i += G)
        S[i] = i < K ? __ldg(p.F + (int64_t)x * K + i) : __ldg(p.indices + c0 + (i - K));
    if (!p.aside32)
      for (int i = tid; i < p.ld; i += G) x32[i] = i < d ? (float)x64[i] : 0.f;
    if (tid == 0) {
      hdr[0] = 0;
      hdr[1] = 0;
      if (an < count) xn = __ldg(alist + an);
    }
    __syncthreads();

    // ---- phase 1: pre-dedup enumeration + hash dedup (one list atomic per warp
    // and group of UNR1 ids per thread)
    if constexpr (PF) {
      // ids two groups ahead (as in join_warp_kernel): a group's friend-row loads
      // are issued two iterations before its inserts, the select deferred to then
      int s = s_init, j = j_init;
      const int iters = (total + G - 1) / G;
      int fA[UNR1], vA[UNR1], fB[UNR1], vB[UNR1];  // friend id loaded; S value, or -1 (out) / -2 (use friend)
      auto load_group = [&](int (&f)[UNR1], int (&v)[UNR1], int it0) {
#pragma unroll
        for (int u = 0; u < UNR1; ++u) {
          const int e = (it0 + u) * G + tid;
          const bool in = e < total;
          const int sv = S[in ? s : 0];
          f[u] = __ldg(p.F + (int64_t)sv * K + (j > 0 ? j - 1 : 0));
          v[u] = in ? (j == 0 ? sv : -2) : -1;
          s += Gq;
          j += Gr;
          const bool wrap = j >= K1;
          j -= wrap ? K1 : 0;
          s += wrap ? 1 : 0;
        }
      };
      load_group(fA, vA, 0);
      load_group(fB, vB, UNR1);
      for (int it = 0; it < iters; it += UNR1) {
        int id[UNR1];
#pragma unroll
        for (int u = 0; u < UNR1; ++u) {
          id[u] = vA[u] == -2 ? fA[u] : vA[u];
          fA[u] = fB[u];
          vA[u] = vB[u];
        }
        if (it + 2 * UNR1 < iters) {
          load_group(fB, vB, it + 2 * UNR1);
        } else {
#pragma unroll
          for (int u = 0; u < UNR1; ++u) vB[u] = -1;
        }
        bool nw[UNR1];
        hash_insert4(table, id, x, sha, (unsigned)Ha - 1u, nw);
        unsigned m[UNR1];
        int tot = 0;
#pragma unroll
        for (int u = 0; u < UNR1; ++u) {
          m[u] = __ballot_sync(FULL, nw[u]);
          tot += __popc(m[u]);
        }
        if (tot) {
          int b0 = 0;
          if (lane == 0) b0 = atomicAdd(&hdr[0], tot);
          b0 = __shfl_sync(FULL, b0, 0);
          KNND_DCHECK(b0 + tot <= (Ha >> 1));
#pragma unroll
          for (int u = 0; u < UNR1; ++u) {
            KNND_DCHECK(!nw[u] || (id[u] >= 0 && id[u] < p.n));
            if (nw[u]) list[b0 + __popc(m[u] & lanemask_lt())] = id[u];
            b0 += __popc(m[u]);
          }
        }
      }
    } else {
      int s = s_init, j = j_init;
      const int iters = (total + G - 1) / G;
      for (int it = 0; it < iters; it += UNR1) {
        int id[UNR1];
#pragma unroll
        for (int u = 0; u < UNR1; ++u) {
          const int e = (it + u) * G + tid;
          id[u] = -1;
          if (e < total) {
            const int v = S[s];
            id[u] = (j == 0) ? v : __ldg(p.F + (int64_t)v * K + (j - 1));
          }
          s += Gq;
          j += Gr;
          if (j >= K1) {
            j -= K1;
            ++s;
          }
        }
        bool nw[UNR1];
#pragma unroll
        for (int u = 0; u < UNR1; ++u)
          nw[u] = id[u] >= 0 && id[u] != x && hash_insert_cas(table, id[u], sha, (unsigned)Ha - 1u);
        unsigned m[UNR1];
        int tot = 0;
#pragma unroll
        for (int u = 0; u < UNR1; ++u) {
          m[u] = __ballot_sync(FULL, nw[u]);
          tot += __popc(m[u]);
        }
        if (tot) {
          int b0 = 0;
          if (lane == 0) b0 = atomicAdd(&hdr[0], tot);
          b0 = __shfl_sync(FULL, b0, 0);
          KNND_DCHECK(b0 + tot <= (Ha >> 1));
#pragma unroll
          for (int u = 0; u < UNR1; ++u) {
            KNND_DCHECK(!nw[u] || (id[u] >= 0 && id[u] < p.n));
            if (nw[u]) list[b0 + __popc(m[u] & lanemask_lt())] = id[u];
            b0 += __popc(m[u]);
          }
        }
      }
    }
    if (tid == 0 && xn >= 0) {
      nc0 = __ldg(p.indptr + ((int64_t)xn - p.lo));
      nc1 = __ldg(p.indptr + ((int64_t)xn - p.lo + 1));
    }
    __syncthreads();
    const int U = hdr[0];

    // ---- phase 2: fp32 screen, one staged batch of rows per warp at a time
    float *scores = reinterpret_cast<float *>(table);  // the hash table is dead now
    if constexpr (!GTAB) {
      // staging: the table past the scores ([0, U), U <= H/2), split over warps,
      // two buffers per warp
      const int u4 = (U + 3) & ~3;
      const int per_warp_floats = ((H + XT - u4) / W) & ~3;
      wrows = min(32, per_warp_floats / (2 * ld));
      wstage = reinterpret_cast<float *>(table + u4) + (size_t)warp * per_warp_floats;
      KNND_DCHECK(U == 0 || (wrows >= 1 && u4 + (size_t)(warp + 1) * per_warp_floats <= (size_t)(H + XT) &&
                             2 * wrows * ld <= per_warp_floats));
    }
    float mn = __int_as_float(0x7f800000), mx = -mn, am = 0.f;
    float slack = p.slack, abq = 0.f;  // (abq: Q23, Euclidean — the bound on every candidate's sum |w F|)
    float best0 = mn, best1 = mn;  // this lane's two smallest screened values
    float4 xreg[NV4 > 0 && !Q23S ? NV4 : 1];  // the anchor's fp32 row in registers
    float wq[Q23<Q23S ? NV4 : 1>::NQ];  // Q23: the anchor's weights
    if constexpr (!Q23S && NV4 > 0) {
#pragma unroll
      for (int q = 0; q < NV4; ++q) xreg[q] = reinterpret_cast<const float4 *>(x32)[q];
    }
    {
      // this warp's batches: k0 = warp*wrows + it*W*wrows; lane r holds the id of
      // row r of the batch being staged (ids of the batch after that in id_after)
      const int kstep = W * wrows;
      int k0 = warp * wrows;
      int id_next = (k0 < U && lane < wrows && k0 + lane < U) ? list[k0 + lane] : 0;
      int id_after = (k0 + kstep < U && lane < wrows && k0 + kstep + lane < U) ? list[k0 + kstep + lane] : 0;
      if (k0 < U) {
        if constexpr (NV4 > 0)
          stage_rows_f32_reg<NV4, SLD>(wstage, p.log32, id_next, min(wrows, U - k0), lane);
        else
          stage_rows_f32<NV4>(wstage, p.log32, list + k0, min(wrows, U - k0), ld, lane);
        cp_async_commit();
      }
      if constexpr (Q23S) {
        // the anchor's weights, computed while the first batch is in flight; the return value is
        // the quantisation part of the bound, per anchor (+ the Euclidean scorer's fp64 term)
        if constexpr (Q23SIGNED)
          slack = q23_weights_signed<NV4>(x32, p.qh, p.d64, wq, abq) + p.slack * 0x1p-23f;
        else
          slack = q23_weights<NV4>(x64, p.qh, d, wq);
      }
      for (int buf = 0; k0 < U; k0 += kstep, buf ^= 1) {
        const int nrow = min(wrows, U - k0);
        const int k1 = k0 + kstep;
        if (k1 < U) {  // prefetch this warp's next batch into the other buffer
          if constexpr (NV4 > 0)
            stage_rows_f32_reg<NV4, SLD>(wstage + (buf ^ 1) * wrows * ld, p.log32, id_after, min(wrows, U - k1), lane);
          else
            stage_rows_f32<NV4>(wstage + (buf ^ 1) * wrows * ld, p.log32, list + k1, min(wrows, U - k1), ld, lane);
          cp_async_commit();
          const int k2 = k1 + kstep;
          id_after = (lane < wrows && k2 + lane < U) ? list[k2 + lane] : 0;
          cp_async_wait_1();
        } else {
          cp_async_wait_0();
        }
        __syncwarp();
        const int rr = (lane - k0) & 31;  // rotate lanes across batches (k0 is a multiple of wrows)
        const bool in = rr < nrow;
        const int rl = in ? rr : 0;
        float ce, ab;
        if constexpr (Q23S) {
          ce = screen_row_q23<NV4>(wstage + buf * wrows * ld + rl * ld, wq);
          ab = ce;  // KL: every term is >= 0 (the Euclidean scorer replaces the maximum by abq below)
        } else if constexpr (NV4 > 0) {
          screen_row_reg<NV4>(wstage + buf * wrows * ld + rl * ld, xreg, p.nonpos, ce, ab);
        } else {
          screen_row<NV4>(wstage + buf * wrows * ld + rl * ld, x32, ld, p.nonpos, ce, ab);
        }
        if (in) {
          scores[k0 + rl] = ce;
          mn = fminf(mn, ce);
          mx = fmaxf(mx, ce);
          am = fmaxf(am, ab);
          const float lo_ = fminf(best0, ce);
          best1 = fminf(best1, fmaxf(best0, ce));
          best0 = lo_;
        }
        __syncwarp();
      }
    }
    if constexpr (Q23SIGNED) am = abq;  // signed weights: the bound on every candidate's sum |w F|
    if (tid == 0) {  // publish the next anchor (read after the threshold section's barrier)
      hdr[8] = an;
      hdr[9] = xn;
      hdr64[0] = nc0;
      hdr[12] = (int)(nc1 - nc0);
    }
    float T;
    int32_t *R = table + (Ha >> 1);
    bool collected = false;  // R already gathered (by the previous round's bound)
    if constexpr (KPL == 1) {
      // The previous round's bound of this row is a valid T (all current friends
      // are in U); with it, R is gathered in the same pass that counts it, and
      // the threshold networks are skipped when it admits at most 32 candidates.
      const float T0 = p.bound_in ? __ldg(p.bound_in + xr) : __int_as_float(0x7fc00000);
      if (isfinite(T0) && U >= K) {
        float aw = am;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) aw = fmaxf(aw, __shfl_xor_sync(FULL, aw, o));
        if (lane == 0) red[warp * 4 + 2] = aw;
        __syncthreads();  // every warp's scores and max |x log y|
        float ab = 0.f;
#pragma unroll
        for (int w = 0; w < W; ++w) ab = fmaxf(ab, red[w * 4 + 2]);
        const float th0 = T0 + 2.f * (p.band * ab + slack) + fabsf(T0) * 1e-6f;
        collect_r(scores, list, U, th0, R, rval, &hdr[1], tid, lane, G);
        __syncthreads();
        if (hdr[1] <= 32) {
          T = T0;
          am = ab;
          collected = true;
        }
      }
    }
    if (collected) {
    } else if constexpr (KPL == 1) {
      // T >= the K-th smallest ce: each warp takes the 32 smallest of its lanes'
      // two smallest (asc/desc networks + merge), warp 0 merges the W lists
      const KeyF a = warp_sort32(KeyF{best0}, lane);
      const KeyF b = warp_sort32_desc(KeyF{best1}, lane);
      const KeyF m = warp_merge32(kmin(a, b), lane);
      float *mlist = reinterpret_cast<float *>(hist);  // W x 32 floats (histograms unused here)
      mlist[warp * 32 + lane] = m.v;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) am = fmaxf(am, __shfl_xor_sync(FULL, am, o));
      if (lane == 0) red[warp * 4 + 2] = am;
      __syncthreads();
      if (warp == 0) {
        KeyF acc{mlist[lane]};
        for (int w = 1; w < W; ++w) acc = warp_merge32(kmin(acc, KeyF{mlist[w * 32 + 31 - lane]}), lane);
        const float t = acc.shfl(K - 1).v;
        if (lane == 0) {
          reinterpret_cast<float *>(hdr)[2] = t;
          hdr[1] = 0;  // a failed bound pass may have counted
        }
      }
      __syncthreads();
      T = reinterpret_cast<const float *>(hdr)[2];
#pragma unroll
      for (int w = 0; w < W; ++w) am = fmaxf(am, red[w * 4 + 2]);
      if (U < K) T = __int_as_float(0x7f800000);
    } else {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(FULL, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
        am = fmaxf(am, __shfl_xor_sync(FULL, am, o));
      }
      if (lane == 0) {
        red[warp * 4 + 0] = mn;
        red[warp * 4 + 1] = mx;
        red[warp * 4 + 2] = am;
      }
      __syncthreads();
#pragma unroll
      for (int w = 0; w < W; ++w) {
        mn = fminf(mn, red[w * 4 + 0]);
        mx = fmaxf(mx, red[w * 4 + 1]);
        am = fmaxf(am, red[w * 4 + 2]);
      }

      // T >= the K-th smallest ce (two histogram passes)
      T = mx;
      const float range = mx - mn;
      if (U > 2 * K && range > 0.f) {
        const float inv = (float)NBIN / range;
        for (int k = tid; k < U; k += G) {
          const float t = (scores[k] - mn) * inv;
          atomicAdd(&hist[min(NBIN - 1, (int)t)], 1);
        }
        __syncthreads();
        if (warp == 0) hist_find(hist, K, hdr, 2, lane);
        __syncthreads();
        const int b1 = hdr[2], before = hdr[3];
        for (int k = tid; k < U; k += G) {
          const float t = (scores[k] - mn) * inv;
          if (min(NBIN - 1, (int)t) == b1)
            atomicAdd(&hist2[min(NBIN - 1, (int)((t - (float)b1) * (float)NBIN))], 1);
        }
        __syncthreads();
        if (warp == 0) hist_find(hist2, K - before, hdr, 4, lane);
        __syncthreads();
        const int b2 = hdr[4];
        T = mn + ((float)b1 + (float)(b2 + 1) * (1.0f / NBIN)) / inv;
        T += (fabsf(T) + range) * 1e-6f;  // covers the rounding of t and of this line
      }
    }
    const float ebase = p.band * am + slack;  // the screen's error bound at this anchor
    const float theta = T + 2.f * ebase + fabsf(T) * 1e-6f;
    // the error bound among the members of R: a candidate's error is band * its
    // own sum |x log y| (+ slack), which equals its screened value (<= theta)
    // when every term has one sign — usually several times tighter than the
    // bound over all of U, so fewer rows fall back to the fp64 ranking
    const float ebase_r =
        (!Q23SIGNED && (Q23S || (p.metric == METRIC_KL && p.nonpos))) ? p.band * fminf(am, theta) + slack : ebase;
    if (hdr[8] < count) prefetch(pb ^ 1, hdr[9], hdr64[0], hdr[12]);

    // ---- phase 3: collect every candidate the screen cannot exclude
    if (!collected) {
      collect_r(scores, list, U, theta, R, rval, &hdr[1], tid, lane, G);
      __syncthreads();
    }
    const int nR = hdr[1];

    // ---- phase 4: exact fp64 ranking of R, output (warp 0)
    if (warp == 0) {
      bool diff;
      float kth = theta;  // every member of the new row has a screened value <= theta
      if (!(KPL == 1 && p.out_kl == nullptr && nR <= 32 &&
            certify_row(p, R, rval, nR, 2.f * ebase_r, x, xr, lane, diff, kth))) {
        diff = exact_row<KPL>(p, R, nR, stage64, rcap64, x64, x, xr, lane);
        ++acc_exact;
      }
      if (p.bound_out && lane == 0) p.bound_out[xr] = kth;
      if (lane == 0) {
        acc_comp += (unsigned long long)U;
        acc_changed += diff ? 1ull : 0ull;
        acc_bad += (U < K) ? 1ull : 0ull;
        if (p.out_ucount) p.out_ucount[xr] = U;
      }
    }
    cp_async_wait_all();  // the next anchor's inputs (prefetched into the other buffer)
    __syncthreads();
    pb ^= 1;
  }
  cp_async_wait_all();
  if (p.npeers) __threadfence_system();  // peer rows performed before the caller's cross-rank barrier
  if (tid == 0) {
    if (acc_comp) atomicAdd(&p.tally[0], acc_comp);
    if (acc_changed) atomicAdd(&p.tally[1], acc_changed);
    if (acc_bad) atomicAdd(&p.tally[2], acc_bad);
    if (acc_exact) atomicAdd(&p.tally[3], acc_exact);
  }
}

// ---------------------------------------------------------------------------
// warp-per-anchor kernel (classes W1, W2).  One warp owns one anchor and a
// private smem slab, so nothing waits on a block barrier and the unique list
// needs no atomics:
//   * dedup: __match_any_sync elects one lane per distinct id in a batch;
//     leaders claim slots by store-then-verify (a slot keeps the last id
//     written; losers probe on) — no shared-memory atomics
//   * threshold: every lane keeps its 2*KPL smallest screened values; the
//     K-th smallest of that subset is >= the K-th smallest overall, so it is
//     a valid T (tight unless one lane holds > 2*KPL of the best K)

struct WarpSlab {
  size_t x32, x64, S, pre, table, list, total;  // (x32, x64, S) twice, `pre` bytes apart
};

__host__ __device__ inline WarpSlab warp_slab(int d, int ld, int H, int SW, int cap) {
  WarpSlab L;
  size_t o = 0;
  L.x32 = o;
  o = al16(o + (size_t)ld * 4);
  L.x64 = o;
  o = al16(o + (size_t)d * 8);
  L.S = o;
  o = al16(o + (size_t)SW * 4);
  L.pre = o;  // one anchor's inputs; the next anchor's are prefetched into the second copy
  o *= 2;
  L.table = o;
  o = al16(o + (size_t)H * 4);
  L.list = o;
  o = al16(o + (size_t)cap * 4);  // the unique list: up to `cap` ids (the class's pre-dedup bound)
  L.total = o;
  return L;
}

// cp.async the inputs of anchor x (S = F(x) then C(x); its fp64 row; for L2 its
// fp32 anchor-side row) into one input buffer of a warp slab
__device__ __forceinline__ void prefetch_anchor(const JoinParams &p, int x, int64_t c0, int c, int32_t *S,
                                                float *x32, double *x64, int lane) {
  const int K = p.K;
#pragma unroll 1
  for (int i = lane; i < K + c; i += 32)
    cp_async4(S + i, i < K ? p.F + (int64_t)x * K + i : p.indices + c0 + (i - K));
#pragma unroll 1
  for (int i = lane; i < p.d; i += 32) cp_async8(x64 + i, p.points + (int64_t)x * p.pstride + i);
  if (p.aside32)
#pragma unroll 1
    for (int i = lane; i < p.ld / 4; i += 32) cp_async16(x32 + 4 * i, p.aside32 + (int64_t)x * p.ld + 4 * i);
  cp_async_commit();
}

template <int NV4, int KPL, bool VF, int SCR>
__global__ void __launch_bounds__(128, 4)
    join_warp_kernel(JoinParams p, const int32_t *__restrict__ alist, const int32_t *__restrict__ acount, int logH,
                     int SW, int cap) {
  constexpr int Q = 2 * KPL;  // per-lane kept screened values
  constexpr bool Q23S = SCR != SCR_F32, Q23SIGNED = SCR == SCR_Q23L2;
  extern __shared__ __align__(16) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int H = 1 << logH;
  const unsigned shift = 32u - (unsigned)logH;
  const WarpSlab L = warp_slab(p.d, p.ld, H, SW, cap);
  unsigned char *base = sm + (size_t)warp * L.total;
  int32_t *table = reinterpret_cast<int32_t *>(base + L.table);
  int32_t *list = reinterpret_cast<int32_t *>(base + L.list);
#ifdef KNND_CHECKED
  {
    unsigned dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    KNND_DCHECK((size_t)(warp + 1) * L.total <= dyn);  // this warp's slab lies inside the launch's smem
  }
#endif
  float *scores = reinterpret_cast<float *>(table);            // phase 2-3: [0, U)
  double *stage64 = reinterpret_cast<double *>(table);         // phase 4: whole table
  const int K = p.K, K1 = K + 1;
  const int d = p.d, sd = p.d64 | 1;
  // staged row stride (floats): the Q23 rows are 16 * NV4 bytes, staged an odd
  // number of 16-byte units apart (64-byte rows 64 bytes apart would make the
  // screen's LDS.128 reads 4-way bank conflicts)
  constexpr int SLD = Q23S ? (NV4 | 1) * 4 : NV4 * 4;
  const int ld = Q23S ? SLD : p.ld;
  const int rcap64 = min(32, (4 * H) / (sd * 8));
  const int Gq = 32 / K1, Gr = 32 % K1;
  const int s_init = lane / K1, j_init = lane % K1;
  unsigned long long acc_comp = 0, acc_changed = 0, acc_bad = 0, acc_exact = 0;
  const int count = *acount;
  int *cursor = const_cast<int *>(acount) + 8;  // dynamic anchor fetch, 4 anchors per atomic
  // The next anchor is known one anchor ahead: its id is loaded when the
  // current one starts, its CSR range after the dedup, and its inputs (S and
  // rows) are cp.async'd into the other input buffer after the screen, so the
  // load chain alist -> indptr -> S -> F(S) is off the critical path.
  auto fetch4 = [&]() {
    int got = 0;
    if (lane == 0) got = atomicAdd(cursor, 4);
    return __shfl_sync(FULL, got, 0);
  };
  int a = fetch4(), a_rem = 3;
  int x = -1, c = 0;
  int64_t c0 = 0;
  int pb = 0;
  if (a < count) {
    x = alist[a];
    c0 = p.indptr[(int64_t)x - p.lo];
    c = (int)(p.indptr[(int64_t)x - p.lo + 1] - c0);
    prefetch_anchor(p, x, c0, c, reinterpret_cast<int32_t *>(base + L.S), reinterpret_cast<float *>(base + L.x32),
                    reinterpret_cast<double *>(base + L.x64), lane);
  }

  while (a < count) {
    int a_nxt;
    if (a_rem > 0) {
      a_nxt = a + 1;
      --a_rem;
    } else {
      a_nxt = fetch4();
      a_rem = 3;
    }
    const int xn = a_nxt < count ? __ldg(alist + a_nxt) : -1;  // consumed after the dedup
    unsigned char *inb = base + (size_t)pb * L.pre;
    float *x32 = reinterpret_cast<float *>(inb + L.x32);
    double *x64 = reinterpret_cast<double *>(inb + L.x64);
    int32_t *S = reinterpret_cast<int32_t *>(inb + L.S);
    const int64_t xr = (int64_t)x - p.lo;
    // the previous round's row bound, loaded now: it is needed after the screen
    const float T0 = p.bound_in ? __ldg(p.bound_in + xr) : __int_as_float(0x7fc00000);
    const int nS = K + c;
    const int total = nS * K1;
    KNND_DCHECK(nS <= SW && xr >= 0 && xr < p.m && x >= 0 && x < p.n);

    // ---- phase 0
    {
      int4 *t4 = reinterpret_cast<int4 *>(table);
      for (int i = lane; i < (H >> 2); i += 32) t4[i] = make_int4(EMPTY, EMPTY, EMPTY, EMPTY);
    }
    cp_async_wait_all();  // this anchor's prefetched inputs
    __syncwarp();
    if (!p.aside32)
      for (int i = lane; i < p.ld; i += 32) x32[i] = i < d ? (float)x64[i] : 0.f;
    __syncwarp();
    float4 xreg[NV4 > 0 && !Q23S ? NV4 : 1];  // the anchor's fp32 row in registers
    float wq[Q23<Q23S ? NV4 : 1>::NQ];  // Q23: the anchor's weights
    float slack = p.slack, abq = 0.f;           // the absolute part of the fp32 / Q23 bound (abq: Euclidean Q23)
    if constexpr (!Q23S && NV4 > 0) {
#pragma unroll
      for (int q = 0; q < NV4; ++q) xreg[q] = reinterpret_cast<const float4 *>(x32)[q];
    }

    // ---- phase 1: dedup
    int U = 0;
    if constexpr (VF) {
      // K % 4 == 0: friend rows read as int4.  Unit u < nF holds ids 4q..4q+3
      // of F(S[s]) (s = u / K4, q = u % K4); the ceil(nS/4) units after them
      // hold S itself.  One unit (4 ids) per lane per pass, loaded two passes ahead.
      const int K4 = K >> 2;
      const int nF = nS * K4, nU = nF + ((nS + 3) >> 2);
      const int ds = 32 / K4, dq = 32 - ds * K4;
      int s = lane / K4, q = lane - (lane / K4) * K4;
      auto load_unit = [&](int4 &v, int u) {
        if (u < nF) {
          v = __ldg(reinterpret_cast<const int4 *>(p.F + (int64_t)S[s] * K) + q);
        } else if (u < nU) {
          const int b = (u - nF) * 4;
          v = reinterpret_cast<const int4 *>(S)[u - nF];
          v.y = b + 1 < nS ? v.y : -1;
          v.z = b + 2 < nS ? v.z : -1;
          v.w = b + 3 < nS ? v.w : -1;
        } else {
          v = make_int4(-1, -1, -1, -1);
        }
        s += ds;
        q += dq;
        const bool wrap = q >= K4;
        q -= wrap ? K4 : 0;
        s += wrap ? 1 : 0;
      };
      int4 vA, vB;
      load_unit(vA, lane);
      load_unit(vB, 32 + lane);
#pragma unroll 1
      for (int u0 = 0; u0 < nU; u0 += 32) {
        const int id[UNR1] = {vA.x, vA.y, vA.z, vA.w};
        vA = vB;
        if (u0 + 64 < nU)
          load_unit(vB, u0 + 64 + lane);
        else
          vB = make_int4(-1, -1, -1, -1);
        bool nw[UNR1];
        hash_insert4(table, id, x, shift, (unsigned)H - 1u, nw);
#pragma unroll
        for (int u = 0; u < UNR1; ++u) {
          const unsigned m = __ballot_sync(FULL, nw[u]);
          KNND_DCHECK(!nw[u] || (id[u] >= 0 && id[u] < p.n));
          if (nw[u]) list[U + __popc(m & lanemask_lt())] = id[u];
          U += __popc(m);
          KNND_DCHECK(U <= cap);
        }
      }
    } else {
      int s = s_init, j = j_init;
      // Pre-dedup ids two groups ahead: the friend-row loads stay in flight until
      // their group is consumed (the select is deferred to that point).  Slot A
      // is consumed, slot B rotates into A, the group two ahead loads into B —
      // one copy of the loop body (the kernel is instruction-fetch sensitive).
      int fA[UNR1], vA[UNR1], fB[UNR1], vB[UNR1];  // friend id loaded; S value, or -1 (out) / -2 (use friend)
      auto load_group = [&](int (&f)[UNR1], int (&v)[UNR1], int e0) {
#pragma unroll
        for (int u = 0; u < UNR1; ++u) {
          const int e = e0 + u * 32 + lane;
          const bool in = e < total;
          const int sv = S[in ? s : 0];
          f[u] = __ldg(p.F + (int64_t)sv * K + (j > 0 ? j - 1 : 0));
          v[u] = in ? (j == 0 ? sv : -2) : -1;
          s += Gq;
          j += Gr;
          const bool wrap = j >= K1;
          j -= wrap ? K1 : 0;
          s += wrap ? 1 : 0;
        }
      };
      load_group(fA, vA, 0);
      load_group(fB, vB, 32 * UNR1);
#pragma unroll 1
      for (int e0 = 0; e0 < total; e0 += 32 * UNR1) {
        int id[UNR1];
#pragma unroll
        for (int u = 0; u < UNR1; ++u) {
          id[u] = vA[u] == -2 ? fA[u] : vA[u];
          fA[u] = fB[u];
          vA[u] = vB[u];
        }
        if (e0 + 64 * UNR1 < total) {
          load_group(fB, vB, e0 + 64 * UNR1);
        } else {
#pragma unroll
          for (int u = 0; u < UNR1; ++u) vB[u] = -1;
        }
        // shared-memory CAS insert (hash_insert_cas): in-warp duplicates resolve in
        // the CAS itself; the ballots append the winners in lane order
        bool nw[UNR1];
        hash_insert4(table, id, x, shift, (unsigned)H - 1u, nw);
#pragma unroll
        for (int u = 0; u < UNR1; ++u) {
          const unsigned m = __ballot_sync(FULL, nw[u]);
          KNND_DCHECK(!nw[u] || (id[u] >= 0 && id[u] < p.n));
          if (nw[u]) list[U + __popc(m & lanemask_lt())] = id[u];
          U += __popc(m);
          KNND_DCHECK(U <= cap);
        }
      }
    }
    __syncwarp();

    int64_t nc0 = 0, nc1 = 0;
    if (xn >= 0) {
      nc0 = __ldg(p.indptr + ((int64_t)xn - p.lo));
      nc1 = __ldg(p.indptr + ((int64_t)xn - p.lo + 1));
    }

    // ---- phase 2: screen; per-lane Q smallest, max |x log y| sum
    float best[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) best[q] = __int_as_float(0x7f800000);
    float am = 0.f;
    // ids of batch b+1 are in a register while batch b computes; batch b+2's are being loaded
    // two staging buffers in the table past the scores ([0, U), U <= H/2)
    const int u4 = (U + 3) & ~3;
    float *stage = reinterpret_cast<float *>(table + u4);
    const int rows = min(32, (H - u4) / (ld * 2));
    KNND_DCHECK(U == 0 || (rows >= 1 && u4 + 2 * rows * ld <= H));
    int id_next = (lane < min(rows, U)) ? list[lane] : 0;
    int id_after = (rows + lane < U && lane < rows) ? list[rows + lane] : 0;
    if (U > 0) {
      if constexpr (NV4 > 0)
        stage_rows_f32_reg_full<NV4, SLD>(stage, p.log32, id_next, min(rows, U), lane);
      else
        stage_rows_f32<NV4>(stage, p.log32, list, min(rows, U), ld, lane);
      cp_async_commit();
    }
    if constexpr (Q23S) {
      // The anchor's weights, computed while the first batch is in flight — and not before
      // the dedup, where they would hold NQ registers through it.  The return value is the
      // quantisation part of the bound, per anchor (+ the Euclidean scorer's fp64 term in
      // these units).
      if constexpr (Q23SIGNED)
        slack = q23_weights_signed<NV4>(x32, p.qh, p.d64, wq, abq) + p.slack * 0x1p-23f;
      else
        slack = q23_weights<NV4>(x64, p.qh, d, wq);
    }
    for (int k0 = 0, buf = 0; k0 < U; k0 += rows, buf ^= 1) {
      const int nrow = min(rows, U - k0);
      if (k0 + rows < U) {  // prefetch the next batch into the other buffer
        const int n1 = min(rows, U - k0 - rows);
        if constexpr (NV4 > 0)
          stage_rows_f32_reg_full<NV4, SLD>(stage + (buf ^ 1) * rows * ld, p.log32, id_after, n1, lane);
        else
          stage_rows_f32<NV4>(stage + (buf ^ 1) * rows * ld, p.log32, list + k0 + rows, n1, ld, lane);
        cp_async_commit();
        const int k2 = k0 + 2 * rows;
        id_after = (lane < rows && k2 + lane < U) ? list[k2 + lane] : 0;
        cp_async_wait_1();
      } else {
        cp_async_wait_0();
      }
      __syncwarp();
      {
        // rotate the lanes that take this batch's rows, so every lane's two
        // smallest cover its share of U even when a batch holds < 32 rows
        const int rot = rows < 24 ? (k0 & 31) : 0;  // (k0 is a multiple of rows)
        const int rr = (lane - rot) & 31;
        const bool in = rr < nrow;
        const int rl = in ? rr : 0;  // lanes past nrow recompute row 0, discarded
        float ce, ab;
        if constexpr (Q23S) {
          ce = screen_row_q23<NV4>(stage + buf * rows * ld + rl * ld, wq);
          ab = ce;  // KL: every term is >= 0 (the Euclidean scorer replaces the maximum by abq below)
        } else if constexpr (NV4 > 0) {
          screen_row_reg<NV4>(stage + buf * rows * ld + rl * ld, xreg, p.nonpos, ce, ab);
        } else {
          screen_row<NV4>(stage + buf * rows * ld + rl * ld, x32, ld, p.nonpos, ce, ab);
        }
        if (in) scores[k0 + rl] = ce;
        am = in ? fmaxf(am, ab) : am;
        float v = in ? ce : __int_as_float(0x7f800000);
#pragma unroll
        for (int q = 0; q < Q; ++q) {  // insertion into the sorted per-lane list
          const float lo_ = fminf(best[q], v);
          v = fmaxf(best[q], v);
          best[q] = lo_;
        }
      }
      __syncwarp();
    }
    if (xn >= 0) {  // the staging groups are complete: start the next anchor's inputs
      unsigned char *nb = base + (size_t)(pb ^ 1) * L.pre;
      prefetch_anchor(p, xn, nc0, (int)(nc1 - nc0), reinterpret_cast<int32_t *>(nb + L.S),
                      reinterpret_cast<float *>(nb + L.x32), reinterpret_cast<double *>(nb + L.x64), lane);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) am = fmaxf(am, __shfl_xor_sync(FULL, am, o));
    if constexpr (Q23SIGNED) am = abq;  // signed weights: the bound on every candidate's sum |w F|
    // Threshold.  The previous round's bound of this row (the largest screened
    // value among the current friends, all of which are in U) is a valid T; it
    // is used when it admits at most 32 candidates, else T comes from the lanes'
    // two smallest values.
    auto lane_pair_T = [&]() -> float {
      float t = __int_as_float(0x7f800000);
      if (rows * Q >= K) {  // otherwise the kept subset may hold fewer than K values
        if constexpr (KPL == 1) {
          // the 32 smallest of {best0} u {best1}: best0 ascending, best1 descending
          // (two independent networks), elementwise min, one bitonic merge
          const KeyF a = warp_sort32(KeyF{best[0]}, lane);
          const KeyF b = warp_sort32_desc(KeyF{best[1]}, lane);
          const KeyF m = warp_merge32(kmin(a, b), lane);
          t = m.shfl(K - 1).v;  // >= the K-th smallest screened value (U >= K)
        } else {
          WarpTopK<KeyF, KPL> top;
          top.init();
          top.first(KeyF{best[0]}, lane);
#pragma unroll
          for (int q = 1; q < Q; ++q) top.insert(KeyF{best[q]}, K, lane);
          t = top.get(K - 1).v;
        }
      }
      return t;
    };
    float T;
    const float ebase = p.band * am + slack;  // the screen's error bound at this anchor
    if (KPL == 1 && isfinite(T0)) {
      const float th0 = T0 + 2.f * ebase + fabsf(T0) * 1e-6f;
      int cnt = 0;
      for (int k0 = 0; k0 < U; k0 += 32) {
        const int k = k0 + lane;
        cnt += __popc(__ballot_sync(FULL, k < U && scores[k] <= th0));
      }
      T = cnt <= 32 ? T0 : lane_pair_T();
    } else {
      T = lane_pair_T();
    }
    const float theta = T + 2.f * ebase + fabsf(T) * 1e-6f;
    // the error bound among the members of R: a candidate's error is band * its
    // own sum |x log y| (+ slack), which equals its screened value (<= theta)
    // when every term has one sign — usually several times tighter than the
    // bound over all of U, so fewer rows fall back to the fp64 ranking
    const float ebase_r =
        (!Q23SIGNED && (Q23S || (p.metric == METRIC_KL && p.nonpos))) ? p.band * fminf(am, theta) + slack : ebase;

    // ---- phase 3: R (ids and screened values) in place at the front of list / scores
    int nR = 0;
    for (int k0 = 0; k0 < U; k0 += 32) {
      const int k = k0 + lane;
      const float v = k < U ? scores[k] : 0.f;
      const bool take = k < U && v <= theta;
      const int y = take ? list[k] : 0;
      const unsigned m = __ballot_sync(FULL, take);
      if (take) {
        const int r = nR + __popc(m & lanemask_lt());
        list[r] = y;
        scores[r] = v;
      }
      nR += __popc(m);
    }
    __syncwarp();

    // ---- phase 4: certify the screened order, else rank R exactly in fp64
    bool diff;
    float kth = theta;  // every member of the new row has a screened value <= theta
    if (!(KPL == 1 && p.out_kl == nullptr && nR <= 32 &&
          certify_row(p, list, scores, nR, 2.f * ebase_r, x, xr, lane, diff, kth))) {
      diff = exact_row<KPL>(p, list, nR, stage64, rcap64, x64, x, xr, lane);
      ++acc_exact;
    }
    if (p.bound_out && lane == 0) p.bound_out[xr] = kth;
    if (lane == 0) {
      acc_comp += (unsigned long long)U;
      acc_changed += diff ? 1ull : 0ull;
      acc_bad += (U < K) ? 1ull : 0ull;
      if (p.out_ucount) p.out_ucount[xr] = U;
    }
    __syncwarp();
    a = a_nxt;
    x = xn;
    c0 = nc0;
    c = (int)(nc1 - nc0);
    pb ^= 1;
  }
  cp_async_wait_all();
  if (p.npeers) __threadfence_system();  // peer rows performed before the caller's cross-rank barrier
  if (lane == 0) {
    if (acc_comp) atomicAdd(&p.tally[0], acc_comp);
    if (acc_changed) atomicAdd(&p.tally[1], acc_changed);
    if (acc_bad) atomicAdd(&p.tally[2], acc_bad);
    if (acc_exact) atomicAdd(&p.tally[3], acc_exact);
  }
}

// bin the anchors of [lo, hi) by pre-dedup bound P = (K+c)(K+1): class i is
// the first with P <= lim[i]; the last class (global-memory tables) takes the rest
constexpr int MAXCLS = 6;
struct Lims {
  int64_t v[MAXCLS];
  int n;  // number of classes (the last one is unbounded)
};

static __global__ void classify_kernel(const int64_t *__restrict__ indptr, int64_t m, int64_t lo, int K, Lims lims,
                                int32_t *__restrict__ lists, int32_t *__restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < m; base += stride) {
    const int64_t xr = base + threadIdx.x;
    int cls = -1;
    if (xr < m) {
      const int64_t c = indptr[xr + 1] - indptr[xr];
      const int64_t P = ((int64_t)K + c) * (K + 1);
      cls = lims.n - 1;
      for (int i = lims.n - 2; i >= 0; --i)
        if (P <= lims.v[i]) cls = i;
    }
    for (int k = 0; k < lims.n; ++k) warp_append(cls == k, (int)(lo + xr), counts + k, lists + (int64_t)k * m, lane);
  }
}

// ---------------------------------------------------------------------------
// host side: the size-class plan

enum { KIND_WARP = 0, KIND_BLOCK128 = 1, KIND_BLOCK256 = 2, KIND_GLOBAL = 3, KIND_BLOCK512 = 4 };

struct Cls {
  int kind, logH, sw;
  int cap;      // warp class: capacity of the unique list (= lim)
  int64_t lim;  // pre-dedup bound handled (H/2 for shared-memory tables)
  bool need;
};

struct Plan {
  int kpl, nv4, ncls;
  Cls c[MAXCLS];
  int nslab;
  int64_t slab_ints;
  size_t lists_off, counts_off, slab_off, total;
};

constexpr int WARP_BLOCK = 128, GL = 512;

static int ilog2_ceil(int64_t v) {
  int l = 0;
  while (((int64_t)1 << l) < v) ++l;
  return l;
}

// KNND_PLAN overrides the shared-memory classes, e.g. "w11,b128:12,b256:14"
// (w = warp per anchor, bG = G-thread block per anchor, :L = log2 table slots)
static int parse_plan(const char *spec, int kind[], int logH[]) {
  int n = 0;
  const char *q = spec;
  while (*q && n < MAXCLS - 1) {
    int k, l = 0;
    if (q[0] == 'w') {
      k = KIND_WARP;
      l = atoi(q + 1);
    } else if (q[0] == 'b' && !strncmp(q + 1, "128:", 4)) {
      k = KIND_BLOCK128;
      l = atoi(q + 5);
    } else if (q[0] == 'b' && !strncmp(q + 1, "256:", 4)) {
      k = KIND_BLOCK256;
      l = atoi(q + 5);
    } else if (q[0] == 'b' && !strncmp(q + 1, "512:", 4)) {
      k = KIND_BLOCK512;
      l = atoi(q + 5);
    } else {
      return 0;
    }
    if (l < 8 || l > 15) return 0;
    kind[n] = k;
    logH[n] = l;
    ++n;
    q = strchr(q, ',');
    if (!q) break;
    ++q;
  }
  return n;
}

constexpr int64_t HUB_SLAB_BUDGET = (int64_t)4 << 30;

static Plan make_plan(int64_t n_items, int64_t m, int d, int K, int max_indeg) {
  Plan P{};
  P.kpl = K <= 32 ? 1 : 2;
  P.nv4 = (d + 3) / 4;
  const int64_t K1 = K + 1;
  const int ld = (d + 3) / 4 * 4;
  // default: warp per anchor for in-degrees up to ~1.4K (the bulk of a random
  // K-out graph), 128-thread blocks up to ~2.3x that, 256-thread blocks for the
  // tail, global tables for the hubs
  int l1 = ilog2_ceil(2 * K1 * (K + (2 * K) / 5));
  const int lstage = ilog2_ceil(64 * (int64_t)ld);  // 32 staged fp32 rows fit in H/2 slots
  if (l1 < lstage) l1 = lstage;
  if (l1 < 9) l1 = 9;
  if (l1 > 12) l1 = 12;
  // measured on B200 at C3 (KNND_PLAN sweeps): warp / 128-thread blocks for two
  // table sizes / 256-thread blocks for 2^14 slots / 512-thread blocks for 2^15
  // (one block per SM there: the extra warps cut that class's time by 25%) /
  // global tables
  int kind[MAXCLS] = {KIND_WARP, KIND_BLOCK128, KIND_BLOCK128, KIND_BLOCK256, KIND_BLOCK256};
  int logH[MAXCLS] = {l1, l1 + 1, l1 + 2, l1 + 3 < 15 ? l1 + 3 : 15, 15};
  int n = l1 + 3 < 15 ? 5 : 4;
  for (int i = 0; i < n; ++i)
    if (kind[i] == KIND_BLOCK256 && logH[i] == 15) kind[i] = KIND_BLOCK512;
  if (const char *env = getenv("KNND_PLAN")) {
    int k2[MAXCLS], l2[MAXCLS];
    const int n2 = parse_plan(env, k2, l2);
    if (n2 > 0) {
      n = n2;
      for (int i = 0; i < n; ++i) {
        kind[i] = k2[i];
        logH[i] = l2[i];
      }
    }
  }
  const int64_t Pmax = ((int64_t)K + max_indeg) * K1;
  int64_t prev = 0;
  for (int i = 0; i < n; ++i) {
    Cls &c = P.c[i];
    c.kind = kind[i];
    c.logH = logH[i];
    c.lim = ((int64_t)1 << c.logH) / 2;
    // the warp class fills its table past one half (4-slot buckets take it): its
    // slab has room for a longer unique list, and warp anchors run ~35% faster
    // than the 2^12 block class they would otherwise join (KNND_WLIM overrides)
    if (c.kind == KIND_WARP && i == 0) {
      int64_t wl = c.lim * 5 / 4;
      if (const char *env = getenv("KNND_WLIM")) wl = atoll(env);
      if (wl >= c.lim && wl <= c.lim * 11 / 8) c.lim = wl;
    }
    c.cap = (int)c.lim;
    c.sw = (int)(c.lim / K1 + 1);
    // a shared-memory class must fit: the staged S list (up to lim / (K + 1)
    // ids, double-buffered) grows as K shrinks (K = 2: a third of the table);
    // the classes from the first that does not fit on are left to the
    // global-memory class, whose S and table live in its slab
    const size_t need = c.kind == KIND_WARP
                            ? warp_slab(d, ld, 1 << c.logH, c.sw, c.cap).total
                            : smem_layout(c.kind == KIND_BLOCK128 ? 128 : c.kind == KIND_BLOCK256 ? 256 : 512, false,
                                          d, ld, 1 << c.logH, c.sw)
                                  .total;
    if (i > 0 && need > 227 * 1024) {
      n = i;
      break;
    }
    c.need = i == 0 || Pmax > prev;
    prev = c.lim;
  }
  Cls &g = P.c[n];
  g.kind = KIND_GLOBAL;
  g.need = Pmax > prev;
  g.lim = INT64_MAX;
  g.logH = g.need ? ilog2_ceil(2 * Pmax) : 0;
  g.sw = (K + max_indeg + 31) & ~31;  // keeps the table int4-aligned in the slab
  P.ncls = n + 1;
  P.slab_ints = g.need ? (int64_t)align_up((size_t)g.sw + ((size_t)3 << g.logH) / 2, 64) : 0;
  // hub slabs: one per resident block (2 per SM), but no more than the anchors
  // the class can hold — its in-degrees exceed cmin and they sum to at most
  // n*K — and at most HUB_SLAB_BUDGET bytes in all (at least one slab): every
  // slab is sized for the largest hub, so skewed in-degrees (duplicate points,
  // hubness) would otherwise ask for tens of GB.  Fewer slabs only means fewer
  // hub blocks in flight (the class kernel's grid is capped at nslab).
  P.nslab = 0;
  if (g.need) {
    int64_t ns = 2 * (int64_t)num_sms();
    const int64_t cmin = prev / K1 - K;  // the global class: (K + c)(K + 1) > prev, so c > cmin
    const int64_t hubs = cmin >= 0 ? (n_items * K) / (cmin + 1) : m;
    if (ns > hubs) ns = hubs;
    if (ns > m) ns = m;
    const int64_t by_budget = HUB_SLAB_BUDGET / (P.slab_ints * 4);
    if (ns > by_budget) ns = by_budget;
    P.nslab = (int)(ns < 1 ? 1 : ns);
  }
  size_t o = 0;
  P.lists_off = o;
  o = align_up(o + (size_t)P.ncls * m * 4, 256);
  P.counts_off = o;
  o = align_up(o + 64, 256);
  P.slab_off = o;
  o = align_up(o + (size_t)P.nslab * P.slab_ints * 4, 256);
  P.total = o;
  return P;
}

template <int G, int NV4, int KPL, bool GTAB, int SCR = SCR_F32>
static int launch_join(const JoinParams &p, const int32_t *alist, const int32_t *acount, int logH, int SW,
                       int32_t *gslab, int64_t slab_ints, int grid_cap, cudaStream_t st) {
  // friend ids two groups ahead pays for the larger shared tables (B128 at 2^13:
  // -8%); at 2^12 (at most 4 groups per anchor) it measured 20% slower
  auto kern = (!GTAB && logH >= 13) ? join_kernel<G, NV4, KPL, GTAB, !GTAB, SCR>
                                    : join_kernel<G, NV4, KPL, GTAB, false, SCR>;
  const SmemLayout L = smem_layout(G, GTAB, p.d, p.ld, 1 << logH, SW);
  size_t smem = L.total;
  if (smem > 227 * 1024) {
    set_error("local join: shared memory %zu exceeds 227 KB (d=%d, H=%d)", smem, p.d, 1 << logH);
    return KNND_EUNSUPPORTED;
  }
  int per_sm = 0;
  if (int rc = kernel_occupancy((const void *)kern, G, smem, &per_sm)) return rc;
  if (per_sm < 1) {
    set_error("local join: kernel cannot be resident (smem=%zu)", smem);
    return KNND_EUNSUPPORTED;
  }
  // The staging rows of the screen live in the table past the scores: when that
  // leaves a warp fewer than 32 rows per buffer (the 2^12 class: 18), the shared
  // memory the resident blocks leave unused extends the table — the per-batch
  // instructions are amortised over more rows (the block classes are issue-bound).
  int XT = 0;
  if constexpr (!GTAB) {
    const int H = 1 << logH;
    const int srow = 2 * (SCR != SCR_F32 ? (NV4 | 1) * 4 : p.ld);  // floats per staged row, two buffers
    const int have = (H / 2) / (G / 32) / srow;                    // rows per buffer at the largest |U| = H / 2
    if (have < 32) {
      // (a block's allocation is rounded up to 1 KB, plus 1 KB the system reserves per block)
      const size_t cap_b = (((size_t)228 * 1024 / per_sm - 1024) >> 10) << 10;
      const size_t spare = cap_b > smem ? cap_b - smem : 0;
      const size_t want = (size_t)(32 - have) * srow * (G / 32) * 4;
      const size_t extra = spare < want ? spare : want;
      int per_sm2 = 0;
      if (extra >= 1024 && smem + extra <= 227 * 1024 &&
          kernel_occupancy((const void *)kern, G, smem + extra, &per_sm2) == KNND_OK && per_sm2 == per_sm) {
        XT = (int)(extra / 4);
        smem += extra;
      }
    }
  }
  int grid = per_sm * num_sms();
  if (grid_cap > 0 && grid > grid_cap) grid = grid_cap;
  if (getenv("KNND_CLASS_TIMING"))
    fprintf(stderr, "knnd block class G=%d logH=%d: %d blocks/SM, smem %zu B (%d extra staging ints)\n", G, logH, per_sm,
            smem, XT);
  kern<<<grid, G, smem, st>>>(p, alist, acount, logH, SW, gslab, slab_ints, XT);
  KNND_LAUNCHED(1);
  return KNND_OK;
}

template <int NV4, int KPL, int SCR = SCR_F32>
static int launch_warp(const JoinParams &p, const int32_t *alist, const int32_t *acount, int logH, int SW,
                       int cap, cudaStream_t st) {
  // friend rows as int4 when they are 16-B aligned (K % 4 == 0)
  auto kern = (p.K % 4 == 0) ? join_warp_kernel<NV4, KPL, true, SCR> : join_warp_kernel<NV4, KPL, false, SCR>;
  const WarpSlab L = warp_slab(p.d, p.ld, 1 << logH, SW, cap);
  // warps per block: the largest of 4/2/1 that keeps the most warps resident
  // (big tables leave room for fewer than 4 slabs per block slot)
  int best_wpb = 0, best_warps = 0;
  size_t smem = 0;
  for (int wpb = WARP_BLOCK / 32; wpb >= 1; wpb >>= 1) {
    const size_t sm_b = L.total * wpb;
    if (sm_b > 227 * 1024) continue;
    int per_sm = 0;
    if (int rc = kernel_occupancy((const void *)kern, wpb * 32, sm_b, &per_sm)) return rc;
    if (per_sm * wpb > best_warps) {
      best_warps = per_sm * wpb;
      best_wpb = wpb;
      smem = sm_b;
    }
  }
  if (best_warps < 1) {
    set_error("local join: warp slabs %zu B exceed 227 KB (d=%d, H=%d)", L.total, p.d, 1 << logH);
    return KNND_EUNSUPPORTED;
  }
  kern<<<(best_warps / best_wpb) * num_sms(), best_wpb * 32, smem, st>>>(p, alist, acount, logH, SW, cap);
  KNND_LAUNCHED(1);
  return KNND_OK;
}

// compile-time row widths (float4 count); anything else takes the generic path
#define KNND_NV_SWITCH(CALL)               \
  switch (p.ld == P.nv4 * 4 ? P.nv4 : 0) { \
    case 2: CALL(2);                       \
    case 3: CALL(3);                       \
    case 5: CALL(5);                       \
    case 13: CALL(13);                     \
    default: CALL(0);                      \
  }

// The kernel instantiations are split over three translation units by family, so the
// build compiles them in parallel (one file had made join.cu a 4-minute long pole):
//   FAM_F32K1  fp32 rows, K <= 32        (join.cu)
//   FAM_F32K2  fp32 rows, K in 33..64    (join_f32k2.cu)
//   FAM_Q23    Q23 rows, KL and Euclidean (join_q23.cu)
constexpr int FAM_F32K1 = 0, FAM_F32K2 = 1, FAM_Q23 = 2;

template <int FAM, int G, bool GTAB>
static int dispatch_block(const Plan &P, const JoinParams &p, const int32_t *alist, const int32_t *acount,
                          int logH, int SW, int32_t *gslab, int64_t slab_ints, int grid_cap, cudaStream_t st) {
  if constexpr (FAM == FAM_Q23) {
    if (p.scr == SCR_Q23L2) {  // Euclidean: K <= 32, rows of 2 to 4 16-byte chunks; checked at the entry
      if (p.nvq == 2)
        return launch_join<G, 2, 1, GTAB, SCR_Q23L2>(p, alist, acount, logH, SW, gslab, slab_ints, grid_cap, st);
      if (p.nvq == 3)
        return launch_join<G, 3, 1, GTAB, SCR_Q23L2>(p, alist, acount, logH, SW, gslab, slab_ints, grid_cap, st);
      return launch_join<G, 4, 1, GTAB, SCR_Q23L2>(p, alist, acount, logH, SW, gslab, slab_ints, grid_cap, st);
    }
    // KL: K <= 32, rows of 1 to 4 (or 10) 16-byte chunks; checked at the entry
    if (p.nvq == 1)
      return launch_join<G, 1, 1, GTAB, SCR_Q23>(p, alist, acount, logH, SW, gslab, slab_ints, grid_cap, st);
    if (p.nvq == 2)
      return launch_join<G, 2, 1, GTAB, SCR_Q23>(p, alist, acount, logH, SW, gslab, slab_ints, grid_cap, st);
    if (p.nvq == 3)
      return launch_join<G, 3, 1, GTAB, SCR_Q23>(p, alist, acount, logH, SW, gslab, slab_ints, grid_cap, st);
    if (p.nvq == 10)
      return launch_join<G, 10, 1, GTAB, SCR_Q23>(p, alist, acount, logH, SW, gslab, slab_ints, grid_cap, st);
    return launch_join<G, 4, 1, GTAB, SCR_Q23>(p, alist, acount, logH, SW, gslab, slab_ints, grid_cap, st);
  } else {
    constexpr int KPL = FAM == FAM_F32K1 ? 1 : 2;
#define KNND_CALL(NV) return launch_join<G, NV, KPL, GTAB>(p, alist, acount, logH, SW, gslab, slab_ints, grid_cap, st)
    KNND_NV_SWITCH(KNND_CALL)
#undef KNND_CALL
  }
}

template <int FAM>
static int dispatch_warp(const Plan &P, const JoinParams &p, const int32_t *alist, const int32_t *acount, int logH,
                         int SW, int cap, cudaStream_t st) {
  if constexpr (FAM == FAM_Q23) {
    if (p.scr == SCR_Q23L2) {
      if (p.nvq == 2) return launch_warp<2, 1, SCR_Q23L2>(p, alist, acount, logH, SW, cap, st);
      if (p.nvq == 3) return launch_warp<3, 1, SCR_Q23L2>(p, alist, acount, logH, SW, cap, st);
      return launch_warp<4, 1, SCR_Q23L2>(p, alist, acount, logH, SW, cap, st);
    }
    if (p.nvq == 1) return launch_warp<1, 1, SCR_Q23>(p, alist, acount, logH, SW, cap, st);
    if (p.nvq == 2) return launch_warp<2, 1, SCR_Q23>(p, alist, acount, logH, SW, cap, st);
    if (p.nvq == 3) return launch_warp<3, 1, SCR_Q23>(p, alist, acount, logH, SW, cap, st);
    if (p.nvq == 10) return launch_warp<10, 1, SCR_Q23>(p, alist, acount, logH, SW, cap, st);
    return launch_warp<4, 1, SCR_Q23>(p, alist, acount, logH, SW, cap, st);
  } else {
    constexpr int KPL = FAM == FAM_F32K1 ? 1 : 2;
#define KNND_CALL(NV) return launch_warp<NV, KPL>(p, alist, acount, logH, SW, cap, st)
    KNND_NV_SWITCH(KNND_CALL)
#undef KNND_CALL
  }
}

// one size class of one family (defined once per family, in its translation unit)
template <int FAM>
static int dispatch_class_family(const Plan &P, int i, const JoinParams &p, const int32_t *lists,
                                 const int32_t *counts, int64_t m, int32_t *slabs, cudaStream_t st) {
  const Cls &c = P.c[i];
  const int32_t *alist = lists + (int64_t)i * m;
  const int32_t *acount = counts + i;
  switch (c.kind) {
    case KIND_WARP:
      return dispatch_warp<FAM>(P, p, alist, acount, c.logH, c.sw, c.cap, st);
    case KIND_BLOCK128:
      return dispatch_block<FAM, 128, false>(P, p, alist, acount, c.logH, c.sw, nullptr, 0, 0, st);
    case KIND_BLOCK256:
      return dispatch_block<FAM, 256, false>(P, p, alist, acount, c.logH, c.sw, nullptr, 0, 0, st);
    case KIND_BLOCK512:
      return dispatch_block<FAM, 512, false>(P, p, alist, acount, c.logH, c.sw, nullptr, 0, 0, st);
    default:
      return dispatch_block<FAM, GL, true>(P, p, alist, acount, c.logH, c.sw, slabs, P.slab_ints, P.nslab, st);
  }
}

int join_dispatch_f32k1(const Plan &P, int i, const JoinParams &p, const int32_t *lists, const int32_t *counts,
                        int64_t m, int32_t *slabs, cudaStream_t st);
int join_dispatch_f32k2(const Plan &P, int i, const JoinParams &p, const int32_t *lists, const int32_t *counts,
                        int64_t m, int32_t *slabs, cudaStream_t st);
int join_dispatch_q23(const Plan &P, int i, const JoinParams &p, const int32_t *lists, const int32_t *counts,
                      int64_t m, int32_t *slabs, cudaStream_t st);

}  // namespace knnd
