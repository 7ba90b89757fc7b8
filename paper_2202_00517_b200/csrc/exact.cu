// Brute-force exact K nearest neighbours for a set of queries — the ground
// truth behind recall (evaluation.py:83-90 exact_knn, per query x:
//   s = batch_scores(x); s[x] = inf; row = _smallest_k(s, K)   (evaluation.py:53-71)
// i.e. the K smallest (fp64 score, id) over every other point).
//
// The all-pairs screen is a GEMM (queries x d) * (d x candidates), so it runs
// on the tensor cores (tcgen05.mma kind::tf32, accumulators in TMEM, B tiles
// by TMA; exact_tc_kernel below), with the same screen-then-rescore scheme as
// the local join:
//   sweep 1  every query against every candidate; per thread (= query) the
//            minima of SLOTS column slots -> T_q >= the K-th smallest;
//   sweep 2  the same products again; every candidate with ce <= theta_q (T_q
//            plus the rigorous tf32 error band) is appended to the query's list;
//   rank     one warp per query rescoring its list in fp64 (score.cuh, the
//            join's exact scorer) and keeping the K smallest (score, id).
// A list longer than `cap` is reported through out_count and the caller reruns
// that query with a larger cap (never silently truncated).
#include <cuda.h>

#include <cstdlib>

#include "common.cuh"
#include "score.cuh"

namespace knnd {

struct ExactParams {
  const double *points;
  const float *log32;
  const double *log64;
  const double *xlogx;
  int64_t n;
  int d, ld, K;
  const int32_t *queries;
  int64_t nq;
  int nonpos;  // every log coordinate <= 0 (then |x log y| sums equal the screen)
  int32_t *cand;   // nq x cap candidate ids
  int cap;
  int32_t *count;  // nq candidate counts (may exceed cap)
  int32_t *out_ids;
  double *out_scores;
  int metric;      // score.cuh
  int d64;         // fp64 row length (d, or d+1 for L2)
  int pstride;     // row stride of `points`
  const float *aside32;  // L2: anchor-side fp32 rows (null for KL)
  float slack;            // L2: absolute error bound of the fp64 values (join.cu JoinParams::slack)
};

// ---------------------------------------------------------------------------
// The screen on the 5th-generation tensor cores.  A CTA owns 256 queries (two
// halves of 128, A operands resident in shared memory) and streams every
// candidate in tiles of 128 rows; for each tile tcgen05.mma kind::tf32
// computes D_h = A_h * B^T = the screened cross entropies ce(q, y) of both
// 128 x 128 blocks into tensor memory (A holds -x, or -anchor32 for L2); the
// epilogue warps read D with tcgen05.ld, one query row per thread.
//   warp 0       producer (one lane): each tile is one contiguous bulk copy
//                (cp.async.bulk) of its pre-tiled image into a STAGES-deep ring
//   warp 1       MMA issuer (one lane), owns the TMEM allocation
//   warps 2..9   epilogue: build A (swizzled) at start, then per tile
//                sweep 1: per-thread minima of SLOTS column slots
//                sweep 2: append every candidate with ce <= theta_q
// TMEM holds two accumulator buffers per half (4 x 128 columns), so the MMAs
// of tile t+1 run while the epilogue reads tile t.  Operands are K-major with
// the 128-byte swizzle; the candidate table is re-laid out once per call into
// that exact shared-memory image (tc_image_kernel), so a tile moves as one
// 16-KB bulk copy instead of 128 row copies (per-row TMA tiles and per-row
// gathers measured ~8 SM cycles per row, the bottleneck).
//
// Error band.  kind::tf32 keeps 10 explicit mantissa bits of each fp32
// operand (truncated or rounded: relative error < 2^-10 per operand), the
// products and the fp32 accumulation add < d 2^-23 relative of sum |x l|; so
// |ce~ - ce| <= eps * sum_j |x_j log y_j| with eps = 2^-9 + 64 * 2^-23, and
// the band uses TC_EPS = 2^-8.  sum |x l| is ce itself when every log is
// <= 0 (simplex data); otherwise it is bounded by |a|_2 * max_y |c_y|_2
// (Cauchy-Schwarz: per-query anchor norm, global candidate-row norm).
//
// Threshold.  Sweep 1 keeps, per thread, the minimum of each of SLOTS column
// slots (candidate column mod SLOTS) over a subset of the tiles: SLOTS values
// of distinct candidates, so their K-th smallest T_q is >= the K-th smallest
// screened value (an upper bound, needing SLOTS >= K).  One 3-input min per two scores, no branch.
// theta_q = T_q + band; sweep 2 keeps ce <= theta_q, which contains every
// exact top-K member (same argument as the local join).
constexpr int TC_M = 128;           // queries per half (TMEM lanes)
constexpr int TC_Q = 2 * TC_M;      // queries per CTA
constexpr int TC_BN = 128;          // candidates per tile
constexpr int TC_EPI = 8;           // epilogue warps (2 per TMEM lane quadrant)
constexpr int TC_THREADS = 32 * (2 + TC_EPI);
constexpr float TC_EPS = 0x1p-8f;   // tf32 screen error, relative to sum |x log y| (see above)
constexpr uint32_t TC_SUB = TC_BN * 128;  // bytes of one 32-wide K sub-tile of a candidate tile
// Sweep 1 reads one candidate tile in TC_SUB1: its threshold, the K-th smallest
// of the slot minima over that subset, is still an upper bound (a subset's K-th
// smallest is >= the whole set's), only looser — sweep 2 then keeps ~TC_SUB1
// times more candidates (a few hundred; lists that overflow are rerun with a
// larger capacity), and the tensor memory is read 1 + 1/TC_SUB1 times per
// pair instead of twice.  TMEM reads (64 B/cycle/SM) bound this kernel.
constexpr int TC_SUB1 = 4;

struct TcParams {
  const double *points;
  const float *aside32;  // L2 anchor rows (fp32, ld) or null (KL: -x from points)
  int pstride;
  int d, ld, KT, ksteps, stages;
  int64_t n;
  const unsigned char *image;  // pre-tiled candidate table: ceil(n/128) tiles of KT * 16 KB
  const int32_t *queries;
  int64_t nq;
  int K;
  int nonpos;
  const float *maxc;  // max_y |c_y|_2 (device scalar; unused when nonpos)
  float slack;
  int32_t *cand;      // nq x cap candidate ids
  int cap;
  int32_t *count;
  uint32_t idesc;
};

__device__ __forceinline__ void tc_mbar_init(uint64_t *b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void tc_mbar_expect(uint64_t *b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tc_mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void tc_mbar_wait(uint64_t *b, unsigned parity) {
  asm volatile(
      "{\n.reg .pred P;\nTCW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra TCW_%=;\n}" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}
// one contiguous global -> shared bulk copy completing on an mbarrier (SASS UBLKCP)
__device__ __forceinline__ void tc_bulk(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// K-major, 128-byte swizzle, 8-row atoms of 1024 B: start (16-B units), LBO 1, SBO 64, sm100 version 1
__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void tc_mma(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(dtmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// issue one 32-column TMEM load (no wait: several are put in flight, then tc_ld_wait)
__device__ __forceinline__ void tc_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// wait for this thread's TMEM loads; the registers pass through the asm so no
// use of them can be scheduled before the wait
__device__ __forceinline__ void tc_ld_wait(uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.wait::ld.sync.aligned;"
      : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]), "+r"(r[8]),
        "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]), "+r"(r[16]),
        "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), "+r"(r[24]),
        "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
      :
      : "memory");
}
__device__ __forceinline__ float tc_min3(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// shared-memory layout (bytes from the 1024-aligned base)
struct TcSmem {
  uint32_t a, b, bars, total;
  __host__ __device__ TcSmem(int KT, int stages) {
    a = 0;
    b = (uint32_t)KT * TC_Q * 128;
    bars = b + (uint32_t)stages * KT * TC_SUB;
    total = bars + 8 * (2 * stages + 4) + 16;
  }
};

// the candidate table as the shared-memory image of each tile: 128 rows, K
// padded with zeros to KT x 32, 128-byte swizzle (16-B chunk c of row r at
// chunk c ^ (r & 7)), rows past n zero; one thread per 16-byte chunk
__global__ void tc_image_kernel(const float *__restrict__ c, int64_t n, int ld, int KT, unsigned char *__restrict__ img) {
  const int64_t total = ((n + TC_BN - 1) / TC_BN) * TC_BN * KT * 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int ch = (int)(i & 7);
    const int64_t rk = i >> 3;       // (row, kt) in row-major order of the table
    const int kt = (int)(rk % KT);
    const int64_t y = rk / KT;       // global row
    const int r = (int)(y % TC_BN);
    const int64_t tile = y / TC_BN;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const int k0 = kt * 32 + ch * 4;
    if (y < n && k0 < ld) v = *reinterpret_cast<const float4 *>(c + y * ld + k0);  // ld % 4 == 0
    unsigned char *dst = img + (tile * KT + kt) * (int64_t)TC_SUB + (r >> 3) * 1024 + (r & 7) * 128 +
                         ((ch ^ (r & 7)) * 16);
    KNND_DCHECK(dst + 16 <= img + ((n + TC_BN - 1) / TC_BN) * KT * (int64_t)TC_SUB);
    *reinterpret_cast<float4 *>(dst) = v;
  }
}

// SL: slot groups of 32 (SLOTS = 32 * SL kept minima per thread, SLOTS >= K)
template <int SL>
__global__ void __launch_bounds__(TC_THREADS, 1) exact_tc_kernel(TcParams p) {
  extern __shared__ unsigned char sm_raw[];
  const uint32_t raw = smem_u32(sm_raw);
  unsigned char *sm = sm_raw + (((raw + 1023u) & ~1023u) - raw);  // 1024-aligned (128-B swizzle atoms)
  const TcSmem L(p.KT, p.stages);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ST = p.stages, KT = p.KT;
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + L.bars);
  uint64_t *empty = full + ST;
  uint64_t *tfull = empty + ST;  // [2]
  uint64_t *tempty = tfull + 2;  // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
  const int64_t q0 = (int64_t)blockIdx.x * TC_Q;
  const int64_t ntile = (p.n + TC_BN - 1) / TC_BN;
  const int64_t ntile1 = (ntile + TC_SUB1 - 1) / TC_SUB1;  // sweep 1 reads every TC_SUB1-th tile
  const int64_t total_tiles = ntile1 + ntile;
  constexpr uint32_t TMEM_COLS = 4 * TC_BN;  // (buffer, half) accumulators

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < ST; ++s) {
      tc_mbar_init(full + s, 1);
      tc_mbar_init(empty + s, 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc_mbar_init(tfull + i, 1);
      tc_mbar_init(tempty + i, TC_EPI);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // epilogue threads: query row r of half h; build A_h (the row's -x, fp32,
  // zero padded to KT*32) in the K-major 128-B-swizzled layout, and the row's
  // anchor norm for the non-simplex band
  const bool is_epi = warp >= 2;
  const int half = is_epi ? (warp - 2) / 4 : 0;
  const int r = (warp & 3) * 32 + lane;  // TMEM lane quadrant = warp % 4
  const int64_t qa = q0 + half * TC_M + r;
  int64_t qid = -1;
  float anorm = 0.f;
  if (is_epi) {
    if (qa < p.nq) qid = p.queries[qa];
    KNND_DCHECK(qid < p.n);
#ifdef KNND_CHECKED
    {
      unsigned dyn;
      asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
      KNND_DCHECK((size_t)(sm - sm_raw) + L.total <= dyn);
    }
#endif
    unsigned char *arow = sm + L.a + (uint32_t)half * KT * TC_M * 128 + (uint32_t)(r >> 3) * 1024 + (uint32_t)(r & 7) * 128;
    for (int kt = 0; kt < KT; ++kt) {
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {  // 16-byte chunks of the 128-byte row
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        float *vv = reinterpret_cast<float *>(&v);
        if (qid >= 0) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int k = kt * 32 + c * 4 + e;
            float a = 0.f;
            if (p.aside32) {
              if (k < p.ld) a = -p.aside32[qid * p.ld + k];
            } else if (k < p.d) {
              a = -(float)p.points[qid * p.pstride + k];
            }
            vv[e] = a;
            anorm = fmaf(a, a, anorm);
          }
        }
        *reinterpret_cast<float4 *>(arow + (uint32_t)kt * TC_M * 128 + (uint32_t)((c ^ (r & 7)) * 16)) = v;
      }
    }
    anorm = sqrtf(anorm) * (1.f + 0x1p-20f);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // A is read by the tensor core (async proxy)
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---- producer: one bulk copy per tile image
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)KT * TC_SUB;
      int s = 0;
      unsigned ph = 0;
      for (int sweep = 0; sweep < 2; ++sweep) {
        const unsigned char *src = p.image;
        const int64_t step = sweep == 0 ? TC_SUB1 : 1;
        for (int64_t t = 0; t < ntile; t += step, src += step * bytes) {
          tc_mbar_wait(empty + s, ph ^ 1);
          tc_mbar_expect(full + s, bytes);
          tc_bulk(sm + L.b + (uint32_t)s * bytes, src, bytes, full + s);
          if (++s == ST) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer
    if (lane == 0) {
      const uint32_t a_base = smem_u32(sm + L.a);
      int s = 0;
      unsigned ph = 0;
      for (int64_t t = 0; t < total_tiles; ++t) {
        const int acc = (int)(t & 1);
        const unsigned aph = (unsigned)((t >> 1) & 1);
        tc_mbar_wait(tempty + acc, aph ^ 1);  // the epilogue has drained this buffer
        tc_mbar_wait(full + s, ph);           // the candidate tile has landed
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t b_base = smem_u32(sm + L.b + (uint32_t)s * KT * TC_SUB);
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          const uint32_t d = tmem + (uint32_t)((2 * acc + h) * TC_BN);
          const uint32_t ah = a_base + (uint32_t)h * KT * TC_M * 128;
          for (int kk = 0; kk < p.ksteps; ++kk) {
            const int kt = kk >> 2, ks = kk & 3;
            tc_mma(d, tc_desc(ah + (uint32_t)kt * TC_M * 128 + ks * 32), tc_desc(b_base + (uint32_t)kt * TC_SUB + ks * 32),
                   p.idesc, kk > 0 ? 1u : 0u);
          }
        }
        tc_commit(empty + s);     // the tile's slot is free once these MMAs complete
        tc_commit(tfull + acc);   // both halves' accumulators are ready
        if (++s == ST) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else {
    // ---- epilogue: one query row per thread
    constexpr int SLOTS = 32 * SL;
    float best[SLOTS];
#pragma unroll
    for (int i = 0; i < SLOTS; ++i) best[i] = __int_as_float(0x7f800000);
    float theta = -__int_as_float(0x7f800000);
    int cnt = 0;
    int32_t *my = p.cand + (qa < p.nq ? qa : 0) * p.cap;
    const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(half * TC_BN);
    for (int64_t t = 0; t < total_tiles; ++t) {
      const int acc = (int)(t & 1);
      const unsigned aph = (unsigned)((t >> 1) & 1);
      const bool sweep2 = t >= ntile1;
      if (t == ntile1) {
        // ---- end of sweep 1: T_q = K-th smallest of the slot minima, then the band
        // (bitonic sort of the SLOTS minima, fully unrolled: register indices only)
#pragma unroll
        for (int k = 2; k <= SLOTS; k <<= 1)
#pragma unroll
          for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
            for (int i = 0; i < SLOTS; ++i) {
              const int l = i ^ j;
              if (l > i) {
                const float lo = fminf(best[i], best[l]), hi = fmaxf(best[i], best[l]);
                const bool up = (i & k) == 0;
                best[i] = up ? lo : hi;
                best[l] = up ? hi : lo;
              }
            }
        float T = best[0];
#pragma unroll
        for (int i = 1; i < SLOTS; ++i) T = (i == p.K - 1) ? best[i] : T;
        if (p.nonpos) {
          // ce >= 0 and sum |x log y| == ce: K candidates have ce <= T / (1 - eps), and
          // a member y of the exact top K then screens at ce~ <= T (1 + eps) / (1 - eps)
          theta = T * ((1.f + TC_EPS) / (1.f - TC_EPS)) * (1.f + 1e-6f);
        } else {
          theta = T + 2.f * (TC_EPS * anorm * __ldg(p.maxc) + p.slack) + fabsf(T) * 1e-6f;
        }
        theta = fminf(theta, 3.402823466e38f);  // T may be inf (fewer than K finite values): masked columns stay out
        if (qid < 0) theta = -__int_as_float(0x7f800000);  // padding rows take nothing
      }
      tc_mbar_wait(tfull + acc, aph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int64_t y0 = (sweep2 ? t - ntile1 : t * TC_SUB1) * TC_BN;
      const uint32_t col0 = (uint32_t)(2 * acc * TC_BN);
      // warp-uniform: does this tile hold padding columns or any of the warp's queries?
      const bool edge = __any_sync(FULL, y0 + TC_BN > p.n || (qid >= y0 && qid < y0 + TC_BN));
      // columns of chunk c that never rank: the query itself and padding past n
      // (32-bit masks, computed on the rare edge tiles only)
      auto edge_mask = [&](int c) -> unsigned {
        const int64_t yc = y0 + c * 32;
        unsigned em = 0;
        const int64_t sc = qid - yc;
        if (sc >= 0 && sc < 32) em |= 1u << (int)sc;
        const int64_t nv = p.n - yc;
        if (nv < 32) em |= nv <= 0 ? ~0u : (~0u << (int)nv);
        return em;
      };
      if (!sweep2) {
        // sweep 1 (every TC_SUB1-th tile): slot minima, chunk c of tile t -> slot
        // group c % SL (SL = 4: (c + 2) % 4 on odd tiles); one chunk in flight
        // keeps the minima in registers.  Edge tiles take their own loop, so the
        // masking never runs (predicated) on the others.
        auto fold = [&](int c, const uint32_t(&rv)[32]) {
          if (SL == 4 && (t & 1)) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int j = ((c + 2) % SL) * 32 + i;
              best[j] = fminf(best[j], __uint_as_float(rv[i]));
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int j = (c % SL) * 32 + i;
              best[j] = fminf(best[j], __uint_as_float(rv[i]));
            }
          }
        };
        if (!edge) {
#pragma unroll
          for (int c = 0; c < TC_BN / 32; ++c) {
            uint32_t rv[32];
            tc_ld32(lane_base + col0 + c * 32, rv);
            tc_ld_wait(rv);
            fold(c, rv);
          }
        } else {
#pragma unroll 1
          for (int c = 0; c < TC_BN / 32; ++c) {
            uint32_t rv[32];
            tc_ld32(lane_base + col0 + c * 32, rv);
            tc_ld_wait(rv);
            const unsigned em = edge_mask(c);
#pragma unroll
            for (int i = 0; i < 32; ++i) rv[i] = (em >> i) & 1u ? 0x7f800000u : rv[i];
            if (c == 0) fold(0, rv);
            else if (c == 1) fold(1, rv);
            else if (c == 2) fold(2, rv);
            else fold(3, rv);
          }
        }
      } else {
        // sweep 2: append every column with ce <= theta (a 3-input min tree per
        // chunk; the rare hits are walked through a bit mask, minus the edge mask)
#pragma unroll
        for (int c = 0; c < TC_BN / 32; ++c) {
          uint32_t rv[32];
          tc_ld32(lane_base + col0 + c * 32, rv);
          tc_ld_wait(rv);
          float m[11];
#pragma unroll
          for (int i = 0; i < 10; ++i)
            m[i] = tc_min3(__uint_as_float(rv[3 * i]), __uint_as_float(rv[3 * i + 1]), __uint_as_float(rv[3 * i + 2]));
          m[10] = fminf(__uint_as_float(rv[30]), __uint_as_float(rv[31]));
          const float mm = tc_min3(tc_min3(tc_min3(m[0], m[1], m[2]), tc_min3(m[3], m[4], m[5]),
                                           tc_min3(m[6], m[7], m[8])),
                                   m[9], m[10]);
          if (mm <= theta) {  // rare: ~K..3K hits per query over all candidates (and the self tile)
            unsigned hit = 0;
#pragma unroll
            for (int i = 0; i < 32; ++i) hit |= (__uint_as_float(rv[i]) <= theta ? 1u : 0u) << i;
            if (edge) hit &= ~edge_mask(c);
            const int64_t yc = y0 + c * 32;
            while (hit) {
              const int i = __ffs(hit) - 1;
              hit &= hit - 1;
              if (cnt < p.cap) my[cnt] = (int32_t)(yc + i);
              ++cnt;
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) tc_mbar_arrive(tempty + acc);
    }
    if (qa < p.nq) p.count[qa] = cnt;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
}

// max_y |c_y|_2 over the candidate table (non-simplex band), as float bits (>= 0)
__global__ void row_norm_max_kernel(const float *__restrict__ c, int64_t n, int ld, float *out) {
  float m = 0.f;
  for (int64_t y = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; y < n; y += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int j = 0; j < ld; ++j) s = fmaf(c[y * ld + j], c[y * ld + j], s);
    m = fmaxf(m, sqrtf(s) * (1.f + 0x1p-20f));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(FULL, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int *>(out), __float_as_int(m));
}

inline int tc_kt(int ld) { return (ld + 31) / 32; }
inline size_t tc_image_bytes(int64_t n, int ld) {
  return (size_t)((n + TC_BN - 1) / TC_BN) * (size_t)tc_kt(ld) * TC_SUB;
}

// launch the tensor-core screen over the candidate table `cand32` (log32 / L2 cand32)
static int launch_tc_screen(TcParams &p, const float *cand32, unsigned char *image, cudaStream_t st) {
  p.KT = tc_kt(p.ld);
  p.ksteps = (p.ld + 7) / 8;
  // stages: as many 16-KB x KT tiles as fit beside the two A halves (up to 4)
  const int budget = 220 * 1024 - p.KT * TC_Q * 128;
  p.stages = budget / (p.KT * (int)TC_SUB);
  if (p.stages > 4) p.stages = 4;
  if (p.stages < 2) {
    set_error("exact knn: ld32=%d too large for the tensor-core screen", p.ld);
    return KNND_EUNSUPPORTED;
  }
  // kind::tf32, fp32 accumulate, K-major A and B, N = 128, M = 128
  p.idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TC_BN >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);
  {
    int64_t blocks = ((p.n + TC_BN - 1) / TC_BN) * TC_BN * p.KT * 8 / 256;
    if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
    if (blocks < 1) blocks = 1;
    tc_image_kernel<<<(unsigned)blocks, 256, 0, st>>>(cand32, p.n, p.ld, p.KT, image);
    KNND_LAUNCHED(1);
  }
  p.image = image;
  const TcSmem L(p.KT, p.stages);
  const size_t smem = L.total + 1024;
  const unsigned grid = (unsigned)((p.nq + TC_Q - 1) / TC_Q);
  auto launch = [&](auto kern) -> int {
    int per_sm = 0;
    if (int rc = kernel_occupancy((const void *)kern, TC_THREADS, smem, &per_sm)) return rc;
    if (per_sm < 1) {
      set_error("exact knn: the tensor-core screen cannot be resident (smem=%zu)", smem);
      return KNND_EUNSUPPORTED;
    }
    kern<<<grid, TC_THREADS, smem, st>>>(p);
    KNND_LAUNCHED(1);
    return KNND_OK;
  };
  // SLOTS >= K distinct slot minima, and a few times K so the K-th of them is
  // close to the subset's K-th smallest: 32 for K <= 8, 64 for K <= 32, 128 above
  if (p.K <= 8) return launch(exact_tc_kernel<1>);
  if (p.K <= 32) return launch(exact_tc_kernel<2>);
  return launch(exact_tc_kernel<4>);
}

// one warp per query: fp64 rescoring of its candidates, K smallest (score, id)
template <int KPL>
__global__ void exact_rank_kernel(ExactParams p, int32_t *__restrict__ out_ids, double *__restrict__ out_scores) {
  extern __shared__ double sx[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double *x64 = sx + (size_t)w * p.d;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t a = (int64_t)blockIdx.x * (blockDim.x >> 5) + w; a < p.nq; a += warps) {
    const int nc = p.count[a];
    if (nc > p.cap) continue;  // overflow: the caller reruns this query
    const int x = p.queries[a];
    __syncwarp();
    for (int j = lane; j < p.d; j += 32) x64[j] = p.points[(int64_t)x * p.pstride + j];
    __syncwarp();
    const double xl = p.xlogx[x];
    WarpTopK<KeyD, KPL> top;
    top.init();
    const int32_t *c = p.cand + a * p.cap;
    for (int b = 0; b < nc; b += 32) {
      KeyD k = KeyD::inf();
      if (b + lane < nc) {
        const int y = c[b + lane];
        k = {exact_score_m(x64, p.log64 + (int64_t)y * p.d64, p.d, xl, p.metric), y};
      }
      if (b == 0)
        top.first(k, lane);
      else
        top.insert(k, p.K, lane);
    }
#pragma unroll
    for (int q = 0; q < KPL; ++q) {
      const int i = q * 32 + lane;
      if (i < p.K) {
        out_ids[a * p.K + i] = top.b[q].id;
        if (out_scores) out_scores[a * p.K + i] = top.b[q].s;
      }
    }
  }
}

}  // namespace knnd

using namespace knnd;

extern "C" {

size_t knnd_exact_knn_workspace_bytes(int64_t n, int32_t ld32, int64_t nq, int32_t cap) {
  if (n < 1 || ld32 < 1 || nq < 0 || cap < 1) return 0;
  // candidate lists, the tensor-core image of the candidate table, the norm bound
  return align_up((size_t)nq * (size_t)cap * 4, 256) + align_up(tc_image_bytes(n, ld32), 256) + 256;
}

static int exact_run(const char *who, ExactParams &p, int32_t dplan, int32_t k, void *ws, size_t ws_bytes,
                     void *stream) {
  const int64_t n = p.n, nq = p.nq;
  const int32_t d = p.d, ld32 = p.ld, cap = p.cap;
  KNND_CHECK_ARG(p.count && (nq == 0 || (p.queries && p.out_ids)), "%s: null pointer", who);
  KNND_CHECK_ARG(n >= 2 && d >= 1, "%s: bad shape n=%lld d=%d", who, (long long)n, d);
  KNND_CHECK_ARG(ld32 >= dplan && ld32 % 4 == 0, "%s: ld32=%d must be >= %d and a multiple of 4", who, ld32, dplan);
  KNND_CHECK_ARG(n < ((int64_t)1 << 31), "%s: n must be < 2^31", who);
  KNND_CHECK_ARG(cap >= 1 && nq >= 0, "%s: bad cap %d / nq %lld", who, cap, (long long)nq);
  if (k < 1 || k > 64 || k >= n) {
    set_error("%s: K=%d unsupported (1..64, < n)", who, k);
    return KNND_EUNSUPPORTED;
  }
  if (nq == 0) return KNND_OK;
  const size_t need = knnd_exact_knn_workspace_bytes(n, ld32, nq, cap);
  if (!ws || ws_bytes < need) {
    set_error("%s: workspace %zu < %zu bytes", who, ws_bytes, need);
    return KNND_EWORKSPACE;
  }
  cudaStream_t st = as_stream(stream);
  p.K = k;
  p.cand = static_cast<int32_t *>(ws);
  TcParams t{};
  t.points = p.points;
  t.aside32 = p.aside32;
  t.pstride = p.pstride;
  t.d = p.d;
  t.ld = p.ld;
  t.n = p.n;
  t.queries = p.queries;
  t.nq = nq;
  t.K = k;
  t.nonpos = p.nonpos;
  t.slack = p.slack;
  t.cand = p.cand;
  t.cap = cap;
  t.count = p.count;
  const size_t list_bytes = align_up((size_t)nq * (size_t)cap * 4, 256);
  unsigned char *image = static_cast<unsigned char *>(ws) + list_bytes;
  if (!p.nonpos) {  // the candidate rows' largest norm, for the Cauchy-Schwarz band
    float *maxc = reinterpret_cast<float *>(image + align_up(tc_image_bytes(n, ld32), 256));
    KNND_CUDA(cudaMemsetAsync(maxc, 0, sizeof(float), st));
    row_norm_max_kernel<<<num_sms() * 4, 256, 0, st>>>(p.log32, n, ld32, maxc);
    KNND_LAUNCHED(1);
    t.maxc = maxc;
  }
  if (int rc = launch_tc_screen(t, p.log32, image, st)) return rc;
  const int wpb = 8;
  int64_t blocks = (nq + wpb - 1) / wpb;
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
  const size_t smem = (size_t)wpb * d * sizeof(double);
  if (k <= 32)
    exact_rank_kernel<1><<<(unsigned)blocks, wpb * 32, smem, st>>>(p, p.out_ids, p.out_scores);
  else
    exact_rank_kernel<2><<<(unsigned)blocks, wpb * 32, smem, st>>>(p, p.out_ids, p.out_scores);
  KNND_LAUNCHED(1);
  return KNND_OK;
}

int knnd_exact_knn(const double *points, const float *log32, const double *log64, const double *xlogx, int64_t n,
                   int32_t d, int32_t ld32, const int32_t *queries, int64_t nq, int32_t k, int32_t cap,
                   int32_t *out_ids, double *out_scores, int32_t *out_count, void *ws, size_t ws_bytes,
                   uint32_t flags, void *stream) {
  KNND_CHECK_ARG(points && log32 && log64 && xlogx, "knnd_exact_knn: null pointer");
  ExactParams p{};
  p.points = points;
  p.log32 = log32;
  p.log64 = log64;
  p.xlogx = xlogx;
  p.n = n;
  p.d = d;
  p.ld = ld32;
  p.queries = queries;
  p.nq = nq;
  p.nonpos = (flags & KNND_JOIN_NONPOS_LOG) ? 1 : 0;
  p.cap = cap;
  p.count = out_count;
  p.out_ids = out_ids;
  p.out_scores = out_scores;
  p.metric = METRIC_KL;
  p.d64 = d;
  p.pstride = d;
  return exact_run("knnd_exact_knn", p, d, k, ws, ws_bytes, stream);
}

int knnd_l2_exact_knn(const float *anchor32, const float *cand32, const double *rows64, const double *sq64,
                      int64_t n, int32_t d, int32_t ld32, double maxnorm, const int32_t *queries, int64_t nq,
                      int32_t k, int32_t cap, int32_t *out_ids, double *out_d2, int32_t *out_count, void *ws,
                      size_t ws_bytes, void *stream) {
  KNND_CHECK_ARG(anchor32 && cand32 && rows64 && sq64, "knnd_l2_exact_knn: null pointer");
  ExactParams p{};
  p.points = rows64;
  p.log32 = cand32;
  p.log64 = rows64;
  p.xlogx = sq64;
  p.n = n;
  p.d = d;
  p.ld = ld32;
  p.queries = queries;
  p.nq = nq;
  p.nonpos = 0;
  p.cap = cap;
  p.count = out_count;
  p.out_ids = out_ids;
  p.out_scores = out_d2;
  p.metric = METRIC_L2;
  p.d64 = d + 1;
  p.pstride = d + 1;
  p.aside32 = anchor32;
  p.slack = (float)((d + 4) * 0x1p-53 * 4.0 * maxnorm * maxnorm);
  return exact_run("knnd_l2_exact_knn", p, d + 1, k, ws, ws_bytes, stream);
}

}  // extern "C"

KNND_CHECK_READER(exact, 2)
