// Brute-force exact K nearest neighbours for a set of queries — the ground
// truth behind recall (evaluation.py:83-90 exact_knn, per query x:
//   s = batch_scores(x); s[x] = inf; row = _smallest_k(s, K)   (evaluation.py:53-71)
// i.e. the K smallest (fp64 score, id) over every other point).
//
// Same screen-then-rescore scheme as the local join, over all n candidates:
//   sweep 1  every query against every candidate in fp32 (a 64-query x
//            128-candidate tile per block step, log rows staged in shared memory
//            by cp.async, 8 queries x 4 candidates per thread); each lane keeps
//            its Q smallest screened values per query -> T_q >= the K-th
//            smallest (warp sorting networks);
//   sweep 2  the same scores again; every candidate with ce <= theta_q (T_q plus
//            the rigorous fp32 error band) is appended to the query's list;
//   rank     one warp per query rescoring its list in fp64 (score.cuh, the
//            join's exact scorer) and keeping the K smallest (score, id).
// A list longer than `cap` is reported through out_count and the caller reruns
// that query with a larger cap (never silently truncated).
#include "common.cuh"
#include "score.cuh"

namespace knnd {

constexpr int XQW = 8;             // queries per warp
constexpr int XWARPS = 8;          // warps per block
constexpr int XQB = XQW * XWARPS;  // queries per block
constexpr int XT = 128;            // candidate rows per staged tile (4 per lane)

struct ExactParams {
  const double *points;
  const float *log32;
  const double *log64;
  const double *xlogx;
  int64_t n;
  int d, ld, K;
  const int32_t *queries;
  int64_t nq;
  float band;  // relative fp32 screen error bound (see knnd_local_join)
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

template <int NV4, int Q, bool ABS>
__global__ void __launch_bounds__(XWARPS * 32) exact_screen_kernel(ExactParams p) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nv4 = NV4 > 0 ? NV4 : p.ld / 4;
  const int ld = p.ld;
  float *xq = reinterpret_cast<float *>(sm);                 // XQB x ld
  float *tiles = xq + (size_t)XQB * ld;                      // 2 x XT x ld
  const int64_t qb = (int64_t)blockIdx.x * XQB;
  // query rows (fp32 copies of the points), zero padded
  for (int i = threadIdx.x; i < XQB * ld; i += blockDim.x) {
    const int r = i / ld, j = i % ld;
    float v = 0.f;
    if (qb + r < p.nq) {
      const int64_t x = p.queries[qb + r];
      if (p.aside32)
        v = p.aside32[x * ld + j];
      else if (j < p.d)
        v = (float)p.points[x * p.pstride + j];
    }
    xq[i] = v;
  }
  int qid[XQW];
#pragma unroll
  for (int qq = 0; qq < XQW; ++qq) {
    const int64_t a = qb + warp * XQW + qq;
    qid[qq] = a < p.nq ? p.queries[a] : -1;
  }
  const int64_t ntiles = (p.n + XT - 1) / XT;
  auto stage = [&](int64_t t, int buf) {
    const int64_t r0 = t * XT;
    const int rows = (int)min((int64_t)XT, p.n - r0);
    const int chunks = rows * ld / 4;
    const float *src = p.log32 + r0 * ld;
    float *dst = tiles + (size_t)buf * XT * ld;
    for (int c = threadIdx.x; c < chunks; c += blockDim.x) cp_async16(dst + c * 4, src + c * 4);
    cp_async_commit();
  };

  float best[XQW][Q];
  float am[XQW];
  float theta[XQW];
  int cnt[XQW];
#pragma unroll
  for (int qq = 0; qq < XQW; ++qq) {
#pragma unroll
    for (int q = 0; q < Q; ++q) best[qq][q] = __int_as_float(0x7f800000);
    am[qq] = 0.f;
    cnt[qq] = 0;
    theta[qq] = 0.f;
  }

  for (int sweep = 0; sweep < 2; ++sweep) {
    stage(0, 0);
    for (int64_t t = 0; t < ntiles; ++t) {
      const int buf = (int)(t & 1);
      if (t + 1 < ntiles) {
        stage(t + 1, buf ^ 1);
        cp_async_wait_1();
      } else {
        cp_async_wait_0();
      }
      __syncthreads();
      const float4 *rows4 = reinterpret_cast<const float4 *>(tiles + (size_t)buf * XT * ld);
      const float4 *xq4 = reinterpret_cast<const float4 *>(xq) + (size_t)warp * XQW * nv4;
      float acc[XQW][4];
      float aab[ABS ? XQW : 1][4];
#pragma unroll
      for (int qq = 0; qq < XQW; ++qq)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[qq][i] = 0.f;
          if constexpr (ABS) aab[qq][i] = 0.f;
        }
#pragma unroll(NV4 > 0 ? NV4 : 1)
      for (int c = 0; c < nv4; ++c) {
        float4 cv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) cv[i] = rows4[(size_t)(lane + 32 * i) * nv4 + c];
#pragma unroll
        for (int qq = 0; qq < XQW; ++qq) {
          const float4 xv = xq4[qq * nv4 + c];  // broadcast
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            acc[qq][i] = fmaf(-xv.x, cv[i].x, acc[qq][i]);
            acc[qq][i] = fmaf(-xv.y, cv[i].y, acc[qq][i]);
            acc[qq][i] = fmaf(-xv.z, cv[i].z, acc[qq][i]);
            acc[qq][i] = fmaf(-xv.w, cv[i].w, acc[qq][i]);
            if constexpr (ABS) {
              aab[qq][i] = fmaf(fabsf(xv.x), fabsf(cv[i].x), aab[qq][i]);
              aab[qq][i] = fmaf(fabsf(xv.y), fabsf(cv[i].y), aab[qq][i]);
              aab[qq][i] = fmaf(fabsf(xv.z), fabsf(cv[i].z), aab[qq][i]);
              aab[qq][i] = fmaf(fabsf(xv.w), fabsf(cv[i].w), aab[qq][i]);
            }
          }
        }
      }
      // candidates past n, and each query itself, never rank (s[x] = inf)
      const int64_t y0 = t * XT + lane;
      const bool edge = (t + 1) * XT > p.n;
      bool self = false;
#pragma unroll
      for (int qq = 0; qq < XQW; ++qq) self |= qid[qq] >= t * XT && qid[qq] < (t + 1) * XT;
      if (__any_sync(FULL, edge || self)) {
#pragma unroll
        for (int qq = 0; qq < XQW; ++qq)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int64_t y = y0 + 32 * i;
            if (y >= p.n || y == qid[qq]) {
              acc[qq][i] = __int_as_float(0x7f800000);
              if constexpr (ABS) aab[qq][i] = 0.f;
            }
          }
      }
      if (sweep == 0) {
#pragma unroll
        for (int qq = 0; qq < XQW; ++qq)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float v = acc[qq][i];
#pragma unroll
            for (int q = 0; q < Q; ++q) {  // insertion into the sorted per-lane list
              const float lo_ = fminf(best[qq][q], v);
              v = fmaxf(best[qq][q], v);
              best[qq][q] = lo_;
            }
            if constexpr (ABS) am[qq] = fmaxf(am[qq], aab[qq][i]);
          }
      } else {
        bool any = false;
#pragma unroll
        for (int qq = 0; qq < XQW; ++qq)
#pragma unroll
          for (int i = 0; i < 4; ++i) any |= acc[qq][i] <= theta[qq];
        if (__any_sync(FULL, any)) {
#pragma unroll
          for (int qq = 0; qq < XQW; ++qq) {
            const int64_t a = qb + warp * XQW + qq;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const bool take = acc[qq][i] <= theta[qq] && acc[qq][i] < __int_as_float(0x7f800000);
              const unsigned m = __ballot_sync(FULL, take);
              if (take) {
                const int r = cnt[qq] + __popc(m & lanemask_lt());
                if (r < p.cap) p.cand[a * p.cap + r] = (int32_t)(y0 + 32 * i);
              }
              cnt[qq] += __popc(m);
            }
          }
        }
      }
      __syncthreads();  // the buffer is restaged two tiles later
    }
    if (sweep == 0) {
      // T_q >= the K-th smallest screened value; theta_q adds the error band
#pragma unroll
      for (int qq = 0; qq < XQW; ++qq) {
        float T;
        if constexpr (Q == 2) {
          const KeyF a = warp_sort32(KeyF{best[qq][0]}, lane);
          const KeyF b = warp_sort32_desc(KeyF{best[qq][1]}, lane);
          const KeyF m = warp_merge32(kmin(a, b), lane);
          T = m.shfl(p.K - 1).v;
        } else {
          WarpTopK<KeyF, 2> top;
          top.init();
          top.first(KeyF{best[qq][0]}, lane);
#pragma unroll
          for (int q = 1; q < Q; ++q) top.insert(KeyF{best[qq][q]}, p.K, lane);
          T = top.get(p.K - 1).v;
        }
        float th;
        if (p.nonpos) {
          // ab == ce >= 0 for every candidate: |ce - exact| <= band * ce
          th = T + T * (2.f * p.band + 1e-6f);
        } else {
          float a = am[qq];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) a = fmaxf(a, __shfl_xor_sync(FULL, a, o));
          th = T + 2.f * (p.band * a + p.slack) + fabsf(T) * 1e-6f;
        }
        theta[qq] = qid[qq] >= 0 ? th : -__int_as_float(0x7f800000);  // padding queries take nothing
      }
    }
  }
#pragma unroll
  for (int qq = 0; qq < XQW; ++qq) {
    const int64_t a = qb + warp * XQW + qq;
    if (lane == 0 && a < p.nq) p.count[a] = cnt[qq];
  }
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

template <int NV4, int Q>
static int launch_screen(const ExactParams &p, cudaStream_t st) {
  const size_t smem = ((size_t)XQB * p.ld + 2 * (size_t)XT * p.ld) * sizeof(float);
  if (smem > 227 * 1024) {
    set_error("exact knn: d=%d too large for the staged tiles", p.d);
    return KNND_EUNSUPPORTED;
  }
  const unsigned grid = (unsigned)((p.nq + XQB - 1) / XQB);
  if (p.nonpos) {
    auto k = exact_screen_kernel<NV4, Q, false>;
    KNND_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, XWARPS * 32, smem, st>>>(p);
  } else {
    auto k = exact_screen_kernel<NV4, Q, true>;
    KNND_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, XWARPS * 32, smem, st>>>(p);
  }
  KNND_LAUNCHED(1);
  return KNND_OK;
}

template <int Q>
static int dispatch_screen(const ExactParams &p, cudaStream_t st) {
  switch (p.ld / 4) {
    case 2: return launch_screen<2, Q>(p, st);
    case 3: return launch_screen<3, Q>(p, st);
    case 5: return launch_screen<5, Q>(p, st);
    case 13: return launch_screen<13, Q>(p, st);
    default: return launch_screen<0, Q>(p, st);
  }
}

}  // namespace knnd

using namespace knnd;

extern "C" {

size_t knnd_exact_knn_workspace_bytes(int64_t nq, int32_t cap) {
  if (nq < 0 || cap < 1) return 0;
  return align_up((size_t)nq * (size_t)cap * 4, 256) + 256;
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
  const size_t need = knnd_exact_knn_workspace_bytes(nq, cap);
  if (!ws || ws_bytes < need) {
    set_error("%s: workspace %zu < %zu bytes", who, ws_bytes, need);
    return KNND_EWORKSPACE;
  }
  cudaStream_t st = as_stream(stream);
  p.K = k;
  p.band = (float)((ld32 + 8) * 0x1p-24);
  p.cand = static_cast<int32_t *>(ws);
  const int rc = k <= 32 ? dispatch_screen<2>(p, st) : dispatch_screen<4>(p, st);
  if (rc) return rc;
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
