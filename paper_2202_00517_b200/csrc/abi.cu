// C-ABI bookkeeping: per-thread last-error string, launch counter, SM count.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace knnd {

static thread_local char g_err[1024] = "";
static std::atomic<unsigned long long> g_launches{0};

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void count_launch(unsigned n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

namespace {
struct OccKey {
  int dev, block;
  const void *kern;
  size_t smem;
  bool operator==(const OccKey &o) const {
    return dev == o.dev && block == o.block && kern == o.kern && smem == o.smem;
  }
};
struct OccKeyHash {
  size_t operator()(const OccKey &k) const {
    return std::hash<const void *>()(k.kern) ^ (std::hash<size_t>()(k.smem) * 31) ^ ((size_t)k.block << 20) ^
           ((size_t)k.dev << 40);
  }
};
std::mutex g_occ_mu;
std::unordered_map<OccKey, int, OccKeyHash> g_occ;                      // -> blocks per SM
std::unordered_map<const void *, size_t> g_smem_attr[64];               // per device: the smem limit set
}  // namespace

int kernel_occupancy(const void *kern, int block, size_t smem, int *per_sm) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    set_error("kernel_occupancy: no current device");
    return KNND_ECUDA;
  }
  std::lock_guard<std::mutex> lock(g_occ_mu);
  const OccKey key{dev, block, kern, smem};
  auto it = g_occ.find(key);
  if (it != g_occ.end()) {
    *per_sm = it->second;
    return KNND_OK;
  }
  size_t &lim = g_smem_attr[dev][kern];
  if (smem > lim) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      set_error("cudaFuncSetAttribute(smem=%zu) failed: %s", smem, cudaGetErrorString(e));
      return KNND_ECUDA;
    }
    lim = smem;
  }
  int n = 0;
  const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, block, smem);
  if (e != cudaSuccess) {
    set_error("occupancy query failed: %s", cudaGetErrorString(e));
    return KNND_ECUDA;
  }
  g_occ.emplace(key, n);
  *per_sm = n;
  return KNND_OK;
}

int num_sms() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

}  // namespace knnd

extern "C" {

int knnd_abi_version(void) { return KNND_ABI_VERSION; }

const char *knnd_last_error(void) { return knnd::g_err; }

unsigned long long knnd_launch_count(void) { return knnd::g_launches.load(); }

int knnd_check_failures(unsigned long long *count, unsigned long long *first) {
  if (!count || !first) return KNND_EINVAL;
  *count = 0;
  *first = 0;
#ifdef KNND_CHECKED
  int rc = KNND_OK;
  if ((rc = knnd::check_read_abi(count, first)) || (rc = knnd::check_read_join(count, first)) ||
      (rc = knnd::check_read_join_f32k2(count, first)) || (rc = knnd::check_read_join_q23(count, first)) || (rc = knnd::check_read_exact(count, first)) ||
      (rc = knnd::check_read_csr(count, first)) || (rc = knnd::check_read_prep(count, first)) ||
      (rc = knnd::check_read_rng(count, first))) {
    knnd::set_error("knnd_check_failures: reading the check words failed");
    return rc;
  }
  return KNND_OK;
#else
  knnd::set_error("knnd_check_failures: this is the product build (checks compiled out)");
  return KNND_EUNSUPPORTED;
#endif
}

#ifdef KNND_CHECKED
// not part of knnd.h: a kernel whose checks fail on purpose (lanes 3 and 5), so
// tests can see the checked build's reporting work end to end
__global__ void check_selftest_kernel() { KNND_DCHECK(threadIdx.x != 3 && threadIdx.x != 5); }
int knnd_internal_check_selftest(void *stream) {
  check_selftest_kernel<<<1, 32, 0, knnd::as_stream(stream)>>>();
  return cudaGetLastError() == cudaSuccess ? KNND_OK : KNND_ECUDA;
}
#endif

}  // extern "C"

KNND_CHECK_READER(abi, 9)
