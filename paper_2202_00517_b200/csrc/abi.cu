// C-ABI bookkeeping: per-thread last-error string, launch counter, SM count.
#include <atomic>
#include <cstdarg>
#include <cstdio>

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
  if ((rc = knnd::check_read_abi(count, first)) || (rc = knnd::check_read_join(count, first)) || (rc = knnd::check_read_exact(count, first)) ||
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
