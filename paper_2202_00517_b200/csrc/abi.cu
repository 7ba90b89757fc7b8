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

}  // extern "C"
