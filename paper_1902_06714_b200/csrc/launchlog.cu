// launchlog.cu -- debug record of every kernel launch of this library (template
// instantiation, grid, block, dynamic shared memory, runtime variant), so that tests can show
// which instantiations a workload launches and that each one is covered by an oracle-compared
// parity test.  Enabled by NF_LOG_LAUNCHES=1 at load or nf_debug_log_enable(1); off by
// default (one relaxed load per launch).
#include <cxxabi.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <tuple>
#include <string>

#include "../../include/nf.h"
#include "kernels.cuh"

namespace nf {
namespace {
std::atomic<int> g_log_on{-1};
std::mutex g_log_mu;
std::string g_log;
}  // namespace

bool launch_log_on() {
  int v = g_log_on.load(std::memory_order_relaxed);
  if (v < 0) {
    const char *e = getenv("NF_LOG_LAUNCHES");
    v = (e && atoi(e)) ? 1 : 0;
    int expect = -1;
    g_log_on.compare_exchange_strong(expect, v);
    v = g_log_on.load();
  }
  return v == 1;
}

void host_trace(const char *what) {
  static const bool on = getenv("NF_TRACE_HOST") != nullptr;
  if (!on) return;
  static thread_local std::chrono::steady_clock::time_point t0;
  const auto t = std::chrono::steady_clock::now();
  if (!strcmp(what, "enter")) t0 = t;
  fprintf(stderr, "[host] %-12s %8.2f us\n", what, std::chrono::duration<double, std::micro>(t - t0).count());
}

cudaError_t set_max_smem(const void *kern, int bytes) {
  static std::mutex mu;
  static std::set<std::tuple<const void *, int, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const auto key = std::make_tuple(kern, dev, bytes);
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(key)) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert(key);
  return e;
}

void log_launch(const void *func, dim3 grid, dim3 block, size_t smem, const char *note) {
  if (!launch_log_on()) return;
  const char *name = nullptr;
  std::string nm = "?";
  if (cudaFuncGetName(&name, func) == cudaSuccess && name) {
    int st = 0;
    char *d = abi::__cxa_demangle(name, nullptr, nullptr, &st);
    nm = (st == 0 && d) ? d : name;
    free(d);
  } else {
    cudaGetLastError();
  }
  char buf[160];
  snprintf(buf, sizeof buf, " grid=(%u,%u,%u) block=%u smem=%zu%s%s\n", grid.x, grid.y, grid.z,
           block.x * block.y * block.z, smem, note && *note ? " " : "", note ? note : "");
  std::lock_guard<std::mutex> lk(g_log_mu);
  g_log += nm;
  g_log += buf;
}

}  // namespace nf

extern "C" {
void nf_debug_log_enable(int on) {
  std::lock_guard<std::mutex> lk(nf::g_log_mu);
  nf::g_log.clear();
  nf::g_log_on.store(on ? 1 : 0);
}

int64_t nf_debug_log_read(char *buf, int64_t cap) {
  std::lock_guard<std::mutex> lk(nf::g_log_mu);
  const int64_t need = (int64_t)nf::g_log.size() + 1;
  if (buf && cap > 0) {
    const int64_t n = need < cap ? need - 1 : cap - 1;
    memcpy(buf, nf::g_log.data(), (size_t)n);
    buf[n] = 0;
  }
  return need;
}
}
