// Internal plumbing shared by every translation unit of libcatgnn.so:
// error categories (mirroring proj/include/gnnpart/common.hpp:16-24),
// CUDA checking, device buffers and the per-device context.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <initializer_list>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "catgnn.h"

namespace catgnn {

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InternalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);

// Runs fn, translating exceptions into the ABI's return codes.
template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return CATGNN_OK;
  } catch (const ConfigError& e) {
    set_last_error(std::string("bad-config: ") + e.what());
    return CATGNN_ECONFIG;
  } catch (const DataError& e) {
    set_last_error(std::string("bad-input: ") + e.what());
    return CATGNN_EDATA;
  } catch (const std::exception& e) {
    set_last_error(std::string("internal: ") + e.what());
    return CATGNN_EINTERNAL;
  }
}

#define CG_CUDA(expr)                                                                       \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      throw ::catgnn::InternalError(std::string("CUDA: ") + cudaGetErrorString(e_) + " (" + \
                                    #expr + ") at " + __FILE__ + ":" +                      \
                                    std::to_string(__LINE__));                              \
  } while (0)

#define CG_CHECK_LAUNCH() CG_CUDA(cudaGetLastError())

// Owning device buffer (cudaMalloc; grow-only reserve for scratch).
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    release();
    if (count == 0) return;
    CG_CUDA(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void reserve(size_t count) {
    if (count > n) alloc(count);
  }
  size_t bytes() const { return n * sizeof(T); }
};

inline uint32_t round_up(uint32_t x, uint32_t m) { return (x + m - 1) / m * m; }
inline uint64_t round_up64(uint64_t x, uint64_t m) { return (x + m - 1) / m * m; }

}  // namespace catgnn

// Per-device context: stream, SM count, scratch pool, launch accounting and
// optional per-kernel event timing for the roofline measurement.
struct catgnn_ctx_s {
  int device = 0;
  int refs = 1;  // the owner handle + every shard / model / comm created on it
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  uint64_t launches = 0;
  // kernel timing (K2 aggregation, K3 GEMM)
  bool timing = false;
  struct Pending {
    cudaEvent_t a, b;
    int kind;  // 0 agg, 1 gemm, 2 other (label only)
    std::string label;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  std::vector<cudaEvent_t> order_events;  // ring of events for wait_for
  size_t order_next = 0;
  double agg_ms = 0, gemm_ms = 0;
  // per-label totals of the timed launches (step breakdown diagnostics)
  std::map<std::string, std::pair<double, uint64_t>> by_label;
  uint64_t agg_n = 0, gemm_n = 0;
  // named grow-only scratch buffers
  std::map<std::string, catgnn::DevBuf<unsigned char>> scratch;
  // last (rows, row stride) each named activation buffer was used with
  std::map<std::string, std::pair<uint64_t, uint32_t>> act_shape;

  template <typename T>
  T* scratch_buf(const std::string& name, size_t count) {
    auto& b = scratch[name];
    b.reserve(count * sizeof(T));
    return reinterpret_cast<T*>(b.p);
  }
  // Free the named scratch buffers whose names start with one of `prefixes`
  // (after the stream drained): one-time temporaries — K1's sort buffers, the
  // edge-mapping staging — do not stay resident next to the activations.
  void release_scratch(std::initializer_list<const char*> prefixes) {
    cudaStreamSynchronize(stream);
    for (auto it = scratch.begin(); it != scratch.end();) {
      bool hit = false;
      for (const char* p : prefixes) hit = hit || it->first.rfind(p, 0) == 0;
      it = hit ? scratch.erase(it) : std::next(it);
    }
  }
  cudaEvent_t take_event();
  // SMs the persistent K2 grid covers and CTAs (SMs) the persistent K3 grid
  // uses; 0 = all.  Budgets < num_sms let kernels of contexts on other
  // streams run beside them (shard lanes, catgnn_ctx_set_sm_budget).
  int agg_sms = 0, gemm_sms = 0;
  // Make this context's stream wait for the work enqueued so far on `other`'s
  // stream (no-op for the same stream); capturable.
  void wait_for(const catgnn_ctx_s* other);
  // Bracket a kernel for timing; returns an index to close with end_timed.
  int begin_timed(int kind, std::string label = std::string());
  void end_timed(int idx);
  void drain_timing();
  ~catgnn_ctx_s();
};

namespace catgnn {
inline void ctx_retain(catgnn_ctx c) { c->refs++; }
// Drops one reference; the context is freed with its last user.
inline void ctx_release(catgnn_ctx c) {
  if (c && --c->refs == 0) delete c;
}
}  // namespace catgnn
