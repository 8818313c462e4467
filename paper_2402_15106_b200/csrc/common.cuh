// common.cuh - shared helpers of libdsmpnn.so (sm_100a).  Status handling,
// workspace carving, launch helpers.  No method arithmetic lives here except
// the counter hash (hash.cuh).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/dsmpnn.h"

namespace dsmpnn {

void set_error(const char *fmt, ...);

#define DS_CHECK_ARG(cond, code, ...)      \
  do {                                     \
    if (!(cond)) {                         \
      ::dsmpnn::set_error(__VA_ARGS__);    \
      return code;                         \
    }                                      \
  } while (0)

#define DS_CUDA(expr)                                                                   \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess) {                                                            \
      ::dsmpnn::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e), __FILE__,  \
                          __LINE__, cudaGetErrorString(_e));                            \
      return DSMPNN_ERR_CUDA;                                                           \
    }                                                                                   \
  } while (0)

#define DS_LAUNCH_CHECK() DS_CUDA(cudaGetLastError())

#define DS_TRY(expr)                       \
  do {                                     \
    dsmpnn_status _s = (expr);             \
    if (_s != DSMPNN_OK) return _s;        \
  } while (0)

static inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Bump allocator over a caller-provided workspace (256-byte aligned slices).
struct Carver {
  char *base;
  size_t cap;
  size_t off = 0;
  Carver(void *b, size_t c) : base(static_cast<char *>(b)), cap(c) {}
  template <typename T>
  T *take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T *p = reinterpret_cast<T *>(base ? base + off : nullptr);
    off += count * sizeof(T);
    return p;
  }
  bool ok() const { return off <= cap; }
  size_t used() const { return (off + 255) & ~size_t(255); }
};

static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

constexpr int kNumSMs = 148;

// Programmatic dependent launch (PDL) along the layer's kernel chain: the
// chain's kernels are launched with launch_pdl (stream attribute
// ProgrammaticStreamSerialization) and each calls pdl_wait() before it reads
// or writes data of another kernel (weights packed by dsmpnn_pack_weights and
// the graph arrays may be read earlier: no kernel that lets its successor
// start early writes them), then pdl_trigger(), so its successor's launch and
// prologue (barrier init, TMEM allocation, resident weight loads) overlap its
// own tail (with the early trigger, see below).  A kernel launched without
// the attribute passes pdl_wait at once.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// The early trigger (successor CTAs launched while this grid's last CTAs run)
// shortens the layer chain a little more (8.23 vs 8.29 ms per Darcy step of
// layers) but its resident successor CTAs take every SM a finishing CTA
// frees, so the next step's graph build on the high-priority stream starves
// and the pipelined step slows from 8.6 to 9.5 ms: by default successors
// launch at the grid's completion (the implicit trigger), which still hides
// the launch latency between the chain's kernels.
#ifdef DSMPNN_PDL_EARLY_TRIGGER
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#else
__device__ __forceinline__ void pdl_trigger() {}
#endif
bool pdl_enabled();  // DSMPNN_PDL=0 turns the launch attribute off (A/B timing)

template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// live timing probe (dsmpnn_probe_begin/end): true if launches of `id` are recorded
bool probe_armed(int id);
void probe_before(int id, cudaStream_t s);
void probe_after(int id, cudaStream_t s);
struct ProbeScope {
  int id;
  cudaStream_t s;
  bool on;
  ProbeScope(int id_, cudaStream_t s_) : id(id_), s(s_), on(probe_armed(id_)) { if (on) probe_before(id, s); }
  ~ProbeScope() { if (on) probe_after(id, s); }
};

#ifdef DSMPNN_TIMELINE
// development builds: print the clock64 timeline of CTA 0 (slots relative to
// the first stamp of tile 0), one line per tile
static inline void dump_timeline(const char *name, const unsigned long long *dbg, int nslots, cudaStream_t s) {
  unsigned long long h[32 * 32];
  cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  unsigned long long t0 = ~0ull;
  for (int k = 0; k < 32 * 32; ++k)
    if (h[k] && h[k] < t0) t0 = h[k];
  fprintf(stderr, "%s timeline (cycles since first stamp), tiles x slots\n", name);
  for (int t = 0; t < 16; ++t) {
    fprintf(stderr, "t%02d", t);
    for (int k = 0; k < nslots; ++k) fprintf(stderr, " %7lld", h[t * 32 + k] ? (long long)(h[t * 32 + k] - t0) : -1ll);
    fprintf(stderr, "\n");
  }
}
#endif

}  // namespace dsmpnn
