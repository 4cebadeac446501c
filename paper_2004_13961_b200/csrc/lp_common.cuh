// Shared helpers for the legpcg_b200 CUDA library (sm_100a, fp64).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/legpcg_b200.h"

namespace lp {

void set_error(const char *fmt, ...);
int cuda_fail(cudaError_t e, const char *what, const char *file, int line);

#define LP_CUDA(call)                                                          \
    do {                                                                       \
        cudaError_t e_ = (call);                                               \
        if (e_ != cudaSuccess) return lp::cuda_fail(e_, #call, __FILE__, __LINE__); \
    } while (0)

#define LP_CHECK_LAUNCH() LP_CUDA(cudaGetLastError())

#define LP_ARG(cond, ...)                                                      \
    do {                                                                       \
        if (!(cond)) { lp::set_error(__VA_ARGS__); return LP_ERR_ARG; }        \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// Device allocation that records an LP_ERR_OOM message on failure.
int dalloc(void **p, size_t bytes, const char *what);
// Release a dalloc'd buffer, stream-ordered after the work already queued on
// `st` (the legacy stream by default; pass the stream that last used it).
void dfree(void *p, cudaStream_t st = nullptr);
template <class T>
int dalloc(T **p, size_t count, const char *what) {
    return dalloc(reinterpret_cast<void **>(p), count * sizeof(T), what);
}

// Multiprocessor count of the current device (cached per device).
int num_sms();
// Stream-ordered scratch from the device pool: no device synchronisation, so
// per-call workspaces are cheap and concurrent calls on different streams get
// their own buffers.  The buffer may be used on `st` only (or after an event).
int salloc(void **p, size_t bytes, const char *what, cudaStream_t st);
template <class T>
int salloc(T **p, size_t count, const char *what, cudaStream_t st) {
    return salloc(reinterpret_cast<void **>(p), count * sizeof(T), what, st);
}
void sfree(void *p, cudaStream_t st);

// Resident CTAs of kernel `fn` on the whole device (occupancy x SMs) with
// `threads` per CTA and `smem` dynamic shared memory; sets the kernel's
// dynamic-smem limit first.  Cached per (device, kernel, threads, smem),
// thread-safe.  Returns 0 when the kernel does not fit an SM.
int resident_blocks(const void *fn, int threads, size_t smem);
// Same for thread-block clusters of `csize` CTAs (non-portable sizes allowed):
// resident clusters x csize, or 0.
int resident_cluster_blocks(const void *fn, int threads, size_t smem, int csize);

// Count of this library's kernel launches (reported by the PCG loop).
extern int64_t g_launches;
inline void count_launch(int64_t n = 1) { g_launches += n; }

}  // namespace lp
