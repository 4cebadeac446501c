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
// Release a dalloc'd buffer (stream-ordered on the legacy stream; callers that
// may still have work in flight on other streams synchronise first).
void dfree(void *p);
template <class T>
int dalloc(T **p, size_t count, const char *what) {
    return dalloc(reinterpret_cast<void **>(p), count * sizeof(T), what);
}

// Count of this library's kernel launches (reported by the PCG loop).
extern int64_t g_launches;
inline void count_launch(int64_t n = 1) { g_launches += n; }

}  // namespace lp
