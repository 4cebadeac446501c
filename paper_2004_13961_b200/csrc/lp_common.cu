// Error state, device checks and allocation helpers.
#include <stdarg.h>

#include "lp_common.cuh"

namespace lp {

static thread_local std::string t_error;
int64_t g_launches = 0;

void set_error(const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    t_error = buf;
}

int cuda_fail(cudaError_t e, const char *what, const char *file, int line) {
    set_error("CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
              cudaGetErrorString(e), what, file, line);
    return e == cudaErrorMemoryAllocation ? LP_ERR_OOM : LP_ERR_CUDA;
}

// Library buffers come from the device's default stream-ordered memory pool
// with an unbounded release threshold, so the per-solve factor and workspace
// buffers (hundreds of MB) are recycled instead of hitting cudaMalloc/cudaFree
// (which also synchronise the device) on every pcg_solve.
static void init_pool() {
    static bool done = false;
    if (done) return;
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t threshold = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
    }
    cudaGetLastError();
    done = true;
}

int dalloc(void **p, size_t bytes, const char *what) {
    *p = nullptr;
    if (bytes == 0) bytes = 8;
    init_pool();
    cudaError_t e = cudaMallocAsync(p, bytes, 0);
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *p = nullptr;
        set_error("device allocation of %zu bytes for %s failed: %s", bytes, what,
                  cudaGetErrorString(e));
        return LP_ERR_OOM;
    }
    return LP_OK;
}

void dfree(void *p) {
    if (p) cudaFreeAsync(p, 0);
}

}  // namespace lp

extern "C" const char *lp_last_error(void) { return lp::t_error.c_str(); }

extern "C" const char *lp_version(void) { return "legpcg_b200 0.2 (sm_100a, fp64)"; }

extern "C" int64_t lp_kernel_launches(void) { return lp::g_launches; }

extern "C" int lp_init(int device) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        lp::set_error("no CUDA device available (%s)", cudaGetErrorString(e));
        return LP_ERR_NODEVICE;
    }
    if (device < 0 || device >= count) {
        lp::set_error("device %d out of range (have %d)", device, count);
        return LP_ERR_NODEVICE;
    }
    cudaDeviceProp prop;
    LP_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0) {
        lp::set_error("device %d is sm_%d%d; this library is built for sm_100a only",
                      device, prop.major, prop.minor);
        return LP_ERR_NODEVICE;
    }
    LP_CUDA(cudaSetDevice(device));
    return LP_OK;
}
