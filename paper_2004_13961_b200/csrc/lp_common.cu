// Error state, device checks and allocation helpers.
#include <stdarg.h>

#include <atomic>
#include <map>
#include <mutex>
#include <tuple>

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
    static std::atomic<bool> done[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        cudaGetLastError();
        return;
    }
    if (done[dev].load(std::memory_order_relaxed)) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t threshold = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
    }
    cudaGetLastError();
    done[dev].store(true, std::memory_order_relaxed);
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

void dfree(void *p, cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
}

int salloc(void **p, size_t bytes, const char *what, cudaStream_t st) {
    *p = nullptr;
    if (bytes == 0) bytes = 8;
    init_pool();
    const cudaError_t e = cudaMallocAsync(p, bytes, st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *p = nullptr;
        set_error("device allocation of %zu bytes for %s failed: %s", bytes, what,
                  cudaGetErrorString(e));
        return LP_ERR_OOM;
    }
    return LP_OK;
}

void sfree(void *p, cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
}

int num_sms() {
    static std::atomic<int> cache[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        cudaGetLastError();
        return 148;
    }
    int v = cache[dev].load(std::memory_order_relaxed);
    if (v <= 0) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
            cudaGetLastError();
            v = 148;
        }
        cache[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

namespace {
std::mutex g_occ_mu;
std::map<std::tuple<int, const void *, int, size_t, int>, int> g_occ;
std::map<std::pair<int, const void *>, size_t> g_smem_limit;   // dynamic-smem limit set per kernel

// Raise the kernel's dynamic shared-memory limit to at least `smem` (never
// lowers it: launches with a smaller request stay valid).  Caller holds g_occ_mu.
bool ensure_smem_limit(int dev, const void *fn, size_t smem) {
    size_t &cur = g_smem_limit[std::make_pair(dev, fn)];
    if (cur >= smem && cur > 0) return true;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    cur = smem;
    return true;
}
}  // namespace

static int occupancy_query(const void *fn, int threads, size_t smem, int csize) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    const auto key = std::make_tuple(dev, fn, threads, smem, csize);
    std::lock_guard<std::mutex> lk(g_occ_mu);
    {
        auto it = g_occ.find(key);
        if (it != g_occ.end()) return ensure_smem_limit(dev, fn, smem) ? it->second : 0;
    }
    int blocks = 0;
    if (ensure_smem_limit(dev, fn, smem)) {
        if (csize <= 1) {
            int occ = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) == cudaSuccess)
                blocks = occ * num_sms();
        } else if (cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                   cudaSuccess) {
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = csize;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.gridDim = dim3(csize, 1, 1);
            cfg.blockDim = dim3(threads, 1, 1);
            cfg.dynamicSmemBytes = smem;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int ncl = 0;
            if (cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg) == cudaSuccess) blocks = ncl * csize;
        }
    }
    cudaGetLastError();
    g_occ[key] = blocks;
    return blocks;
}

int resident_blocks(const void *fn, int threads, size_t smem) {
    return occupancy_query(fn, threads, smem, 1);
}

int resident_cluster_blocks(const void *fn, int threads, size_t smem, int csize) {
    return occupancy_query(fn, threads, smem, csize);
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
