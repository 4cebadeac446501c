// Multi-GPU collectives of the C ABI (lp_comm_init(ncclComm_t, rank,
// size, slab_axis)): the three exchanges the distributed PCG needs, on the
// caller's NCCL communicator and stream.
//
//   lp_comm_allreduce_dd  the PCG scalars (pcg.py:150-159): every rank's
//                         double-double partial is all-gathered and summed in
//                         RANK ORDER by one thread, so every rank holds the same
//                         bits and a G-rank run rounds like the emulation;
//   lp_comm_dot           a slab's deterministic dd dot followed by that;
//   lp_comm_alltoall      the transposes of the slab-sharded matvec (E1-E3 of
//                         sharded.py): grouped ncclSend/ncclRecv of contiguous
//                         chunks with per-peer counts.
//
// NCCL is resolved at run time (dlopen of the libnccl.so.2 the host process
// already uses -- torch's, or the system's), so the library has no link-time
// NCCL dependency and single-GPU users never load it.
#include <dlfcn.h>

#include <vector>

#include "lp_common.cuh"
#include "vector_ops.cuh"

namespace lp {

namespace {

typedef int (*nccl_allgather_t)(const void *, void *, size_t, int, void *, cudaStream_t);
typedef int (*nccl_sendrecv_t)(void *, size_t, int, int, void *, cudaStream_t);
typedef int (*nccl_group_t)();
typedef const char *(*nccl_errstr_t)(int);

struct Nccl {
    void *so = nullptr;
    nccl_allgather_t all_gather = nullptr;
    nccl_sendrecv_t send = nullptr, recv = nullptr;
    nccl_group_t group_start = nullptr, group_end = nullptr;
    nccl_errstr_t errstr = nullptr;
};

constexpr int kNcclDouble = 8;   // ncclFloat64 (nccl.h)

int load_nccl(Nccl &n) {
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *nm : names) {
        // RTLD_NOLOAD first: the copy the process already has (torch's bundled one)
        n.so = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);
        if (!n.so) n.so = dlopen(nm, RTLD_NOW);
        if (n.so) break;
    }
    if (!n.so) {
        set_error("cannot load libnccl.so.2: %s", dlerror());
        return LP_ERR_ARG;
    }
    n.all_gather = (nccl_allgather_t)dlsym(n.so, "ncclAllGather");
    n.send = (nccl_sendrecv_t)dlsym(n.so, "ncclSend");
    n.recv = (nccl_sendrecv_t)dlsym(n.so, "ncclRecv");
    n.group_start = (nccl_group_t)dlsym(n.so, "ncclGroupStart");
    n.group_end = (nccl_group_t)dlsym(n.so, "ncclGroupEnd");
    n.errstr = (nccl_errstr_t)dlsym(n.so, "ncclGetErrorString");
    if (!n.all_gather || !n.send || !n.recv || !n.group_start || !n.group_end) {
        set_error("libnccl.so.2 lacks a required symbol");
        return LP_ERR_ARG;
    }
    return LP_OK;
}

// rank-ordered double-double sum of the gathered partials (one thread: the
// order is the point)
__global__ void ordered_sum_kernel(const double *__restrict__ parts, int size, double *__restrict__ out) {
    dd acc{0.0, 0.0};
    for (int v = 0; v < size; ++v) acc = dd_add(acc, dd{parts[2 * v], parts[2 * v + 1]});
    out[0] = acc.hi;
    out[1] = acc.lo;
}

}  // namespace

}  // namespace lp

struct lp_comm {
    void *nccl_comm = nullptr;
    int rank = 0, size = 1, slab_axis = 2;
    lp::Nccl nccl;
    double *gathered = nullptr;   // [size][2]
    double *mine = nullptr;       // [2] send buffer (all-gather must not alias its output slot)
    double *partial = nullptr;    // dd block partials of lp_comm_dot
};

using namespace lp;

#define LP_NCCL(c, call)                                                                          \
    do {                                                                                          \
        const int r_ = (call);                                                                    \
        if (r_ != 0) {                                                                            \
            set_error("NCCL: %s", (c)->nccl.errstr ? (c)->nccl.errstr(r_) : "error");              \
            return LP_ERR_CUDA;                                                                   \
        }                                                                                         \
    } while (0)

extern "C" int lp_comm_init(void *nccl_comm, int rank, int size, int slab_axis, lp_comm **out) {
    LP_ARG(nccl_comm != nullptr, "null NCCL communicator");
    LP_ARG(size >= 1 && rank >= 0 && rank < size, "rank %d outside [0, %d)", rank, size);
    LP_ARG(slab_axis >= 0 && slab_axis <= 2, "slab_axis must be 0, 1 or 2");
    lp_comm *c = new lp_comm;
    c->nccl_comm = nccl_comm;
    c->rank = rank;
    c->size = size;
    c->slab_axis = slab_axis;
    int rc = load_nccl(c->nccl);
    if (!rc) rc = dalloc(&c->gathered, (size_t)2 * size, "gathered scalars");
    if (!rc) rc = dalloc(&c->mine, 2, "scalar send buffer");
    if (!rc) rc = dalloc(&c->partial, (size_t)2 * RED_BLOCKS, "dot partials");
    if (rc) {
        dfree(c->gathered);
        dfree(c->mine);
        dfree(c->partial);
        delete c;
        return rc;
    }
    *out = c;
    return LP_OK;
}

extern "C" int lp_comm_destroy(lp_comm *c) {
    if (!c) return LP_OK;
    cudaDeviceSynchronize();
    dfree(c->gathered);
    dfree(c->mine);
    dfree(c->partial);
    delete c;   // the NCCL communicator stays the caller's
    return LP_OK;
}

extern "C" int lp_comm_allreduce_dd(lp_comm *c, double *dd_inout, void *stream) {
    cudaStream_t st = as_stream(stream);
    LP_CUDA(cudaMemcpyAsync(c->mine, dd_inout, 2 * sizeof(double), cudaMemcpyDeviceToDevice, st));
    LP_NCCL(c, c->nccl.all_gather(c->mine, c->gathered, 2, kNcclDouble, c->nccl_comm, st));
    ordered_sum_kernel<<<1, 1, 0, st>>>(c->gathered, c->size, dd_inout);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

extern "C" int lp_comm_dot(lp_comm *c, int64_t n, const double *a, const double *b, double *out2, void *stream) {
    cudaStream_t st = as_stream(stream);
    const int rc = dot_dd(n, a, b, c->partial, out2, st);
    return rc ? rc : lp_comm_allreduce_dd(c, out2, stream);
}

extern "C" int lp_comm_alltoall(lp_comm *c, const double *send, const int64_t *send_counts, double *recv,
                                const int64_t *recv_counts, void *stream) {
    cudaStream_t st = as_stream(stream);
    int64_t so = 0, ro = 0;
    LP_ARG(send_counts[c->rank] == recv_counts[c->rank], "own chunk sizes differ");
    for (int v = 0; v < c->size; ++v) LP_ARG(send_counts[v] >= 0 && recv_counts[v] >= 0, "negative chunk size");
    LP_NCCL(c, c->nccl.group_start());
    for (int v = 0; v < c->size; ++v) {
        if (v == c->rank) {
            // own chunk: a device copy on the same stream
            LP_CUDA(cudaMemcpyAsync(recv + ro, send + so, (size_t)send_counts[v] * sizeof(double),
                                    cudaMemcpyDeviceToDevice, st));
        } else {
            if (send_counts[v])
                LP_NCCL(c, c->nccl.send((void *)(send + so), (size_t)send_counts[v], kNcclDouble, v, c->nccl_comm, st));
            if (recv_counts[v])
                LP_NCCL(c, c->nccl.recv(recv + ro, (size_t)recv_counts[v], kNcclDouble, v, c->nccl_comm, st));
        }
        so += send_counts[v];
        ro += recv_counts[v];
    }
    LP_NCCL(c, c->nccl.group_end());
    return LP_OK;
}
