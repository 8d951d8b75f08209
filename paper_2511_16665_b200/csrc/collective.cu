// C1: cross-rank BEG-MAB statistics inside the library.
//
// Every rank runs its own engine and its own replica of the reference bandit
// state (beg_mab.hpp:28-69). After a rollout each rank's new beg_record
// records (arm, reward r, a_bar; beg_mab.hpp:111-134) are packed into a
// FIXED-size record block, all-gathered, and applied to a shared replica in
// rank order, so every rank's shared replica is bit-identical; the local
// replica then restarts from it (with one rank this is exactly the local
// beg_record sequence). The all-gather runs either over NCCL (an
// engine-device communicator on its own non-blocking side stream, never the
// decode stream; libnccl is opened with dlopen so the library does not pin a
// NCCL build against the one the host process already loaded) or through a
// host-provided all-gather callback (MPI, gloo, ... — the CPU tests use gloo).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/tlt_b200.h"
#include "capi_types.h"

namespace {

struct Nccl {  // the few entry points C1 uses, resolved at run time
    void* h = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
    static Nccl n = [] {
        Nccl x;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            x.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (x.h) break;
        }
        if (!x.h) return x;
        x.get_unique_id = reinterpret_cast<decltype(x.get_unique_id)>(dlsym(x.h, "ncclGetUniqueId"));
        x.comm_init_rank = reinterpret_cast<decltype(x.comm_init_rank)>(dlsym(x.h, "ncclCommInitRank"));
        x.all_gather = reinterpret_cast<decltype(x.all_gather)>(dlsym(x.h, "ncclAllGather"));
        x.comm_destroy = reinterpret_cast<decltype(x.comm_destroy)>(dlsym(x.h, "ncclCommDestroy"));
        x.error_string = reinterpret_cast<decltype(x.error_string)>(dlsym(x.h, "ncclGetErrorString"));
        return x;
    }();
    if (!n.h || !n.get_unique_id || !n.comm_init_rank || !n.all_gather || !n.comm_destroy)
        throw tlt::CudaError("C1: libnccl.so.2 not loadable");
    return n;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const Nccl& n = nccl();
        throw tlt::CudaError(std::string("C1: ") + what + ": " + (n.error_string ? n.error_string(r) : "nccl error"));
    }
}

int fail(int code, const char* msg) {
    tlt_set_last_error(msg);
    return code;
}
template <typename F>
int guard(F&& f) {
    try {
        f();
        return TLT_OK;
    } catch (const tlt::ConfigErr& e) {
        return fail(TLT_ERR_CONFIG, e.what());
    } catch (const tlt::CudaError& e) {
        return fail(TLT_ERR_CUDA, e.what());
    } catch (const std::exception& e) {
        return fail(TLT_ERR_INTERNAL, e.what());
    }
}

}  // namespace

// One record block per rank: [count][arm, reward, a_bar] x max_records, as doubles
// (arm ids are small integers, exact in a double).
struct tlt_c1 {
    int world = 1, rank = 0, cap = 0;
    size_t block = 0;  // doubles per rank
    tlt_allgather_fn fn = nullptr;
    void* user = nullptr;
    // NCCL transport
    ncclComm_t comm = nullptr;
    cudaStream_t st = nullptr;
    int device = 0;
    double *d_send = nullptr, *d_recv = nullptr, *h_send = nullptr, *h_recv = nullptr;
    ~tlt_c1() {
        if (comm) {
            int prev = 0;
            cudaGetDevice(&prev);
            cudaSetDevice(device);
            if (st) cudaStreamSynchronize(st);
            nccl().comm_destroy(comm);
            if (d_send) cudaFree(d_send);
            if (d_recv) cudaFree(d_recv);
            if (h_send) cudaFreeHost(h_send);
            if (h_recv) cudaFreeHost(h_recv);
            if (st) cudaStreamDestroy(st);
            cudaSetDevice(prev);
        }
    }
};

extern "C" {

TLT_API int tlt_c1_nccl_unique_id(void* id128) {
    if (!id128) return fail(TLT_ERR_CONFIG, "null argument");
    return guard([&] {
        ncclUniqueId id;
        nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
        static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
        std::memcpy(id128, &id, sizeof id);
    });
}

TLT_API int tlt_c1_create_nccl(tlt_engine* e, const void* id128, int world, int rank, int max_records, tlt_c1** out) {
    if (!e || !id128 || !out) return fail(TLT_ERR_CONFIG, "null argument");
    return guard([&] {
        if (world < 1 || rank < 0 || rank >= world) throw tlt::ConfigErr("rank", "out of range for world");
        if (max_records < 1) throw tlt::ConfigErr("max_records", "must be >= 1");
        auto c = std::make_unique<tlt_c1>();
        c->world = world;
        c->rank = rank;
        c->cap = max_records;
        c->block = 1 + 3 * (size_t)max_records;
        c->device = e->e->device();
        int prev = 0;
        CUDA_CHECK(cudaGetDevice(&prev));
        CUDA_CHECK(cudaSetDevice(c->device));
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof id);
        nccl_check(nccl().comm_init_rank(&c->comm, world, id, rank), "ncclCommInitRank");
        CUDA_CHECK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
        CUDA_CHECK(cudaMalloc(&c->d_send, sizeof(double) * c->block));
        CUDA_CHECK(cudaMalloc(&c->d_recv, sizeof(double) * c->block * world));
        CUDA_CHECK(cudaMallocHost(&c->h_send, sizeof(double) * c->block));
        CUDA_CHECK(cudaMallocHost(&c->h_recv, sizeof(double) * c->block * world));
        CUDA_CHECK(cudaSetDevice(prev));
        *out = c.release();
    });
}

TLT_API int tlt_c1_create_callback(int world, int rank, tlt_allgather_fn fn, void* user, int max_records,
                                   tlt_c1** out) {
    if (!fn || !out) return fail(TLT_ERR_CONFIG, "null argument");
    return guard([&] {
        if (world < 1 || rank < 0 || rank >= world) throw tlt::ConfigErr("rank", "out of range for world");
        if (max_records < 1) throw tlt::ConfigErr("max_records", "must be >= 1");
        auto c = std::make_unique<tlt_c1>();
        c->world = world;
        c->rank = rank;
        c->cap = max_records;
        c->block = 1 + 3 * (size_t)max_records;
        c->fn = fn;
        c->user = user;
        c->h_send = nullptr;
        *out = c.release();
    });
}

TLT_API void tlt_c1_destroy(tlt_c1* c) { delete c; }

TLT_API int tlt_c1_merge(tlt_c1* c, tlt_mab* local, tlt_mab* shared, int32_t* n_merged) {
    if (!c || !local || !shared) return fail(TLT_ERR_CONFIG, "null argument");
    return guard([&] {
        auto& lg = local->m->log;
        if ((int)lg.size() > c->cap) throw tlt::ConfigErr("max_records", "more records than the C1 block holds");
        std::vector<double> send_v, recv_v;
        double* send = c->h_send;
        double* recv = c->h_recv;
        if (!c->comm) {
            send_v.assign(c->block, 0.0);
            recv_v.assign(c->block * c->world, 0.0);
            send = send_v.data();
            recv = recv_v.data();
        } else {
            std::memset(send, 0, sizeof(double) * c->block);
        }
        send[0] = (double)lg.size();
        for (size_t i = 0; i < lg.size(); ++i) {
            send[1 + 3 * i] = (double)lg[i].arm;
            send[2 + 3 * i] = lg[i].reward;
            send[3 + 3 * i] = lg[i].a_bar;
        }
        const size_t bytes = sizeof(double) * c->block;
        if (c->comm) {
            int prev = 0;
            CUDA_CHECK(cudaGetDevice(&prev));
            CUDA_CHECK(cudaSetDevice(c->device));
            CUDA_CHECK(cudaMemcpyAsync(c->d_send, send, bytes, cudaMemcpyHostToDevice, c->st));
            nccl_check(nccl().all_gather(c->d_send, c->d_recv, c->block, ncclFloat64, c->comm, c->st), "ncclAllGather");
            CUDA_CHECK(cudaMemcpyAsync(recv, c->d_recv, bytes * c->world, cudaMemcpyDeviceToHost, c->st));
            CUDA_CHECK(cudaStreamSynchronize(c->st));
            CUDA_CHECK(cudaSetDevice(prev));
        } else if (c->fn(c->user, send, recv, bytes) != 0) {
            throw tlt::CudaError("C1: all-gather callback failed");
        }
        int n = 0;
        for (int r = 0; r < c->world; ++r) {  // rank order: every replica applies the same sequence
            const double* blk = recv + (size_t)r * c->block;
            const int cnt = (int)blk[0];
            if (cnt < 0 || cnt > c->cap) throw tlt::CudaError("C1: corrupt record block");
            for (int i = 0; i < cnt; ++i) {
                const int arm = (int)blk[1 + 3 * i];
                if (arm < 0 || arm >= (int)shared->m->arms.size()) throw tlt::ConfigErr("arm", "record for an unknown arm");
                shared->m->push(shared->m->arms[arm], blk[2 + 3 * i], blk[3 + 3 * i], /*logged=*/false);
                ++n;
            }
        }
        lg.clear();
        *local->m = *shared->m;  // the local replica restarts from the merged state
        local->m->log.clear();
        if (n_merged) *n_merged = n;
    });
}

}  // extern "C"
