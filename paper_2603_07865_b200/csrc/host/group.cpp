// Entry-sharded warm start over the GPUs of one process — the library
// form of sharded.py, so a C++ caller shards without torch.
//
// A group owns one context (one cache shard) per GPU. One batch, per shard s on its own stream:
//   H2D prompts/requests -> sw_local_topk (tcgen05 pre-filter + exact fp64 rescoring on the
//   shard: B x k 128-byte records carrying exact sim, id, segment, s_neg, gater block sums and
//   owner = s) -> all-gather of the records and counts -> sw_merge_select (the deterministic
//   (sim desc, id asc) merge of the N sorted lists — the global top-k of IvfIndex::search,
//   index.cpp:289-326, is contained in the union of the per-shard exact top-ks — then the
//   replicated gate / select / Skip Gater / t*) -> sw_align_noise_owned (only the requests whose
//   chosen entry the shard owns; the latent lives there).
// The all-gather is the only data-path exchange. Transports:
//   NCCL  one communicator per device from ncclCommInitAll, ncclAllGather of the records and
//         counts inside one ncclGroupStart/End (NVLink / NVSwitch on a B200 box). libnccl is
//         opened at run time (dlopen), so the library has no link-time NCCL dependency.
//   COPY  each shard pulls every shard's records with cudaMemcpyPeerAsync after an event on the
//         producer's stream (peer access enabled between distinct devices: NVLink reads). Used
//         when shards share a device (several shards per GPU, or tests on one GPU).
// Every shard computes the same choices; shard 0's are returned.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "semwarm_b200.h"

namespace sw {
void set_last_error(const std::string& m);
}

namespace {

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;

    bool load(std::string& why) {
        if (h) return true;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) {
            why = "libnccl.so.2 not found";
            return false;
        }
        comm_init_all = (decltype(comm_init_all))dlsym(h, "ncclCommInitAll");
        all_gather = (decltype(all_gather))dlsym(h, "ncclAllGather");
        group_start = (decltype(group_start))dlsym(h, "ncclGroupStart");
        group_end = (decltype(group_end))dlsym(h, "ncclGroupEnd");
        comm_destroy = (decltype(comm_destroy))dlsym(h, "ncclCommDestroy");
        error_string = (decltype(error_string))dlsym(h, "ncclGetErrorString");
        if (!comm_init_all || !all_gather || !group_start || !group_end || !comm_destroy) {
            why = "libnccl lacks the collective entry points";
            return false;
        }
        return true;
    }
};

NcclApi g_nccl;
std::mutex g_nccl_mu;

int fail(int code, const std::string& m) {
    sw::set_last_error(m);
    return code;
}

#define GCUDA(x)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (x);                                                           \
        if (e_ != cudaSuccess) return fail(SW_ECUDA, std::string(#x) + ": " +           \
                                                         cudaGetErrorString(e_));        \
    } while (0)

}  // namespace

struct sw_group {
    struct Shard {
        sw_ctx* ctx = nullptr;
        int device = 0;
        cudaStream_t st = nullptr;
        cudaEvent_t ev = nullptr;  // records + counts ready
        void* rec = nullptr;       // [B][k] HitRec
        int32_t* n = nullptr;      // [B]
        void* rec_all = nullptr;   // [N][B][k]
        int32_t* n_all = nullptr;  // [N][B]
        float* q = nullptr;        // [B][D]
        sw_request* req = nullptr;
        sw_choice* ch = nullptr;
        ncclComm_t comm = nullptr;
    };
    std::vector<Shard> shards;
    int transport = SW_GROUP_TRANSPORT_COPY;
    int D = 0, Bmax = 0;
    size_t rec_bytes = 0;  // one shard's records at Bmax x kMax
    float* h_q = nullptr;  // pinned staging
    sw_request* h_req = nullptr;
    sw_choice* h_ch = nullptr;
    std::mutex mu;

    int release() {
        for (Shard& s : shards) {
            if (s.device >= 0) cudaSetDevice(s.device);
            if (s.st) cudaStreamSynchronize(s.st);
            if (s.comm && g_nccl.comm_destroy) g_nccl.comm_destroy(s.comm);
            for (void* p : {s.rec, (void*)s.n, s.rec_all, (void*)s.n_all, (void*)s.q, (void*)s.req,
                            (void*)s.ch})
                if (p) cudaFree(p);
            if (s.ev) cudaEventDestroy(s.ev);
            if (s.st) cudaStreamDestroy(s.st);
            if (s.ctx) sw_ctx_destroy(s.ctx);
        }
        shards.clear();
        if (h_q) cudaFreeHost(h_q);
        if (h_req) cudaFreeHost(h_req);
        if (h_ch) cudaFreeHost(h_ch);
        h_q = nullptr;
        h_req = nullptr;
        h_ch = nullptr;
        return SW_OK;
    }
};

namespace {
constexpr int kMaxK = 32;
constexpr size_t kHitRecBytes = 128;
}  // namespace

extern "C" {

int sw_group_create(const sw_config* cfg, int32_t n_shards, const int32_t* devices,
                    int32_t transport, sw_group** out) {
    if (!cfg || !out || n_shards < 1 || n_shards > 64)
        return fail(SW_EINVAL, "sw_group_create: need a config, 1..64 shards and an out pointer");
    if (transport < SW_GROUP_TRANSPORT_AUTO || transport > SW_GROUP_TRANSPORT_COPY)
        return fail(SW_EINVAL, "sw_group_create: unknown transport");
    std::vector<int> devs((size_t)n_shards);
    for (int s = 0; s < n_shards; ++s) devs[s] = devices ? devices[s] : s;
    const bool distinct = std::set<int>(devs.begin(), devs.end()).size() == devs.size();
    if (transport == SW_GROUP_TRANSPORT_AUTO)
        transport = (distinct && n_shards > 1) ? SW_GROUP_TRANSPORT_NCCL : SW_GROUP_TRANSPORT_COPY;
    if (transport == SW_GROUP_TRANSPORT_NCCL && !distinct)
        return fail(SW_EINVAL, "NCCL transport needs one shard per device");
    auto* g = new sw_group();
    g->transport = transport;
    g->D = cfg->dim;
    g->Bmax = cfg->max_batch;
    g->rec_bytes = (size_t)g->Bmax * kMaxK * kHitRecBytes;
    g->shards.resize((size_t)n_shards);
    for (auto& s : g->shards) s.device = -1;
    auto bail = [&](int rc) {
        g->release();
        delete g;
        return rc;
    };
    for (int s = 0; s < n_shards; ++s) {
        sw_group::Shard& sh = g->shards[s];
        sh.device = devs[s];
        int rc = sw_ctx_create(cfg, sh.device, &sh.ctx);
        if (rc != SW_OK) return bail(rc);
        if (cudaSetDevice(sh.device) != cudaSuccess ||
            cudaStreamCreateWithFlags(&sh.st, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&sh.ev, cudaEventDisableTiming) != cudaSuccess ||
            cudaMalloc(&sh.rec, g->rec_bytes) != cudaSuccess ||
            cudaMalloc((void**)&sh.n, sizeof(int32_t) * g->Bmax) != cudaSuccess ||
            cudaMalloc(&sh.rec_all, g->rec_bytes * n_shards) != cudaSuccess ||
            cudaMalloc((void**)&sh.n_all, sizeof(int32_t) * g->Bmax * n_shards) != cudaSuccess ||
            cudaMalloc((void**)&sh.q, sizeof(float) * (size_t)g->Bmax * g->D) != cudaSuccess ||
            cudaMalloc((void**)&sh.req, sizeof(sw_request) * g->Bmax) != cudaSuccess ||
            cudaMalloc((void**)&sh.ch, sizeof(sw_choice) * g->Bmax) != cudaSuccess)
            return bail(fail(SW_ENOMEM, "sw_group_create: device allocation failed"));
    }
    // NVLink peer access between distinct devices (the COPY transport's reads; harmless for NCCL)
    for (int a = 0; a < n_shards; ++a)
        for (int b = 0; b < n_shards; ++b) {
            const int da = devs[a], db = devs[b];
            if (da == db) continue;
            int ok = 0;
            if (cudaDeviceCanAccessPeer(&ok, da, db) == cudaSuccess && ok) {
                cudaSetDevice(da);
                const cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            }
        }
    if (transport == SW_GROUP_TRANSPORT_NCCL) {
        std::lock_guard<std::mutex> lk(g_nccl_mu);
        std::string why;
        if (!g_nccl.load(why)) return bail(fail(SW_ERUNTIME, "NCCL transport: " + why));
        std::vector<ncclComm_t> comms((size_t)n_shards);
        const ncclResult_t r = g_nccl.comm_init_all(comms.data(), n_shards, devs.data());
        if (r != ncclSuccess)
            return bail(fail(SW_ERUNTIME, std::string("ncclCommInitAll: ") +
                                              (g_nccl.error_string ? g_nccl.error_string(r) : "")));
        for (int s = 0; s < n_shards; ++s) g->shards[s].comm = comms[s];
    }
    if (cudaMallocHost(&g->h_q, sizeof(float) * (size_t)g->Bmax * g->D) != cudaSuccess ||
        cudaMallocHost(&g->h_req, sizeof(sw_request) * g->Bmax) != cudaSuccess ||
        cudaMallocHost(&g->h_ch, sizeof(sw_choice) * g->Bmax) != cudaSuccess)
        return bail(fail(SW_ENOMEM, "sw_group_create: pinned allocation failed"));
    *out = g;
    return SW_OK;
}

int sw_group_destroy(sw_group* g) {
    if (!g) return SW_OK;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        g->release();
    }
    delete g;
    return SW_OK;
}

int sw_group_info(sw_group* g, int32_t* n_shards, int32_t* transport) {
    if (!g) return fail(SW_EINVAL, "null group");
    if (n_shards) *n_shards = (int32_t)g->shards.size();
    if (transport) *transport = g->transport;
    return SW_OK;
}

int sw_group_shard(sw_group* g, int32_t shard, sw_ctx** ctx) {
    if (!g || !ctx || shard < 0 || shard >= (int)g->shards.size())
        return fail(SW_EINVAL, "sw_group_shard: shard out of range");
    *ctx = g->shards[shard].ctx;
    return SW_OK;
}

int32_t sw_group_owner(sw_group* g, uint64_t entry_id) {
    if (!g || g->shards.empty()) return -1;
    return (int32_t)(entry_id % g->shards.size());
}

int sw_group_insert(sw_group* g, uint64_t id, int32_t n_rows, const float* rows,
                    const sw_segment* segs, const float* latent, int32_t t_src) {
    if (!g) return fail(SW_EINVAL, "null group");
    return sw_arena_insert(g->shards[id % g->shards.size()].ctx, id, n_rows, rows, segs, latent,
                           t_src);
}

int sw_group_remove(sw_group* g, uint64_t id) {
    if (!g) return fail(SW_EINVAL, "null group");
    return sw_arena_remove(g->shards[id % g->shards.size()].ctx, id);
}

int sw_group_set_negative(sw_group* g, const float* negative) {
    if (!g) return fail(SW_EINVAL, "null group");
    for (auto& s : g->shards) {
        const int rc = sw_set_negative(s.ctx, negative);
        if (rc != SW_OK) return rc;
    }
    return SW_OK;
}

int sw_group_set_gater(sw_group* g, const float* theta, const float* psi, int32_t feature_dim,
                       double beta) {
    if (!g) return fail(SW_EINVAL, "null group");
    for (auto& s : g->shards) {
        const int rc = sw_set_gater(s.ctx, theta, psi, feature_dim, beta);
        if (rc != SW_OK) return rc;
    }
    return SW_OK;
}

int sw_group_warmstart_host(sw_group* g, const float* h_queries, const sw_request* h_reqs,
                            int32_t B, uint64_t seed, const sw_selector_config* sel,
                            const sw_policy* pol, uint64_t philox_seed, sw_choice* h_choices,
                            float* const* d_out, int32_t t_out_max) {
    if (!g || !sel || !pol || (B > 0 && (!h_queries || !h_reqs || !h_choices)))
        return fail(SW_EINVAL, "sw_group_warmstart_host: null argument");
    if (B < 0 || B > g->Bmax) return fail(SW_EINVAL, "batch exceeds the group's max_batch");
    const int k = sel->top_k;
    if (k < 1 || k > kMaxK) return fail(SW_EINVAL, "top_k must be in [1, 32]");
    if (B == 0) return SW_OK;
    std::lock_guard<std::mutex> lk(g->mu);
    const int N = (int)g->shards.size();
    const size_t qb = sizeof(float) * (size_t)B * g->D, rb = sizeof(sw_request) * B;
    const size_t recb = (size_t)B * k * kHitRecBytes;
    std::memcpy(g->h_q, h_queries, qb);
    std::memcpy(g->h_req, h_reqs, rb);
    // 1. local exact top-k on every shard
    for (int s = 0; s < N; ++s) {
        sw_group::Shard& sh = g->shards[s];
        GCUDA(cudaSetDevice(sh.device));
        GCUDA(cudaMemcpyAsync(sh.q, g->h_q, qb, cudaMemcpyHostToDevice, sh.st));
        GCUDA(cudaMemcpyAsync(sh.req, g->h_req, rb, cudaMemcpyHostToDevice, sh.st));
        const int rc = sw_local_topk(sh.ctx, sh.q, B, k, s, sh.rec, sh.n, (void*)sh.st);
        if (rc != SW_OK) return rc;
        GCUDA(cudaEventRecord(sh.ev, sh.st));
    }
    // 2. all-gather of records and counts (rank-major: [N][B][k], [N][B])
    if (g->transport == SW_GROUP_TRANSPORT_NCCL) {
        if (g_nccl.group_start() != ncclSuccess) return fail(SW_ERUNTIME, "ncclGroupStart");
        for (int s = 0; s < N; ++s) {
            sw_group::Shard& sh = g->shards[s];
            if (g_nccl.all_gather(sh.rec, sh.rec_all, recb, ncclUint8, sh.comm, sh.st) !=
                    ncclSuccess ||
                g_nccl.all_gather(sh.n, sh.n_all, (size_t)B, ncclInt32, sh.comm, sh.st) !=
                    ncclSuccess) {
                g_nccl.group_end();
                return fail(SW_ERUNTIME, "ncclAllGather failed");
            }
        }
        if (g_nccl.group_end() != ncclSuccess) return fail(SW_ERUNTIME, "ncclGroupEnd");
    } else {
        for (int s = 0; s < N; ++s) {
            sw_group::Shard& sh = g->shards[s];
            GCUDA(cudaSetDevice(sh.device));
            for (int r = 0; r < N; ++r) {
                const sw_group::Shard& src = g->shards[r];
                GCUDA(cudaStreamWaitEvent(sh.st, src.ev, 0));
                GCUDA(cudaMemcpyPeerAsync((char*)sh.rec_all + recb * r, sh.device, src.rec,
                                          src.device, recb, sh.st));
                GCUDA(cudaMemcpyPeerAsync(sh.n_all + (size_t)B * r, sh.device, src.n, src.device,
                                          sizeof(int32_t) * B, sh.st));
            }
        }
    }
    // 3. replicated merge + select on every shard, 4. owner-computes align + noise
    for (int s = 0; s < N; ++s) {
        sw_group::Shard& sh = g->shards[s];
        GCUDA(cudaSetDevice(sh.device));
        int rc = sw_merge_select(sh.ctx, sh.rec_all, sh.n_all, N, sh.q, sh.req, B, k, seed, sel,
                                 pol, sh.ch, (void*)sh.st);
        if (rc != SW_OK) return rc;
        if (d_out && d_out[s]) {
            rc = sw_align_noise_owned(sh.ctx, sh.ch, sh.req, B, s, nullptr, philox_seed, d_out[s],
                                      t_out_max, (void*)sh.st);
            if (rc != SW_OK) return rc;
        }
    }
    sw_group::Shard& s0 = g->shards[0];
    GCUDA(cudaSetDevice(s0.device));
    GCUDA(cudaMemcpyAsync(g->h_ch, s0.ch, sizeof(sw_choice) * B, cudaMemcpyDeviceToHost, s0.st));
    for (auto& sh : g->shards) {
        GCUDA(cudaSetDevice(sh.device));
        GCUDA(cudaStreamSynchronize(sh.st));
    }
    std::memcpy(h_choices, g->h_ch, sizeof(sw_choice) * B);
    return SW_OK;
}

int sw_group_shard_choices(sw_group* g, int32_t shard, int32_t B, sw_choice* h_choices) {
    if (!g || !h_choices || shard < 0 || shard >= (int)g->shards.size() || B < 0 || B > g->Bmax)
        return fail(SW_EINVAL, "sw_group_shard_choices: bad argument");
    std::lock_guard<std::mutex> lk(g->mu);
    sw_group::Shard& sh = g->shards[shard];
    GCUDA(cudaSetDevice(sh.device));
    GCUDA(cudaMemcpy(h_choices, sh.ch, sizeof(sw_choice) * B, cudaMemcpyDeviceToHost));
    return SW_OK;
}

}  // extern "C"
