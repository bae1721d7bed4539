// Internal definitions shared by the semwarm_b200 translation units.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <map>
#include <mutex>
#include <set>
#include <shared_mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "semwarm_b200.h"

namespace sw {

namespace dev {
struct SelParams;
}

// --------------------------------------------------------------------------- errors
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
void set_last_error(const std::string& msg);

#define SW_CUDA(call)                                                                     \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            throw ::sw::Error(SW_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)
#define SW_REQUIRE(cond, msg)                                      \
    do {                                                           \
        if (!(cond)) throw ::sw::Error(SW_EINVAL, std::string(msg)); \
    } while (0)

// --------------------------------------------------------------------------- constants
constexpr int kNumArms = 14;          // gater.hpp:13
constexpr int kFeatureDim = 11;       // gater.hpp:28
constexpr int kMaxTopK = 32;          // tcgen05 epilogue keeps a 32-deep running list
constexpr int kCandCap = 16384;       // emitted candidates per query (split over the CTAs)
constexpr int kMaxSlices = 2 * 148;   // (scoring CTA, epilogue group) emission slices per query
constexpr int kMaxRowsPad = 32;       // delta >= 1/16 -> at most 31 rows (index.cpp:20-21)
constexpr int kMaxCentroids = 256;    // IVF lists (index.centroids; reference default 64)
constexpr uint8_t kNotProbed = 255;   // probe-rank sentinel
// Certified-overflow fallback: queries whose candidate slices overflowed are re-searched by an
// exact fp64 scan of the whole arena, kOvfQG queries per pass, one k_overflow CTA of kOvfWarps
// warps per SM. State header: [0] flagged count, [1] chunks merged, [2..3] lifetime total (u64).
constexpr int kOvfQG = 4;
constexpr int kOvfWarps = 8;
constexpr int kOvfRing = 4;
constexpr int kOvfHdr = 4;
// Certified error of a tcgen05 score: |q.e - q~.e~| <= |q| |e - e~| + |q - q~| |e~|
// (Cauchy-Schwarz on q.e - q~.e~ = q.(e - e~) + (q - q~).e~, ~ = bf16) plus the fp32 tensor-core
// accumulation slack kAccSlack * |q~| |e~| (K <= 512 additions at <= 2^-23 relative each, x2).
constexpr float kAccSlack = 0x1.0p-12f;

// Per-shard top-k record (SW_HIT_RECORD_BYTES = 128): everything the replicated select /
// gater stage needs, so the all-gather carries no embeddings.
struct __align__(16) HitRec {
    double sim;        // exact clamped fp64 cosine of the winning segment (core.cpp:33-38)
    uint64_t entry_id;
    int32_t level;
    int32_t slot;      // arena slot on the owner shard
    double start_s;
    double length_s;
    double s_neg;      // clamp01(cos(segment row, negative)) (selector.cpp:41-42)
    double phi[8];     // block sums of the gater features (gater.cpp:18-26)
    int32_t row;       // pyramid row index within the entry
    int32_t owner;     // shard rank
};
static_assert(sizeof(HitRec) == SW_HIT_RECORD_BYTES, "hit record must stay 128 bytes");

// --------------------------------------------------------------------------- order helpers
// float/double -> unsigned key preserving order (for atomicMax and packed comparisons)
__host__ __device__ __forceinline__ uint32_t f2ord(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ __forceinline__ float ord2f(uint32_t u) {
    u = (u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u;
    float f;
    memcpy(&f, &u, 4);
    return f;
}
__host__ __device__ __forceinline__ uint64_t d2ord(double d) {
    uint64_t u;
    memcpy(&u, &d, 8);
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

// --------------------------------------------------------------------------- context
struct Ctx;
struct Ctx {
    sw_config cfg{};
    int device = 0;
    int D = 0, Dp = 0, Df = 0;   // dim, bf16 row stride (mult of 64), fp32 row stride (mult of 4)
    int R = 0, Rp = 0, logRp = 0;
    int64_t S = 0;               // entry slots
    int64_t Lslots = 0;          // latent slots
    int C = 0, Tmax = 0, F = 0;
    int Bmax = 0, BmaxPad = 0;

    // device arena (Cache Manager data plane)
    float* rows = nullptr;            // [S*Rp][Df] fp32 master rows
    __nv_bfloat16* rows_bf = nullptr; // [S*Rp][Dp] bf16 shadow (pad rows = copy of row 0)
    double* sneg = nullptr;           // [S*Rp]
    sw_segment* segs = nullptr;       // [S*Rp]
    uint64_t* ids = nullptr;          // [S]
    int32_t* nrows = nullptr;         // [S]
    uint8_t* valid = nullptr;         // [S]
    uint32_t* valid_bits = nullptr;   // [S/32 + pad] one bit per slot (read by the tcgen05 epilogue)
    int32_t* tsrc = nullptr;          // [S]
    float* latent = nullptr;          // [Lslots][C][Tmax][F]
    uint32_t* norms = nullptr;        // ordered floats: max |e|, max |e - bf16(e)|, max |bf16(e)|
    float* neg = nullptr;             // [Df]
    float* theta = nullptr;           // [14*11]
    float* psi = nullptr;
    double* abar = nullptr;
    float2* s01 = nullptr;  // (sqrt(abar), sqrt(1 - abar)) as floats, per schedule index
    std::vector<float2> h_s01;
    int n_abar = 0;
    double beta = 1.0;
    int fd = kFeatureDim;
    bool have_neg = false;

    // batch scratch
    __nv_bfloat16* q_bf = nullptr;  // [BmaxPad][Dp]
    float* q_norm = nullptr;        // [Bmax]
    float* q_eps = nullptr;         // [Bmax] certified |bf16 score - fp64 score| bound per query
    uint32_t* thr = nullptr;        // [Bmax] shared running k-th best (ordered)
    uint32_t* top1 = nullptr;       // [Bmax][kMaxSlices] each slice's running best (ordered)
    int32_t* cand_n = nullptr;      // [3][Bmax]: unused | compacted count | overflow flag
    int32_t* slice_cnt = nullptr;   // [Bmax][kMaxSlices] emissions per (query, CTA, group)
    float* cta_topk = nullptr;      // [Bmax][kMaxSlices][32] each slice's final top-k (approx)
    int32_t* dbg = nullptr;         // [Bmax][8] per-query finish stats (sw_debug_query_stats)
    int last_chunks = 1;
    bool last_ivf = false;         // last search probed IVF lists (nprobe < C)
    bool last_score_pair = false;  // last scoring launch ran as tcgen05 CTA pairs
    bool last_score_ts = false;    // ... with the queries resident in TMEM (TS MMA)
    bool last_score_pack = false;  // ... on packed pyramid tiles (no pad rows)
    int32_t* cand_slot = nullptr;   // [Bmax][kCandCap]
    float* cand_score = nullptr;    // [Bmax][kCandCap]
    double* cand_exact = nullptr;   // [Bmax][kCandCap]
    int32_t* cand_row = nullptr;    // [Bmax][kCandCap]
    int32_t* cand_list = nullptr;   // [Bmax][kCandCap] compacted certified candidates
    // certified-overflow fallback (finish.cu k_overflow): flagged queries, chunk counters and
    // the ring of per-warp exact top-k lists (see kOvf* below)
    int32_t* ovf_state = nullptr;   // [kOvfHdr + Bmax + 2 * ovf_chunks]
    void* ovf_ring = nullptr;       // [kOvfRing][kOvfQG][num_sms * kOvfWarps][kMaxTopK] records
    HitRec* hits = nullptr;         // [Bmax][kMaxTopK]
    int32_t* nhits = nullptr;       // [Bmax]
    float* d_q_stage = nullptr;     // [Bmax][D] (host e2e staging)
    sw_request* d_req_stage = nullptr;
    sw_choice* d_choice_stage = nullptr;
    void* h_pinned = nullptr;       // pinned host staging
    size_t h_pinned_bytes = 0;
    // device temporaries of arena mutations (MScratch): a grow-once stack, stream-ordered on
    // mstream, so a single-entry admit / evict allocates and frees nothing (cudaFree
    // synchronises the whole device)
    char* mscratch = nullptr;
    size_t mscratch_cap = 0, mscratch_top = 0;

    // TMA descriptors (encoded once at creation; cover the full capacity)
    CUtensorMap tm_rows{};
    CUtensorMap tm_rows_half{};  // 128-row boxes for the CTA-pair scoring kernel
    CUtensorMap tm_rows_q64{};   // 64-row boxes for the CTA-pair TMEM-A (TS) kernel
    // packed pyramid tiles (R in {3, 7}: 32 entries x R rows, the pad row skipped): 3-D boxes
    // (64, R, 32) and (64, R, 16) over the arena viewed as [S][Rp][Dp]
    CUtensorMap tm_pack{};
    CUtensorMap tm_pack_half{};
    bool pack_ok = false;
    CUtensorMap tm_q{};
    bool tc_ok = false;
    int smem_optin = 0;
    int num_sms = 148;

    // IVF coarse quantiser (IvfIndex, index.hpp:47-101). ivf == false: exhaustive (one list).
    bool ivf = false;
    int ivf_target = 1;               // target_centroids_
    int ivf_nprobe = 8;               // nprobe_
    int nprobe_override = 0;          // > 0: this call's search(q, k, nprobe) (index.hpp:67)
    int ivf_C = 0;                    // centroids_.size()
    uint64_t ivf_seed = 0;            // seed_
    uint64_t ivf_interval = 1024;     // rebuild_interval_
    uint64_t ivf_mutations = 0;       // mutations_since_rebuild_
    uint64_t ivf_rebuilds = 0;        // rebuild_count_
    float* cent = nullptr;            // [kMaxCentroids][Df] centroids (device)
    std::vector<float> h_cent;        // [ivf_C][D] host mirror
    int16_t* row_list = nullptr;      // [S*Rp] list (nearest centroid) of every stored row
    uint8_t* prank = nullptr;         // [Bmax][kMaxCentroids] probe rank per list, 255 = not probed
    uint64_t* pmask = nullptr;        // [Bmax][4] probed-list bitmask (read by the tcgen05 epilogue)
    std::vector<int32_t> ivf_rows;    // [S] rows of each slot the index has seen (insert order)
    // alignment of the chosen latent: 0 crop / tile (default), 1 the reference's phase vocoder
    int align_mode = 0;
    int voc_win = 128, voc_hop = 32;  // StftConfig (pipeline.hpp:36)
    void* d_voc = nullptr;            // per-request vocoder plans + aligned flags
    int voc_cap = 0;
    // grouped IVF search (one row per entry): a list-sorted, tile-aligned bf16 copy of the arena
    // (rebuilt lazily after index changes) and per-batch query groups per probed list
    bool grp_dirty = true;
    int64_t grp_rows = 0, grp_cap_rows = 0;
    int grp_C = 0, grp_tpc = 8, grp_ch = 1, grp_max_chunks = 0;
    std::vector<int32_t> grp_tile0, grp_ntiles;
    int32_t* d_sorted_slot = nullptr;        // [grp_cap_rows] arena slot of each sorted row
    __nv_bfloat16* d_rows_sorted = nullptr;  // [grp_cap_rows][Dp]
    uint32_t* d_sorted_vbits = nullptr;      // [grp_cap_rows / 32 + 16]
    int32_t* d_list_tile0 = nullptr;         // [kMaxCentroids]
    int32_t* d_list_ntiles = nullptr;        // [kMaxCentroids]
    int32_t* d_qcnt = nullptr;               // [kMaxCentroids] queries probing each list
    int32_t* d_qlist = nullptr;              // [kMaxCentroids][Bmax]
    int32_t* d_qbase = nullptr;              // [kMaxCentroids + 1] first gathered block per list
    __nv_bfloat16* d_qg = nullptr;           // [qg_cap][Dp] gathered query rows
    int32_t* d_qmap = nullptr;               // [qg_cap] query id of each gathered row
    int64_t qg_cap = 0;
    int4* d_items = nullptr;                 // [items_cap]
    int64_t items_cap = 0;
    CUtensorMap tm_sorted{};
    CUtensorMap tm_sorted_half{};  // 128-row boxes: each CTA of a pair stages half a tile
    bool grp_pair = false;         // grouped IVF items cover two query blocks (CTA pairs)
    CUtensorMap tm_qg{};

    // host bookkeeping (mirrors the reference's entry_vector_counts_, index.hpp:92)
    std::unordered_map<uint64_t, int64_t> slot_of;
    std::vector<int32_t> h_nrows;
    std::set<int64_t> free_slots;
    int64_t high_water = 0;
    mutable std::shared_mutex mu;

    cudaStream_t mstream = nullptr;   // mutation stream
    // Hot-path calls share the context's batch scratch (q_bf, thresholds, candidate buffers,
    // staging): their enqueue is serialised on the host and their GPU work chained through
    // scratch_ev, so concurrent readers on different streams never overlap on it.
    std::mutex scratch_mu;
    cudaEvent_t scratch_ev = nullptr;
    // Cross-batch pipelining (sw_warmstart_async): prep + score of batch i+1 run on the caller's
    // stream while finish + align of batch i run on async_st. The buffers the finish reads and
    // the next scoring writes alternate between two parities; the rest of the scratch is only
    // touched by one of the two streams.
    cudaStream_t async_st = nullptr;
    cudaEvent_t async_score_ev = nullptr, async_join_ev = nullptr;
    cudaEvent_t async_done[2] = {};
    bool async_used[2] = {false, false};
    bool last_user_async = false;
    int async_par = 0;
    int cur_par = 0;  // parity the scratch pointers below currently hold
    float* q_eps_p[2] = {};
    int32_t* slice_cnt_p[2] = {};
    float* cta_topk_p[2] = {};
    int32_t* cand_slot_p[2] = {};
    float* cand_score_p[2] = {};
    uint8_t* prank_p[2] = {};  // IVF probe ranks (read by the finish kernel)
    // pipelined host path (sw_warmstart_host_submit / _wait): kPipe staging slots, H2D on
    // pipe_in, D2H on pipe_out, so batch i+1's copies overlap batch i's kernels
    static constexpr int kPipe = 3;
    std::mutex pipe_mu;
    int64_t pipe_seq = 0;
    cudaStream_t pipe_in = nullptr, pipe_out = nullptr, pipe_al = nullptr;
    cudaEvent_t pipe_h2d[kPipe] = {}, pipe_used[kPipe] = {}, pipe_done[kPipe] = {},
                pipe_planned[kPipe] = {};
    float* pipe_q[kPipe] = {};
    sw_request* pipe_req[kPipe] = {};
    sw_choice* pipe_ch[kPipe] = {};
    // stage profiling (CUDA events on the launching stream; single-threaded use)
    bool prof = false;
    uint32_t prof_mask = 0xFFu;         // stages recorded while prof is on
    std::vector<cudaEvent_t> prof_ev;   // pool, pairs (start, stop)
    std::vector<int> prof_stage;        // stage of each recorded pair
    size_t prof_used = 0;
    double prof_ms[SW_NUM_STAGES] = {};
    int64_t prof_n[SW_NUM_STAGES] = {};
    // synchronous host entry points (sw_search_host, sw_score_select_host, sw_gater_host):
    // persistent staging and stream, so a per-request call allocates nothing
    std::mutex host_mu;
    cudaStream_t host_st = nullptr;
    void* host_stage = nullptr;
    size_t host_stage_bytes = 0;
    // last launch info
    int last_kernels = 0, last_tc = 0, last_cand_max = 0;
    // dynamic shared-memory opt-ins already applied on this context's device (the attribute is
    // per device, so it cannot be a process-wide static)
    std::mutex attr_mu;
    std::map<const void*, size_t> smem_attr;
    // K4 (align.cu): the per-request geometry written by the pre-pass; launches chained through
    // k4_ev so two align launches on different streams never share it concurrently
    std::mutex k4_mu;
    char* k4_state = nullptr;
    int k4_cap = 0;
    cudaEvent_t k4_ev = nullptr;
};

// Host <-> device copies and fills outside the batched hot path: stream-ordered on the context's
// mutation stream and complete on return. A plain cudaMemcpy / cudaMemset runs on the legacy
// default stream, which does NOT order against the non-blocking mutation / caller streams: a
// pageable H2D may still be in flight when a kernel launched right after on mstream reads its
// destination (this raced the IVF k-means and corrupted host state under heavy churn).
inline void mcopy(Ctx& c, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
    if (bytes == 0) return;
    SW_CUDA(cudaMemcpyAsync(dst, src, bytes, kind, c.mstream));
    SW_CUDA(cudaStreamSynchronize(c.mstream));
}
// A typed device temporary for mutation code: carved from the context's scratch stack (LIFO
// with the scoped objects), falling back to cudaMalloc when the stack is exhausted. All users
// touch it on mstream only, so stream order makes the reuse of a popped region safe.
template <typename T>
struct MScratch {
    Ctx& c;
    T* p = nullptr;
    size_t bytes = 0;
    bool owned = false;
    MScratch(Ctx& cc, size_t n) : c(cc) {
        bytes = (sizeof(T) * std::max<size_t>(n, 1) + 255) & ~(size_t)255;
        if (!c.mscratch) {
            c.mscratch_cap = (size_t)32 << 20;
            SW_CUDA(cudaMalloc((void**)&c.mscratch, c.mscratch_cap));
        }
        if (c.mscratch_top + bytes <= c.mscratch_cap) {
            p = reinterpret_cast<T*>(c.mscratch + c.mscratch_top);
            c.mscratch_top += bytes;
        } else {
            SW_CUDA(cudaMalloc((void**)&p, bytes));
            owned = true;
        }
    }
    ~MScratch() {
        if (owned) cudaFree(p);
        else c.mscratch_top -= bytes;
    }
    MScratch(const MScratch&) = delete;
    MScratch& operator=(const MScratch&) = delete;
};

inline void mfill(Ctx& c, void* dst, int value, size_t bytes) {
    if (bytes == 0) return;
    SW_CUDA(cudaMemsetAsync(dst, value, bytes, c.mstream));
    SW_CUDA(cudaStreamSynchronize(c.mstream));
}

// nprobe of the current search: a per-call override (search(q, k, nprobe)) or set_nprobe's
inline int eff_nprobe(const Ctx& c) { return c.nprobe_override > 0 ? c.nprobe_override : c.ivf_nprobe; }

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (context, kernel, size high-water).
template <class K>
inline void ensure_smem_attr(Ctx& c, K* kern, size_t bytes) {
    std::lock_guard<std::mutex> lk(c.attr_mu);
    size_t& have = c.smem_attr[reinterpret_cast<const void*>(kern)];
    if (bytes <= have) return;
    SW_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    have = bytes;
}

// Reader guard of the hot path: shared with other readers against arena mutations, exclusive
// with them on the batch scratch (host enqueue under scratch_mu, device work after the previous
// reader's via scratch_ev).
struct HotGuard {
    std::shared_lock<std::shared_mutex> rd;
    std::unique_lock<std::mutex> sc;
    Ctx& c;
    cudaStream_t st;
    HotGuard(Ctx& c_, cudaStream_t st_) : rd(c_.mu), sc(c_.scratch_mu), c(c_), st(st_) {
        cudaSetDevice(c.device);
        if (c.scratch_ev) cudaStreamWaitEvent(st, c.scratch_ev, 0);
        // a call enqueued on the async stream (the sharded merge / align after
        // sw_local_topk_async) is part of that pipeline, not a synchronous user
        if (st != c.async_st) c.last_user_async = false;
    }
    ~HotGuard() {
        if (c.scratch_ev) cudaEventRecord(c.scratch_ev, st);
    }
};

// RAII stage timer: records a (start, stop) event pair around the enclosed launches.
struct StageScope {
    Ctx& c;
    cudaStream_t st;
    size_t pair = (size_t)-1;
    StageScope(Ctx& cc, int stage, cudaStream_t s) : c(cc), st(s) {
        if (!c.prof || !((c.prof_mask >> stage) & 1u)) return;
        if (2 * (c.prof_used + 1) > c.prof_ev.size()) {
            for (int i = 0; i < 2; ++i) {
                cudaEvent_t e;
                if (cudaEventCreate(&e) != cudaSuccess) return;
                c.prof_ev.push_back(e);
            }
            c.prof_stage.push_back(0);
        }
        pair = c.prof_used++;
        c.prof_stage[pair] = stage;
        cudaEventRecord(c.prof_ev[2 * pair], st);
    }
    ~StageScope() {
        if (pair != (size_t)-1) cudaEventRecord(c.prof_ev[2 * pair + 1], st);
    }
};

// kernel-side launchers (implemented in the .cu files)
void launch_insert_rows_full(Ctx& c, int64_t n, const int64_t* d_slot, const int32_t* d_base,
                             const int64_t* d_row_off, const uint64_t* d_ids, const float* d_rows,
                             const sw_segment* d_segs, cudaStream_t st);
void launch_copy_latents(Ctx& c, int64_t n, const int64_t* d_slot, const float* d_lat,
                         const int64_t* d_lat_off, const int32_t* d_tsrc, cudaStream_t st);
void launch_recompute_sneg(Ctx& c, cudaStream_t st);
void launch_choice_rows(Ctx& c, const sw_choice* d_ch, int B, float* d_rows, cudaStream_t st);
void launch_clear_slot(Ctx& c, int64_t slot, cudaStream_t st);
void launch_fill_synthetic(Ctx& c, int64_t slot0, int64_t n, uint64_t first_id, uint64_t seed,
                           double delta, cudaStream_t st);

int launch_prep(Ctx& c, const float* d_q, int B, const sw_request* d_req, uint64_t seed,
                cudaStream_t st);
int launch_search(Ctx& c, const float* d_q, int B, int k, int rank, cudaStream_t st);
int launch_search_fused(Ctx& c, const float* d_q, int B, int k, int rank, const sw_request* d_req,
                        const dev::SelParams* sp, sw_choice* d_out, cudaStream_t st,
                        cudaStream_t st_finish);
int launch_search_fused(Ctx& c, const float* d_q, int B, int k, int rank, const sw_request* d_req,
                        const dev::SelParams* sp, sw_choice* d_out, cudaStream_t st);
void launch_hits_to_public(Ctx& c, int B, int k, sw_hit* d_out, int32_t* d_n, cudaStream_t st);
void launch_select(Ctx& c, const HitRec* d_hits, const int32_t* d_nh, int ld, const float* d_q,
                   const sw_request* d_req, int B, uint64_t seed, const sw_selector_config& sel,
                   const sw_policy& pol, sw_choice* d_out, uint32_t extra_flags_mask,
                   cudaStream_t st);
void launch_merge(Ctx& c, const HitRec* d_gathered, const int32_t* d_gn, int world, int B,
                  int k, cudaStream_t st);
int launch_align_noise(Ctx& c, const sw_choice* d_ch, const sw_request* d_req, int B,
                        int rank, const float* d_eps, uint64_t seed, float* d_out, int t_out_max,
                        cudaStream_t st);
void launch_score_select_one(Ctx& c, int n, const double* d_sims, const double* d_sneg,
                             const double* d_dur, double L, const sw_selector_config& sel,
                             uint64_t rng_seed, double* d_scores, int32_t* d_pick,
                             cudaStream_t st);
void launch_score_candidates(int n, int D, const double* d_sims, const float* d_audio,
                             const double* d_dur, const float* d_neg, double L, double* d_scores,
                             cudaStream_t st);
void launch_select_draw(int n, const double* d_spos, const double* d_q, double temp, double thr,
                        double u, int32_t* d_pick, cudaStream_t st);
void launch_gater(Ctx& c, const float* d_p, const float* d_s, const int32_t* d_T, int B,
                  int explore, double* d_phi, int32_t* d_arm, cudaStream_t st);

bool encode_tensor_maps(Ctx& c);
// IVF coarse quantiser (ivf.cu)
void ivf_rebuild(Ctx& c);
void ivf_on_insert(Ctx& c, const std::vector<int64_t>& slot, const std::vector<int32_t>& base,
                   const std::vector<int32_t>& nr);
void ivf_on_remove(Ctx& c, int64_t slot);
void ivf_mark_tails(Ctx& c, const std::vector<int64_t>& slots, const std::vector<int32_t>& nr);
void ivf_set_centroids(Ctx& c, const float* h, int C);
void ivf_build_from(Ctx& c, const std::vector<int64_t>& perm);
bool ivf_check_consistent(Ctx& c);
bool launch_probe_rank(Ctx& c, const float* d_q, int B, cudaStream_t st);
// grouped IVF search: returns the upper bound of work items (0 = grouped path not applicable)
int64_t ivf_group_prepare(Ctx& c, int B, cudaStream_t st);
bool encode_2d_map(CUtensorMap* m, void* base, uint64_t inner, uint64_t rows, uint32_t box_rows);
int launch_score_tc_grouped(Ctx& c, int B, int k, int64_t max_items, cudaStream_t st);
// phase-vocoder time stretch (vocoder.cu)
const int32_t* launch_align_vocoder(Ctx& c, const sw_choice* d_ch, const sw_request* d_req,
                                    int B, int rank, float* d_out, int t_out_max,
                                    cudaStream_t st);
int time_stretch_batch(const float* d_in, const int64_t* in_off, const int32_t* in_len, int B,
                       int rate, const double* target_s, int n, int hop_a, float* d_out,
                       int64_t out_cap, int64_t* out_off, int32_t* out_len, int32_t* status,
                       cudaStream_t st);
// snapshots (host/snapshot.cpp)
void swix_load(Ctx& c, const char* path, void (*insert)(Ctx&, int64_t, const uint64_t*,
                                                        const int64_t*, const float*,
                                                        const sw_segment*));
void swix_save(Ctx& c, const char* path);
int64_t swem_read(const char* path, float* out, int64_t cap_floats, int32_t* count, int32_t* dim);
void swmb_read(const char* path, std::vector<float>& theta, std::vector<float>& psi, int& fd);
void swmb_write(const char* path, const float* theta, const float* psi, int fd);

}  // namespace sw
