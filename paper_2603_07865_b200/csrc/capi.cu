// The C-ABI (include/semwarm_b200.h): context lifetime, arena mutations (synchronous, exclusive)
// and the stream-ordered batched hot path. No exception crosses this boundary.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "select_dev.cuh"

struct sw_ctx {
    sw::Ctx c;
};

namespace sw {

static thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }

template <class F>
static int guarded(F&& f) {
    try {
        return f();
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return SW_ENOMEM;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return SW_ERUNTIME;
    }
}

static int next_pow2(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

template <class T>
static void dalloc(T** p, size_t n) {
    if (n == 0) n = 1;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * n);
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw Error(SW_ENOMEM, std::string("cudaMalloc of ") + std::to_string(sizeof(T) * n) +
                                   " bytes failed: " + cudaGetErrorString(e));
    }
}

// (s0, s1) = ((float)sqrt(abar), (float)sqrt(1 - abar)) per schedule index, rounded exactly as the
// restatement rounds them (IEEE double sqrt, then to float)
static std::vector<float2> noise_coefficients(const std::vector<double>& abar) {
    std::vector<float2> s(abar.size());
    for (size_t i = 0; i < abar.size(); ++i)
        s[i] = make_float2((float)std::sqrt(abar[i]), (float)std::sqrt(1.0 - abar[i]));
    return s;
}

static void default_schedule(std::vector<double>& abar) {
    // scaled-linear DDPM betas 0.00085..0.012 over 1000 steps (the LDM/AudioLDM default)
    abar.assign(1001, 1.0);
    const double b0 = std::sqrt(0.00085), b1 = std::sqrt(0.012);
    for (int t = 1; t <= 1000; ++t) {
        double s = b0 + (b1 - b0) * (double)(t - 1) / 999.0;
        abar[t] = abar[t - 1] * (1.0 - s * s);
    }
}

// Arena mutations (exclusive on the host) must also come after every reader's device work:
// hot-path calls return before their kernels run (the async path's finish and align even run
// on the context's own stream), and every one of them ends with scratch_ev.
// (host-side wait: the mutation paths use several streams and synchronous copies)
static void wait_readers(Ctx& c) {
    if (c.scratch_ev) SW_CUDA(cudaEventSynchronize(c.scratch_ev));
}

static void free_ctx(Ctx& c) {
    if (c.async_st) {  // the scratch fields hold parity 0 again; free parity 1 separately
        c.q_eps = c.q_eps_p[0];
        c.slice_cnt = c.slice_cnt_p[0];
        c.cta_topk = c.cta_topk_p[0];
        c.cand_slot = c.cand_slot_p[0];
        c.cand_score = c.cand_score_p[0];
        c.prank = c.prank_p[0];
        for (void* q : {(void*)c.q_eps_p[1], (void*)c.slice_cnt_p[1], (void*)c.cta_topk_p[1],
                        (void*)c.cand_slot_p[1], (void*)c.cand_score_p[1], (void*)c.prank_p[1]})
            if (q) cudaFree(q);
        for (cudaEvent_t e : {c.async_score_ev, c.async_join_ev, c.async_done[0], c.async_done[1]})
            if (e) cudaEventDestroy(e);
        cudaStreamDestroy(c.async_st);
    }
    void* ptrs[] = {c.rows, c.rows_bf, c.sneg, c.segs, c.ids, c.nrows, c.valid, c.valid_bits,
                    c.slice_cnt, c.cta_topk, c.dbg, c.tsrc, c.mscratch,
                    c.latent, c.norms, c.neg, c.theta, c.psi, c.abar, c.s01, c.q_bf, c.q_norm, c.q_eps,
                    c.thr, c.top1, c.cand_n, c.cand_slot, c.cand_score, c.cand_exact, c.cand_row,
                    c.cand_list, c.ovf_state, c.ovf_ring, c.hits, c.nhits, c.d_q_stage, c.d_req_stage, c.d_choice_stage,
                    c.cent, c.row_list, c.prank, c.pmask, c.d_sorted_slot, c.d_rows_sorted,
                    c.d_sorted_vbits, c.d_list_tile0, c.d_list_ntiles, c.d_qcnt, c.d_qlist,
                    c.d_qbase, c.d_qg, c.d_qmap, c.d_items, c.d_voc, c.k4_state};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (c.h_pinned) cudaFreeHost(c.h_pinned);
    for (cudaEvent_t e : c.prof_ev) cudaEventDestroy(e);
    if (c.scratch_ev) cudaEventDestroy(c.scratch_ev);
    if (c.k4_ev) cudaEventDestroy(c.k4_ev);
    for (int i = 0; i < Ctx::kPipe; ++i) {
        if (c.pipe_q[i]) cudaFree(c.pipe_q[i]);
        if (c.pipe_req[i]) cudaFree(c.pipe_req[i]);
        if (c.pipe_ch[i]) cudaFree(c.pipe_ch[i]);
        for (cudaEvent_t e : {c.pipe_h2d[i], c.pipe_used[i], c.pipe_done[i], c.pipe_planned[i]})
            if (e) cudaEventDestroy(e);
    }
    if (c.pipe_in) cudaStreamDestroy(c.pipe_in);
    if (c.pipe_out) cudaStreamDestroy(c.pipe_out);
    if (c.pipe_al) cudaStreamDestroy(c.pipe_al);
    if (c.mstream) cudaStreamDestroy(c.mstream);
    if (c.host_st) cudaStreamDestroy(c.host_st);
    if (c.host_stage) cudaFree(c.host_stage);
}

static void create(Ctx& c, const sw_config& cfg, int device) {
    SW_REQUIRE(cfg.dim >= 1, "dim must be >= 1");
    SW_REQUIRE(cfg.rows_per_entry >= 1 && cfg.rows_per_entry <= kMaxRowsPad,
               "rows_per_entry must be in [1, 32]");
    SW_REQUIRE(cfg.max_entries >= 1, "cache capacity must be >= 1");  // cache.cpp:16
    SW_REQUIRE(cfg.max_batch >= 1, "max_batch must be >= 1");
    c.cfg = cfg;
    if (c.cfg.latent_fps <= 0.0) c.cfg.latent_fps = 25.0;
    c.device = device;
    SW_CUDA(cudaSetDevice(device));
    c.D = cfg.dim;
    c.Dp = (cfg.dim + 63) / 64 * 64;
    c.Df = (cfg.dim + 3) / 4 * 4;
    c.R = cfg.rows_per_entry;
    c.Rp = next_pow2(cfg.rows_per_entry);
    c.logRp = 0;
    while ((1 << c.logRp) < c.Rp) ++c.logRp;
    // round capacity up to whole 256-row tiles so TMA boxes never straddle the allocation. One
    // spare slot beyond max_entries: CacheManager::admit inserts BEFORE it evicts (cache.cpp:
    // 30-52), so a full cache holds capacity + 1 entries for the duration of an admit.
    const int64_t per_tile = std::max(1, 256 / c.Rp);
    c.S = (cfg.max_entries + 1 + per_tile - 1) / per_tile * per_tile;
    c.C = cfg.latent_c;
    c.Tmax = cfg.latent_t_max;
    c.F = cfg.latent_f;
    c.Lslots = cfg.latent_slots > 0 ? std::min<int64_t>(cfg.latent_slots, c.S) : c.S;
    c.Bmax = cfg.max_batch;
    c.BmaxPad = (cfg.max_batch + 127) / 128 * 128;
    const int64_t nrow = c.S * c.Rp;
    SW_CUDA(cudaStreamCreateWithFlags(&c.mstream, cudaStreamNonBlocking));
    dalloc(&c.rows, (size_t)nrow * c.Df);
    dalloc(&c.rows_bf, (size_t)nrow * c.Dp);
    dalloc(&c.sneg, (size_t)nrow);
    dalloc(&c.segs, (size_t)nrow);
    dalloc(&c.ids, (size_t)c.S);
    dalloc(&c.nrows, (size_t)c.S);
    dalloc(&c.valid, (size_t)c.S);
    dalloc(&c.valid_bits, (size_t)(c.S / 32 + 16));
    dalloc(&c.tsrc, (size_t)c.S);
    if (c.C > 0 && c.Tmax > 0 && c.F > 0)
        dalloc(&c.latent, (size_t)c.Lslots * c.C * c.Tmax * c.F);
    dalloc(&c.norms, 4);
    dalloc(&c.neg, (size_t)c.Df);
    dalloc(&c.theta, kNumArms * kFeatureDim);
    dalloc(&c.psi, kNumArms * kFeatureDim);
    dalloc(&c.q_bf, (size_t)c.BmaxPad * c.Dp);
    dalloc(&c.q_norm, (size_t)c.Bmax);
    dalloc(&c.q_eps, (size_t)c.Bmax);
    dalloc(&c.thr, (size_t)c.Bmax);
    dalloc(&c.top1, (size_t)c.Bmax * kMaxSlices);
    dalloc(&c.cand_n, (size_t)3 * c.Bmax);
    dalloc(&c.slice_cnt, (size_t)c.Bmax * kMaxSlices);
    dalloc(&c.cta_topk, (size_t)c.Bmax * kMaxSlices * kMaxTopK);
    dalloc(&c.dbg, (size_t)c.Bmax * 8);
    dalloc(&c.cand_slot, (size_t)c.Bmax * kCandCap);
    dalloc(&c.cand_score, (size_t)c.Bmax * kCandCap);
    dalloc(&c.cand_exact, (size_t)c.Bmax * kCandCap);
    dalloc(&c.cand_row, (size_t)c.Bmax * kCandCap);
    dalloc(&c.cand_list, (size_t)c.Bmax * kCandCap);
    dalloc(&c.hits, (size_t)c.Bmax * kMaxTopK);
    {
        const int64_t chunks = (c.Bmax + kOvfQG - 1) / kOvfQG;
        const size_t words = (size_t)kOvfHdr + (size_t)c.Bmax + 2 * (size_t)chunks;
        dalloc(&c.ovf_state, words);
        mfill(c, c.ovf_state, 0, sizeof(int32_t) * words);
        int nsm = 0;
        SW_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
        const size_t rec = 16;  // {double sim, int32 slot, int32 row}
        SW_CUDA(cudaMalloc(&c.ovf_ring, rec * kOvfRing * kOvfQG * (size_t)nsm * kOvfWarps * kMaxTopK));
    }
    dalloc(&c.nhits, (size_t)c.Bmax);
    dalloc(&c.d_q_stage, (size_t)c.Bmax * c.D);
    dalloc(&c.d_req_stage, (size_t)c.Bmax);
    dalloc(&c.d_choice_stage, (size_t)c.Bmax);
    dalloc(&c.cent, (size_t)kMaxCentroids * c.Df);
    dalloc(&c.row_list, (size_t)nrow);
    dalloc(&c.prank, (size_t)c.Bmax * kMaxCentroids);
    dalloc(&c.pmask, (size_t)c.Bmax * 4);
    c.ivf_rows.assign((size_t)c.S, 0);
    mfill(c, c.row_list, 0xFF, sizeof(int16_t) * (size_t)nrow);  // no list
    SW_CUDA(cudaMemsetAsync(c.valid, 0, (size_t)c.S, c.mstream));
    SW_CUDA(cudaMemsetAsync(c.valid_bits, 0, sizeof(uint32_t) * (size_t)(c.S / 32 + 16), c.mstream));
    SW_CUDA(cudaMemsetAsync(c.nrows, 0, sizeof(int32_t) * (size_t)c.S, c.mstream));
    SW_CUDA(cudaMemsetAsync(c.tsrc, 0, sizeof(int32_t) * (size_t)c.S, c.mstream));
    SW_CUDA(cudaMemsetAsync(c.rows_bf, 0, sizeof(__nv_bfloat16) * (size_t)nrow * c.Dp, c.mstream));
    SW_CUDA(cudaMemsetAsync(c.q_bf, 0, sizeof(__nv_bfloat16) * (size_t)c.BmaxPad * c.Dp, c.mstream));
    SW_CUDA(cudaMemsetAsync(c.neg, 0, sizeof(float) * c.Df, c.mstream));
    SW_CUDA(cudaMemsetAsync(c.theta, 0, sizeof(float) * kNumArms * kFeatureDim, c.mstream));
    SW_CUDA(cudaMemsetAsync(c.psi, 0, sizeof(float) * kNumArms * kFeatureDim, c.mstream));
    const uint32_t zero_norm[4] = {f2ord(0.0f), f2ord(0.0f), f2ord(0.0f), f2ord(0.0f)};
    SW_CUDA(cudaMemcpyAsync(c.norms, zero_norm, 16, cudaMemcpyHostToDevice, c.mstream));
    std::vector<double> ab;
    default_schedule(ab);
    dalloc(&c.abar, ab.size());
    dalloc(&c.s01, ab.size());
    c.n_abar = (int)ab.size();
    SW_CUDA(cudaMemcpyAsync(c.abar, ab.data(), sizeof(double) * ab.size(), cudaMemcpyHostToDevice,
                            c.mstream));
    c.h_s01 = noise_coefficients(ab);
    SW_CUDA(cudaMemcpyAsync(c.s01, c.h_s01.data(), sizeof(float2) * ab.size(),
                            cudaMemcpyHostToDevice, c.mstream));
    c.h_pinned_bytes = (size_t)c.Bmax * (sizeof(float) * c.D + sizeof(sw_request) + sizeof(sw_choice));
    SW_CUDA(cudaMallocHost(&c.h_pinned, c.h_pinned_bytes));
    SW_CUDA(cudaStreamSynchronize(c.mstream));
    c.h_nrows.assign((size_t)c.S, 0);
    int major = 0, minor = 0;
    SW_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    SW_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
    SW_CUDA(cudaDeviceGetAttribute(&c.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    SW_CUDA(cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, device));
    c.tc_ok = major == 10 && minor == 0 && encode_tensor_maps(c);
    SW_CUDA(cudaEventCreateWithFlags(&c.scratch_ev, cudaEventDisableTiming));
}

// Reallocates a device array from n_old to n_new elements, keeping the first n_old and
// filling the tail with byte `fill`.
template <class T>
static void regrow(Ctx& c, T** p, size_t n_old, size_t n_new, int fill) {
    T* q = nullptr;
    dalloc(&q, n_new);
    if (*p && n_old) mcopy(c, q, *p, sizeof(T) * n_old, cudaMemcpyDeviceToDevice);
    mfill(c, q + n_old, fill, sizeof(T) * (n_new - n_old));
    if (*p) cudaFree(*p);
    *p = q;
}

// Grows the arena to hold at least `entries` entries (+1 spare, whole tiles): every per-slot and
// per-row array is reallocated and copied, the TMA descriptors re-encoded. Caller holds c.mu
// exclusively with no reader in flight.
static void grow_arena(Ctx& c, int64_t entries) {
    const int64_t per_tile = std::max(1, 256 / c.Rp);
    const int64_t S2 = (entries + 1 + per_tile - 1) / per_tile * per_tile;
    if (S2 <= c.S) return;
    const int64_t S = c.S, nrow = S * c.Rp, nrow2 = S2 * c.Rp;
    regrow(c, &c.rows, (size_t)nrow * c.Df, (size_t)nrow2 * c.Df, 0);
    regrow(c, &c.rows_bf, (size_t)nrow * c.Dp, (size_t)nrow2 * c.Dp, 0);
    regrow(c, &c.sneg, (size_t)nrow, (size_t)nrow2, 0);
    regrow(c, &c.segs, (size_t)nrow, (size_t)nrow2, 0);
    regrow(c, &c.row_list, (size_t)nrow, (size_t)nrow2, 0xFF);
    regrow(c, &c.ids, (size_t)S, (size_t)S2, 0);
    regrow(c, &c.nrows, (size_t)S, (size_t)S2, 0);
    regrow(c, &c.valid, (size_t)S, (size_t)S2, 0);
    regrow(c, &c.tsrc, (size_t)S, (size_t)S2, 0);
    regrow(c, &c.valid_bits, (size_t)(S / 32 + 16), (size_t)(S2 / 32 + 16), 0);
    const int64_t L2 = c.cfg.latent_slots > 0 ? std::min<int64_t>(c.cfg.latent_slots, S2) : S2;
    if (c.latent && L2 != c.Lslots) {  // slot % Lslots is unchanged for every stored slot
        const size_t per = (size_t)c.C * c.Tmax * c.F;
        regrow(c, &c.latent, (size_t)c.Lslots * per, (size_t)L2 * per, 0);
    }
    c.Lslots = L2;
    c.S = S2;
    c.h_nrows.resize((size_t)S2, 0);
    c.ivf_rows.resize((size_t)S2, 0);
    c.grp_dirty = true;
    const int major_ok = c.tc_ok;
    c.tc_ok = major_ok && encode_tensor_maps(c);
}

// Reserve slots for n new entries (lowest free slot first) and update host bookkeeping.
static int64_t take_slot(Ctx& c) {
    if (!c.free_slots.empty()) {
        int64_t s = *c.free_slots.begin();
        c.free_slots.erase(c.free_slots.begin());
        return s;
    }
    if (c.high_water >= c.S) throw Error(SW_ENOMEM, "arena full (max_entries reached)");
    return c.high_water++;
}

struct InsertPlan {
    std::vector<int64_t> slot;
    std::vector<int32_t> base;
};

// Stage host inputs and run the insert kernels on the mutation stream (synchronously).
static void do_insert(Ctx& c, int64_t n, const uint64_t* ids, const int64_t* row_off,
                      const float* rows, const sw_segment* segs, const float* latents,
                      const int64_t* lat_off, const int32_t* t_src, bool on_device) {
    InsertPlan pl;
    pl.slot.resize((size_t)n);
    pl.base.resize((size_t)n);
    std::vector<uint64_t> h_ids((size_t)n);
    std::vector<int64_t> h_off((size_t)n + 1);
    if (on_device) {
        mcopy(c, h_ids.data(), ids, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost);
        mcopy(c, h_off.data(), row_off, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost);
    } else {
        std::memcpy(h_ids.data(), ids, sizeof(uint64_t) * n);
        std::memcpy(h_off.data(), row_off, sizeof(int64_t) * (n + 1));
    }
    // validate everything before mutating any state
    std::unordered_map<uint64_t, int32_t> pending;
    for (int64_t e = 0; e < n; ++e) {
        const int64_t nr = h_off[e + 1] - h_off[e];
        SW_REQUIRE(nr >= 0, "row offsets must be non-decreasing");
        auto it = c.slot_of.find(h_ids[e]);
        int32_t have = it == c.slot_of.end() ? 0 : c.h_nrows[(size_t)it->second];
        have += pending[h_ids[e]];
        SW_REQUIRE(have + nr <= c.Rp && have + nr <= kMaxRowsPad,
                   "entry has more rows than the arena's rows_per_entry");
        pending[h_ids[e]] += (int32_t)nr;
    }
    // slots: every id not yet in the arena takes one; check they exist before any mutation
    // (a partial batch would leave ids in slot_of whose rows were never written)
    int64_t new_ids = 0;
    for (const auto& kv : pending)
        if (!c.slot_of.count(kv.first)) ++new_ids;
    if ((int64_t)c.free_slots.size() + (c.S - c.high_water) < new_ids) {
        if (!(c.cfg.flags & SW_FLAG_GROW)) throw Error(SW_ENOMEM, "arena full (max_entries reached)");
        const int64_t need = c.high_water + new_ids - (int64_t)c.free_slots.size();
        grow_arena(c, std::max<int64_t>(2 * c.S, need));  // SW_FLAG_GROW: double (amortised)
    }
    for (int64_t e = 0; e < n; ++e) {
        const int64_t nr = h_off[e + 1] - h_off[e];
        auto it = c.slot_of.find(h_ids[e]);
        if (it == c.slot_of.end()) {
            const int64_t s = take_slot(c);
            c.slot_of[h_ids[e]] = s;
            pl.slot[e] = s;
            pl.base[e] = 0;
        } else {
            pl.slot[e] = it->second;
            pl.base[e] = c.h_nrows[(size_t)it->second];
        }
        c.h_nrows[(size_t)pl.slot[e]] = pl.base[e] + (int32_t)nr;
    }
    cudaStream_t st = c.mstream;
    const int64_t total_rows = h_off[n] - h_off[0];
    // temporaries on the mutation scratch stack (no cudaMalloc / cudaFree per admit)
    MScratch<int64_t> s_slot(c, (size_t)n);
    MScratch<int32_t> s_base(c, (size_t)n);
    int64_t *d_slot = s_slot.p, *d_off = nullptr, *d_latoff = nullptr;
    int32_t *d_base = s_base.p, *d_tsrc = nullptr;
    uint64_t* d_ids = nullptr;
    float *d_rows = nullptr, *d_lat = nullptr;
    sw_segment* d_segs = nullptr;
    const bool host_src = !on_device;
    MScratch<uint64_t> s_ids(c, host_src ? (size_t)n : 0);
    MScratch<int64_t> s_off(c, host_src ? (size_t)n + 1 : 0);
    MScratch<float> s_rows(c, host_src ? (size_t)std::max<int64_t>(1, h_off[n]) * c.D : 0);
    MScratch<sw_segment> s_segs(c, host_src ? (size_t)std::max<int64_t>(1, h_off[n]) : 0);
    SW_CUDA(cudaMemcpyAsync(d_slot, pl.slot.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
    SW_CUDA(cudaMemcpyAsync(d_base, pl.base.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    if (on_device) {
        d_ids = const_cast<uint64_t*>(ids);
        d_off = const_cast<int64_t*>(row_off);
        d_rows = const_cast<float*>(rows);
        d_segs = const_cast<sw_segment*>(segs);
    } else {
        d_ids = s_ids.p;
        d_off = s_off.p;
        d_rows = s_rows.p;
        d_segs = s_segs.p;
        SW_CUDA(cudaMemcpyAsync(d_ids, ids, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, st));
        SW_CUDA(cudaMemcpyAsync(d_off, row_off, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, st));
        if (total_rows > 0) {
            SW_CUDA(cudaMemcpyAsync(d_rows, rows, sizeof(float) * h_off[n] * c.D,
                                    cudaMemcpyHostToDevice, st));
            SW_CUDA(cudaMemcpyAsync(d_segs, segs, sizeof(sw_segment) * h_off[n],
                                    cudaMemcpyHostToDevice, st));
        }
    }
    launch_insert_rows_full(c, n, d_slot, d_base, d_off, d_ids, d_rows, d_segs, st);
    int64_t lat_tot = 0;
    if (latents && c.latent && !on_device)
        for (int64_t e = 0; e < n; ++e)
            lat_tot = std::max<int64_t>(lat_tot, lat_off[e] + (int64_t)c.C * t_src[e] * c.F);
    const bool host_lat = latents && c.latent && !on_device;
    MScratch<float> s_lat(c, host_lat ? (size_t)std::max<int64_t>(lat_tot, 1) : 0);
    MScratch<int64_t> s_latoff(c, host_lat ? (size_t)n : 0);
    MScratch<int32_t> s_tsrc(c, host_lat ? (size_t)n : 0);
    if (latents && c.latent) {
        if (on_device) {
            d_lat = const_cast<float*>(latents);
            d_latoff = const_cast<int64_t*>(lat_off);
            d_tsrc = const_cast<int32_t*>(t_src);
        } else {
            const int64_t tot = lat_tot;
            d_lat = s_lat.p;
            d_latoff = s_latoff.p;
            d_tsrc = s_tsrc.p;
            SW_CUDA(cudaMemcpyAsync(d_lat, latents, sizeof(float) * tot, cudaMemcpyHostToDevice, st));
            SW_CUDA(cudaMemcpyAsync(d_latoff, lat_off, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
            SW_CUDA(cudaMemcpyAsync(d_tsrc, t_src, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
        }
        launch_copy_latents(c, n, d_slot, d_lat, d_latoff, d_tsrc, st);
    }
    SW_CUDA(cudaStreamSynchronize(st));
    if (c.ivf) {  // IvfIndex::insert per entry, in order (index.cpp:224-234)
        std::vector<int32_t> nr((size_t)n);
        for (int64_t e = 0; e < n; ++e) nr[(size_t)e] = (int32_t)(h_off[e + 1] - h_off[e]);
        ivf_on_insert(c, pl.slot, pl.base, nr);
    }
}

static void do_remove(Ctx& c, uint64_t id, bool* found) {
    auto it = c.slot_of.find(id);
    if (it == c.slot_of.end()) {
        *found = false;
        return;
    }
    *found = true;
    const int64_t s = it->second;
    c.slot_of.erase(it);
    c.h_nrows[(size_t)s] = 0;
    launch_clear_slot(c, s, c.mstream);
    SW_CUDA(cudaStreamSynchronize(c.mstream));
    if (c.ivf) ivf_on_remove(c, s);  // IvfIndex::remove (index.cpp:236-255)
    if (s == c.high_water - 1) {
        --c.high_water;
        // trim trailing free slots so the scan range stays tight
        while (c.high_water > 0 && c.free_slots.count(c.high_water - 1)) {
            c.free_slots.erase(c.high_water - 1);
            --c.high_water;
        }
    } else {
        c.free_slots.insert(s);
    }
}

static cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static void bulk_insert(Ctx& c, int64_t n, const uint64_t* ids, const int64_t* off,
                        const float* rows, const sw_segment* segs) {
    do_insert(c, n, ids, off, rows, segs, nullptr, nullptr, nullptr, false);
}

}  // namespace sw

using namespace sw;

extern "C" {

int sw_version(void) { return 1; }

int sw_ctx_info(sw_ctx* ctx, int32_t* dim, int32_t* latent_c, int32_t* latent_t_max,
                int32_t* latent_f, int32_t* max_batch, int32_t* device) {
    if (!ctx) return SW_EINVAL;
    const Ctx& c = ctx->c;
    if (dim) *dim = c.D;
    if (latent_c) *latent_c = c.latent ? c.C : 0;
    if (latent_t_max) *latent_t_max = c.Tmax;
    if (latent_f) *latent_f = c.F;
    if (max_batch) *max_batch = c.Bmax;
    if (device) *device = c.device;
    return SW_OK;
}

const char* sw_last_error(void) { return g_last_error.c_str(); }

int sw_ctx_create(const sw_config* cfg, int device, sw_ctx** out) {
    return guarded([&] {
        SW_REQUIRE(cfg && out, "null argument");
        auto* h = new sw_ctx;
        try {
            create(h->c, *cfg, device);
        } catch (...) {
            free_ctx(h->c);
            delete h;
            throw;
        }
        *out = h;
        return SW_OK;
    });
}

int sw_ctx_destroy(sw_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return SW_OK;
        cudaSetDevice(ctx->c.device);
        cudaDeviceSynchronize();
        free_ctx(ctx->c);
        delete ctx;
        return SW_OK;
    });
}

int sw_set_negative(sw_ctx* ctx, const float* neg) {
    return guarded([&] {
        SW_REQUIRE(ctx && neg, "null argument");
        Ctx& c = ctx->c;
        std::unique_lock lk(c.mu);
        wait_readers(c);
        SW_CUDA(cudaSetDevice(c.device));
        SW_CUDA(cudaMemcpyAsync(c.neg, neg, sizeof(float) * c.D, cudaMemcpyHostToDevice, c.mstream));
        c.have_neg = true;
        launch_recompute_sneg(c, c.mstream);
        SW_CUDA(cudaStreamSynchronize(c.mstream));
        return SW_OK;
    });
}

int sw_set_gater(sw_ctx* ctx, const float* theta, const float* psi, int32_t fd, double beta) {
    return guarded([&] {
        SW_REQUIRE(ctx && theta && psi, "null argument");
        SW_REQUIRE(fd == kFeatureDim, "feature dim mismatch");  // gater.cpp:62
        Ctx& c = ctx->c;
        std::unique_lock lk(c.mu);
        wait_readers(c);
        SW_CUDA(cudaSetDevice(c.device));
        SW_CUDA(cudaMemcpyAsync(c.theta, theta, sizeof(float) * kNumArms * fd, cudaMemcpyHostToDevice, c.mstream));
        SW_CUDA(cudaMemcpyAsync(c.psi, psi, sizeof(float) * kNumArms * fd, cudaMemcpyHostToDevice, c.mstream));
        SW_CUDA(cudaStreamSynchronize(c.mstream));
        c.beta = beta;
        c.fd = fd;
        return SW_OK;
    });
}

int sw_set_schedule(sw_ctx* ctx, const double* abar, int32_t n) {
    return guarded([&] {
        SW_REQUIRE(ctx && abar && n >= 2, "schedule needs >= 2 entries");
        Ctx& c = ctx->c;
        std::unique_lock lk(c.mu);
        wait_readers(c);
        SW_CUDA(cudaSetDevice(c.device));
        if (n != c.n_abar) {
            cudaFree(c.abar);
            cudaFree(c.s01);
            c.abar = nullptr;
            c.s01 = nullptr;
            dalloc(&c.abar, (size_t)n);
            dalloc(&c.s01, (size_t)n);
            c.n_abar = n;
        }
        mcopy(c, c.abar, abar, sizeof(double) * n, cudaMemcpyHostToDevice);
        c.h_s01 = noise_coefficients(std::vector<double>(abar, abar + n));
        mcopy(c, c.s01, c.h_s01.data(), sizeof(float2) * n, cudaMemcpyHostToDevice);
        return SW_OK;
    });
}

int sw_arena_insert(sw_ctx* ctx, uint64_t id, int32_t n_rows, const float* rows,
                    const sw_segment* segs, const float* latent, int32_t t_src) {
    return guarded([&] {
        SW_REQUIRE(ctx && (n_rows == 0 || (rows && segs)), "null argument");
        SW_REQUIRE(n_rows >= 0, "n_rows must be >= 0");
        if (n_rows == 0) return SW_OK;  // IvfIndex::insert of nothing (index.cpp:227)
        Ctx& c = ctx->c;
        std::unique_lock lk(c.mu);
        wait_readers(c);
        SW_CUDA(cudaSetDevice(c.device));
        int64_t off[2] = {0, n_rows};
        int64_t loff = 0;
        do_insert(c, 1, &id, off, rows, segs, latent, &loff, &t_src, false);
        return SW_OK;
    });
}

int sw_arena_insert_batch(sw_ctx* ctx, int64_t n, const uint64_t* ids, const int64_t* row_off,
                          const float* rows, const sw_segment* segs, const float* latents,
                          const int64_t* lat_off, const int32_t* t_src, int32_t on_device) {
    return guarded([&] {
        SW_REQUIRE(ctx && ids && row_off, "null argument");
        if (n <= 0) return SW_OK;
        Ctx& c = ctx->c;
        std::unique_lock lk(c.mu);
        wait_readers(c);
        SW_CUDA(cudaSetDevice(c.device));
        do_insert(c, n, ids, row_off, rows, segs, latents, lat_off, t_src, on_device != 0);
        return SW_OK;
    });
}

int sw_arena_remove(sw_ctx* ctx, uint64_t id) {
    return guarded([&] {
        SW_REQUIRE(ctx, "null argument");
        Ctx& c = ctx->c;
        std::unique_lock lk(c.mu);
        wait_readers(c);
        SW_CUDA(cudaSetDevice(c.device));
        bool found = false;
        do_remove(c, id, &found);
        if (!found) {
            set_last_error("remove of unknown entry id " + std::to_string(id));
            return SW_WARN_UNKNOWN_ID;
        }
        return SW_OK;
    });
}

int sw_arena_replace(sw_ctx* ctx, uint64_t id, int32_t n_rows, const float* rows,
                     const sw_segment* segs, const float* latent, int32_t t_src) {
    return guarded([&] {
        SW_REQUIRE(ctx && rows && segs && n_rows >= 1, "bad argument");
        Ctx& c = ctx->c;
        std::unique_lock lk(c.mu);
        wait_readers(c);
        SW_CUDA(cudaSetDevice(c.device));
        auto it = c.slot_of.find(id);
        if (it == c.slot_of.end()) {
            set_last_error("replace of unknown entry id " + std::to_string(id));
            return SW_WARN_UNKNOWN_ID;
        }
        SW_REQUIRE(n_rows <= c.Rp, "entry has more rows than the arena's rows_per_entry");
        // in place: same slot, rows rewritten from row 0 (CacheManager::refine, cache.cpp:129-139)
        // The reference re-indexes with remove + insert; in IVF mode both count as mutations
        // and either may trigger a rebuild (the remove's without this entry).
        if (c.ivf) ivf_on_remove(c, it->second);
        c.h_nrows[(size_t)it->second] = 0;
        int64_t off[2] = {0, n_rows};
        int64_t loff = 0;
        do_insert(c, 1, &id, off, rows, segs, latent, &loff, &t_src, false);
        return SW_OK;
    });
}

int64_t sw_arena_entry_count(const sw_ctx* ctx) {
    if (!ctx) return 0;
    std::shared_lock lk(ctx->c.mu);
    return (int64_t)ctx->c.slot_of.size();
}

int64_t sw_arena_capacity(const sw_ctx* ctx) {
    if (!ctx) return 0;
    std::shared_lock lk(ctx->c.mu);
    return ctx->c.S;
}

int sw_arena_reserve(sw_ctx* ctx, int64_t max_entries) {
    return guarded([&] {
        SW_REQUIRE(ctx && max_entries >= 1, "bad argument");
        Ctx& c = ctx->c;
        std::unique_lock lk(c.mu);
        wait_readers(c);
        SW_CUDA(cudaSetDevice(c.device));
        grow_arena(c, max_entries);
        return SW_OK;
    });
}

int64_t sw_arena_row_count(const sw_ctx* ctx) {  // IvfIndex::total_vectors (index.hpp:70)
    if (!ctx) return 0;
    std::shared_lock lk(ctx->c.mu);
    int64_t n = 0;
    for (const auto& kv : ctx->c.slot_of) n += ctx->c.h_nrows[(size_t)kv.second];
    return n;
}

int64_t sw_arena_export(sw_ctx* ctx, int64_t first, int64_t count, uint64_t* ids,
                        int32_t* nrows, float* rows, sw_segment* segs) {
    try {
        SW_REQUIRE(ctx && ids && nrows, "null argument");
        Ctx& c = ctx->c;
        std::shared_lock lk(c.mu);
        SW_CUDA(cudaSetDevice(c.device));
        // live entries in slot order; count is how many to return starting at the first-th
        std::vector<std::pair<int64_t, uint64_t>> live;
        live.reserve(c.slot_of.size());
        for (const auto& kv : c.slot_of) live.emplace_back(kv.second, kv.first);
        std::sort(live.begin(), live.end());
        const int64_t total = (int64_t)live.size();
        if (first >= total || count <= 0) return 0;
        const int64_t n = std::min(count, total - first);
        const int64_t s0 = live[(size_t)first].first, s1 = live[(size_t)(first + n - 1)].first + 1;
        std::vector<float> blk;
        std::vector<sw_segment> sblk;
        if (rows) blk.resize((size_t)(s1 - s0) * c.Rp * c.Df);
        if (segs) sblk.resize((size_t)(s1 - s0) * c.Rp);
        if (rows)
            mcopy(c, blk.data(), c.rows + s0 * c.Rp * c.Df, sizeof(float) * blk.size(),
                  cudaMemcpyDeviceToHost);
        if (segs)
            mcopy(c, sblk.data(), c.segs + s0 * c.Rp, sizeof(sw_segment) * sblk.size(),
                  cudaMemcpyDeviceToHost);
        for (int64_t i = 0; i < n; ++i) {
            const int64_t slot = live[(size_t)(first + i)].first;
            ids[i] = live[(size_t)(first + i)].second;
            nrows[i] = c.h_nrows[(size_t)slot];
            for (int r = 0; r < c.Rp; ++r) {
                const size_t src = (size_t)((slot - s0) * c.Rp + r);
                if (rows)
                    std::memcpy(rows + ((size_t)i * c.Rp + r) * c.D, blk.data() + src * c.Df,
                                sizeof(float) * c.D);
                if (segs) segs[(size_t)i * c.Rp + r] = sblk[src];
            }
        }
        return n;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return SW_ERUNTIME;
    }
}

int sw_index_check_consistent(sw_ctx* ctx) {
    try {
        if (!ctx) return 0;
        Ctx& c = ctx->c;
        std::unique_lock lk(c.mu);
        wait_readers(c);
        SW_CUDA(cudaSetDevice(c.device));
        int64_t valid = 0;
        for (const auto& kv : c.slot_of) valid += c.h_nrows[(size_t)kv.second] > 0 ? 1 : 0;
        std::vector<uint8_t> v((size_t)c.high_water);
        if (c.high_water)
            mcopy(c, v.data(), c.valid, (size_t)c.high_water, cudaMemcpyDeviceToHost);
        int64_t dv = 0;
        for (uint8_t x : v) dv += x ? 1 : 0;
        if (dv != valid) return 0;
        return ivf_check_consistent(c) ? 1 : 0;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return 0;
    }
}

int sw_arena_contains(const sw_ctx* ctx, uint64_t id) {
    if (!ctx) return 0;
    std::shared_lock lk(ctx->c.mu);
    return ctx->c.slot_of.count(id) ? 1 : 0;
}

int sw_arena_fill_synthetic(sw_ctx* ctx, int64_t n, uint64_t first_id, uint64_t seed, double delta) {
    return guarded([&] {
        SW_REQUIRE(ctx && n >= 0, "bad argument");
        Ctx& c = ctx->c;
        std::unique_lock lk(c.mu);
        wait_readers(c);
        SW_CUDA(cudaSetDevice(c.device));
        SW_REQUIRE(c.free_slots.empty(), "synthetic fill needs a compact arena");
        SW_REQUIRE(c.high_water + n <= c.S, "arena full (max_entries reached)");
        for (int64_t i = 0; i < n; ++i)
            SW_REQUIRE(!c.slot_of.count(first_id + (uint64_t)i), "synthetic id collides");
        const int64_t slot0 = c.high_water;
        launch_fill_synthetic(c, slot0, n, first_id, seed, delta, c.mstream);
        SW_CUDA(cudaStreamSynchronize(c.mstream));
        for (int64_t i = 0; i < n; ++i) {
            c.slot_of[first_id + (uint64_t)i] = slot0 + i;
            c.h_nrows[(size_t)(slot0 + i)] = c.R;
            c.ivf_rows[(size_t)(slot0 + i)] = c.R;
        }
        c.high_water += n;
        // IVF mode: a bulk load like IvfIndex::build(vecs) — no mutation counting; rows join the
        // current centroids' lists (sw_ivf_rebuild re-clusters)
        if (c.ivf) {
            std::vector<int64_t> sl((size_t)n);
            for (int64_t i = 0; i < n; ++i) sl[(size_t)i] = slot0 + i;
            ivf_mark_tails(c, sl, std::vector<int32_t>((size_t)n, c.R));
            if (c.ivf_C > 0) ivf_set_centroids(c, c.h_cent.data(), c.ivf_C);
        }
        return SW_OK;
    });
}

// ---------------------------------------------------------------- IVF coarse quantiser
int sw_ivf_configure(sw_ctx* ctx, int32_t centroids, int32_t nprobe, uint64_t rebuild_interval,
                     uint64_t seed) {
    return guarded([&] {
        SW_REQUIRE(ctx, "null argument");
        SW_REQUIRE(centroids >= 1, "centroid count must be >= 1");  // index.cpp:191
        SW_REQUIRE(centroids <= kMaxCentroids, "at most 256 centroids are supported");
        SW_REQUIRE(nprobe >= 1, "nprobe must be >= 1");
        SW_REQUIRE(rebuild_interval >= 1, "rebuild interval must be >= 1");
        Ctx& c = ctx->c;
        std::unique_lock lk(c.mu);
        wait_readers(c);
        SW_REQUIRE(c.slot_of.empty(), "configure the IVF index on an empty arena");
        c.ivf = true;
        c.ivf_target = centroids;
        c.ivf_nprobe = nprobe;
        c.ivf_interval = rebuild_interval;
        c.ivf_seed = seed;
        c.ivf_C = 0;
        c.ivf_mutations = 0;
        c.ivf_rebuilds = 0;
        c.h_cent.clear();
        return SW_OK;
    });
}

int sw_ivf_config(sw_ctx* ctx, int32_t* enabled, int32_t* centroids, int32_t* nprobe,
                  uint64_t* rebuild_interval, uint64_t* seed) {
    return guarded([&] {
        SW_REQUIRE(ctx, "null argument");
        Ctx& c = ctx->c;
        std::shared_lock lk(c.mu);
        if (enabled) *enabled = c.ivf ? 1 : 0;
        if (centroids) *centroids = c.ivf_target;
        if (nprobe) *nprobe = c.ivf_nprobe;
        if (rebuild_interval) *rebuild_interval = c.ivf_interval;
        if (seed) *seed = c.ivf_seed;
        return SW_OK;
    });
}

int sw_ivf_set_rebuild_interval(sw_ctx* ctx, uint64_t interval) {
    return guarded([&] {  // IvfIndex::set_rebuild_interval (index.hpp:76)
        SW_REQUIRE(ctx && interval >= 1, "rebuild interval must be >= 1");
        std::unique_lock lk(ctx->c.mu);
        wait_readers(ctx->c);
        ctx->c.ivf_interval = interval;
        return SW_OK;
    });
}

int sw_ivf_build(sw_ctx* ctx, int64_t n, const uint64_t* ids, const int64_t* row_off,
                 const float* rows, const sw_segment* segs) {
    return guarded([&] {
        SW_REQUIRE(ctx && (n == 0 || (ids && row_off && rows && segs)), "null argument");
        Ctx& c = ctx->c;
        std::unique_lock lk(c.mu);
        wait_readers(c);
        SW_REQUIRE(c.ivf, "the context is not in IVF mode (sw_ivf_configure)");
        SW_REQUIRE(c.slot_of.empty(), "IvfIndex::build needs an empty arena");
        SW_CUDA(cudaSetDevice(c.device));
        if (n > 0) {
            c.ivf = false;  // a bulk load: no mutation counting, no list assignment yet
            try {
                do_insert(c, n, ids, row_off, rows, segs, nullptr, nullptr, nullptr, false);
            } catch (...) {
                c.ivf = true;
                throw;
            }
            c.ivf = true;
        }
        std::vector<int64_t> perm;  // rows in the vecs order
        std::unordered_map<uint64_t, int32_t> seen;
        for (int64_t e = 0; e < n; ++e) {
            const int64_t slot = c.slot_of.at(ids[e]);
            const int32_t nr = (int32_t)(row_off[e + 1] - row_off[e]);
            const int32_t b = seen[ids[e]];
            for (int r = 0; r < nr; ++r) perm.push_back(slot * c.Rp + b + r);
            seen[ids[e]] = b + nr;
            c.ivf_rows[(size_t)slot] = b + nr;
        }
        ivf_build_from(c, perm);
        return SW_OK;
    });
}

int sw_ivf_set_nprobe(sw_ctx* ctx, int32_t nprobe) {
    return guarded([&] {
        SW_REQUIRE(ctx && nprobe >= 1, "bad argument");
        std::unique_lock lk(ctx->c.mu);
        wait_readers(ctx->c);
        ctx->c.ivf_nprobe = nprobe;
        return SW_OK;
    });
}

int sw_ivf_rebuild(sw_ctx* ctx) {
    return guarded([&] {
        SW_REQUIRE(ctx, "null argument");
        Ctx& c = ctx->c;
        std::unique_lock lk(c.mu);
        wait_readers(c);
        SW_REQUIRE(c.ivf, "the context is not in IVF mode (sw_ivf_configure)");
        SW_CUDA(cudaSetDevice(c.device));
        ivf_rebuild(c);
        return SW_OK;
    });
}

int sw_ivf_info(sw_ctx* ctx, int32_t* n_centroids, uint64_t* mutations, uint64_t* rebuilds) {
    return guarded([&] {
        SW_REQUIRE(ctx, "null argument");
        std::shared_lock lk(ctx->c.mu);
        if (n_centroids) *n_centroids = ctx->c.ivf ? ctx->c.ivf_C : 1;
        if (mutations) *mutations = ctx->c.ivf_mutations;
        if (rebuilds) *rebuilds = ctx->c.ivf_rebuilds;
        return SW_OK;
    });
}

int sw_ivf_centroids(sw_ctx* ctx, float* out, int32_t cap) {
    return guarded([&] {
        SW_REQUIRE(ctx && (out || cap == 0), "null argument");
        Ctx& c = ctx->c;
        std::shared_lock lk(c.mu);
        const int n = std::min(cap, c.ivf_C);
        std::memcpy(out, c.h_cent.data(), sizeof(float) * (size_t)n * c.D);
        return c.ivf_C;
    });
}

int sw_ivf_set_centroids(sw_ctx* ctx, const float* centroids, int32_t n) {
    return guarded([&] {
        SW_REQUIRE(ctx && (centroids || n == 0), "null argument");
        SW_REQUIRE(n >= 0 && n <= kMaxCentroids, "at most 256 centroids are supported");
        Ctx& c = ctx->c;
        std::unique_lock lk(c.mu);
        wait_readers(c);
        SW_REQUIRE(c.ivf, "the context is not in IVF mode (sw_ivf_configure)");
        SW_CUDA(cudaSetDevice(c.device));
        ivf_set_centroids(c, centroids, n);
        return SW_OK;
    });
}

int sw_ivf_entry_lists(sw_ctx* ctx, uint64_t id, int16_t* lists, int32_t cap) {
    return guarded([&] {
        SW_REQUIRE(ctx && lists, "null argument");
        Ctx& c = ctx->c;
        std::shared_lock lk(c.mu);
        auto it = c.slot_of.find(id);
        if (it == c.slot_of.end()) return 0;
        const int nr = std::min(cap, c.ivf_rows[(size_t)it->second]);
        mcopy(c, lists, c.row_list + it->second * c.Rp, sizeof(int16_t) * nr,
              cudaMemcpyDeviceToHost);
        return nr;
    });
}

// ---------------------------------------------------------------- phase vocoder
int sw_set_align_mode(sw_ctx* ctx, int32_t mode, int32_t window, int32_t hop) {
    return guarded([&] {
        SW_REQUIRE(ctx, "null argument");
        SW_REQUIRE(mode == SW_ALIGN_CROP_TILE || mode == SW_ALIGN_VOCODER, "unknown align mode");
        SW_REQUIRE(window >= 2 && (window & (window - 1)) == 0 && window <= 1024,
                   "stft window size must be a power of two >= 2 (at most 1024 here)");
        SW_REQUIRE(hop >= 1 && hop <= window, "stft hop must be in (0, window_size]");
        Ctx& c = ctx->c;
        std::unique_lock lk(c.mu);
        wait_readers(c);
        c.align_mode = mode;
        c.voc_win = window;
        c.voc_hop = hop;
        return SW_OK;
    });
}

int sw_time_stretch(const float* d_in, const int64_t* in_off, const int32_t* in_len, int32_t B,
                    int32_t sample_rate, const double* target_s, int32_t window, int32_t hop,
                    float* d_out, int64_t out_cap, int64_t* out_off, int32_t* out_len,
                    int32_t* status, void* stream) {
    return guarded([&] {
        SW_REQUIRE(B >= 0 && (B == 0 || (d_in && in_off && in_len && target_s && d_out &&
                                         out_off && out_len && status)),
                   "null argument");
        time_stretch_batch(d_in, in_off, in_len, B, sample_rate, target_s, window, hop, d_out,
                           out_cap, out_off, out_len, status, as_stream(stream));
        return SW_OK;
    });
}

// ---------------------------------------------------------------- snapshots
int sw_swix_load(sw_ctx* ctx, const char* path) {
    return guarded([&] {
        SW_REQUIRE(ctx && path, "null argument");
        Ctx& c = ctx->c;
        std::unique_lock lk(c.mu);
        wait_readers(c);
        SW_CUDA(cudaSetDevice(c.device));
        swix_load(c, path, &bulk_insert);
        return SW_OK;
    });
}

int sw_swix_save(sw_ctx* ctx, const char* path) {
    return guarded([&] {
        SW_REQUIRE(ctx && path, "null argument");
        Ctx& c = ctx->c;
        std::unique_lock lk(c.mu);
        wait_readers(c);
        SW_CUDA(cudaSetDevice(c.device));
        swix_save(c, path);
        return SW_OK;
    });
}

int sw_gater_load_swmb(sw_ctx* ctx, const char* path, double beta) {
    return guarded([&] {
        SW_REQUIRE(ctx && path, "null argument");
        std::vector<float> theta, psi;
        int fd = 0;
        swmb_read(path, theta, psi, fd);
        SW_REQUIRE(fd == kFeatureDim, "feature dim mismatch");  // gater.cpp:62
        return sw_set_gater(ctx, theta.data(), psi.data(), fd, beta);
    });
}

int sw_gater_save_swmb(sw_ctx* ctx, const char* path) {
    return guarded([&] {
        SW_REQUIRE(ctx && path, "null argument");
        Ctx& c = ctx->c;
        std::shared_lock lk(c.mu);
        SW_CUDA(cudaSetDevice(c.device));
        std::vector<float> theta((size_t)kNumArms * c.fd), psi((size_t)kNumArms * c.fd);
        mcopy(c, theta.data(), c.theta, sizeof(float) * theta.size(), cudaMemcpyDeviceToHost);
        mcopy(c, psi.data(), c.psi, sizeof(float) * psi.size(), cudaMemcpyDeviceToHost);
        swmb_write(path, theta.data(), psi.data(), c.fd);
        return SW_OK;
    });
}

int64_t sw_swem_read(const char* path, float* out, int64_t cap_floats, int32_t* count,
                     int32_t* dim) {
    try {
        SW_REQUIRE(path, "null argument");
        return swem_read(path, out, cap_floats, count, dim);
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return SW_ERUNTIME;
    }
}

int sw_arena_read_rows(sw_ctx* ctx, uint64_t id, float* rows, int32_t cap) {
    return guarded([&] {
        SW_REQUIRE(ctx && rows, "null argument");
        Ctx& c = ctx->c;
        std::shared_lock lk(c.mu);
        SW_CUDA(cudaSetDevice(c.device));
        auto it = c.slot_of.find(id);
        if (it == c.slot_of.end()) return -1;
        const int n = std::min(cap, c.h_nrows[(size_t)it->second]);
        SW_CUDA(cudaMemcpy2DAsync(rows, sizeof(float) * c.D, c.rows + it->second * c.Rp * c.Df,
                                  sizeof(float) * c.Df, sizeof(float) * c.D, n,
                                  cudaMemcpyDeviceToHost, c.mstream));
        SW_CUDA(cudaStreamSynchronize(c.mstream));
        return n;
    });
}

int sw_search(sw_ctx* ctx, const float* d_q, int32_t B, int32_t k, sw_hit* d_out, int32_t* d_n,
              void* stream) {
    return guarded([&] {
        SW_REQUIRE(ctx && (B == 0 || (d_q && d_out && d_n)), "null argument");
        Ctx& c = ctx->c;
        HotGuard lk(c, as_stream(stream));
        SW_CUDA(cudaSetDevice(c.device));
        cudaStream_t st = as_stream(stream);
        int kn = launch_search(c, d_q, B, k, 0, st);
        launch_hits_to_public(c, B, k, d_out, d_n, st);
        c.last_kernels = kn + 1;
        return SW_OK;
    });
}

// Persistent staging for the synchronous host entry points (grows, never shrinks). Caller
// holds c.host_mu.
static void* host_stage(Ctx& c, size_t bytes) {
    if (!c.host_st) SW_CUDA(cudaStreamCreateWithFlags(&c.host_st, cudaStreamNonBlocking));
    if (bytes > c.host_stage_bytes) {
        if (c.host_stage) cudaFree(c.host_stage);
        c.host_stage = nullptr;
        c.host_stage_bytes = 0;
        const size_t nb = std::max<size_t>(bytes, 64 * 1024);
        SW_CUDA(cudaMalloc(&c.host_stage, nb));
        c.host_stage_bytes = nb;
    }
    return c.host_stage;
}

static int search_host_impl(Ctx& c, const float* q, int32_t B, int32_t k, int32_t nprobe,
                            sw_hit* out, int32_t* n) {
    SW_REQUIRE(B <= c.Bmax, "batch exceeds the context's max_batch");
    SW_REQUIRE(k >= 1, "search k must be >= 1");  // index.cpp:291
    SW_CUDA(cudaSetDevice(c.device));
    std::lock_guard<std::mutex> hl(c.host_mu);
    const size_t hit_bytes = sizeof(sw_hit) * (size_t)std::max(1, B * k);
    char* stage = static_cast<char*>(host_stage(c, hit_bytes + sizeof(int32_t) * (size_t)B + 256));
    sw_hit* d_out = reinterpret_cast<sw_hit*>(stage);
    int32_t* d_n = reinterpret_cast<int32_t*>(stage + (hit_bytes + 255) / 256 * 256);
    cudaStream_t st = c.host_st;
    int rc = SW_OK;
    {
        HotGuard lk(c, st);
        SW_CUDA(cudaMemcpyAsync(c.d_q_stage, q, sizeof(float) * (size_t)B * c.D,
                                cudaMemcpyHostToDevice, st));
        c.nprobe_override = nprobe;
        int kn;
        try {
            kn = launch_search(c, c.d_q_stage, B, k, 0, st);
        } catch (...) {
            c.nprobe_override = 0;
            throw;
        }
        c.nprobe_override = 0;
        launch_hits_to_public(c, B, k, d_out, d_n, st);
        c.last_kernels = kn + 1;
        SW_CUDA(cudaMemcpyAsync(out, d_out, sizeof(sw_hit) * (size_t)B * k, cudaMemcpyDeviceToHost, st));
        SW_CUDA(cudaMemcpyAsync(n, d_n, sizeof(int32_t) * B, cudaMemcpyDeviceToHost, st));
    }
    SW_CUDA(cudaStreamSynchronize(st));
    for (int b = 0; b < B; ++b)
        if (n[b] < 0) {  // never expected: the fallback certifies every overflow
            n[b] = -n[b] - 1;
            set_last_error("search result not certified (candidate overflow)");
            rc = SW_ERUNTIME;
        }
    return rc;
}

int sw_search_host(sw_ctx* ctx, const float* q, int32_t B, int32_t k, sw_hit* out, int32_t* n) {
    return guarded([&] {
        SW_REQUIRE(ctx && (B == 0 || (q && out && n)), "null argument");
        if (B == 0) return SW_OK;
        return search_host_impl(ctx->c, q, B, k, 0, out, n);
    });
}

int sw_search_host_ex(sw_ctx* ctx, const float* q, int32_t B, int32_t k, int32_t nprobe,
                      sw_hit* out, int32_t* n) {
    return guarded([&] {
        SW_REQUIRE(ctx && (B == 0 || (q && out && n)), "null argument");
        SW_REQUIRE(nprobe >= 0, "nprobe must be >= 0");
        if (B == 0) return SW_OK;
        return search_host_impl(ctx->c, q, B, k, nprobe, out, n);
    });
}

static void check_sel(const sw_selector_config* sel, const sw_policy* pol) {
    SW_REQUIRE(sel && pol, "null selector config or policy");
    SW_REQUIRE(sel->top_k >= 1, "selector top_k must be >= 1");               // selector.cpp:9
    SW_REQUIRE(sel->top_k <= kMaxTopK, "selector top_k above 32 is not supported");
    SW_REQUIRE(sel->temperature > 0.0, "selector temperature must be > 0");   // selector.cpp:10
    SW_REQUIRE(sel->quality_threshold >= 0.0 && sel->quality_threshold <= 1.0,
               "selector quality threshold must be in [0, 1]");            // selector.cpp:11-13
    SW_REQUIRE(pol->kind >= 0 && pol->kind <= 3, "unknown gater policy");
    SW_REQUIRE(pol->kind != SW_POLICY_FIXED || (pol->fixed_arm >= 0 && pol->fixed_arm < kNumArms),
               "arm index out of range");                                  // gater.hpp:17
}

static int plan_impl(Ctx& c, const float* d_q, const sw_request* d_req, int B, uint64_t seed,
                     const sw_selector_config* sel, const sw_policy* pol, sw_choice* d_out,
                     cudaStream_t st, cudaStream_t st_finish = nullptr) {
    check_sel(sel, pol);
    const dev::SelParams sp = dev::make_sel_params(c, seed, *sel, *pol);
    return launch_search_fused(c, d_q, B, sel->top_k, 0, d_req, &sp, d_out, st,
                               st_finish ? st_finish : st);
}

// ---------------------------------------------------------------- cross-batch pipelining
static void set_par(Ctx& c, int par) {
    c.q_eps = c.q_eps_p[par];
    c.slice_cnt = c.slice_cnt_p[par];
    c.cta_topk = c.cta_topk_p[par];
    c.cand_slot = c.cand_slot_p[par];
    c.cand_score = c.cand_score_p[par];
    c.prank = c.prank_p[par];
    c.cur_par = par;
}

static void ensure_async(Ctx& c) {
    if (c.async_st) return;
    SW_CUDA(cudaStreamCreateWithFlags(&c.async_st, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&c.async_score_ev, &c.async_join_ev, &c.async_done[0], &c.async_done[1]})
        SW_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    c.q_eps_p[0] = c.q_eps;
    c.slice_cnt_p[0] = c.slice_cnt;
    c.cta_topk_p[0] = c.cta_topk;
    c.cand_slot_p[0] = c.cand_slot;
    c.cand_score_p[0] = c.cand_score;
    c.prank_p[0] = c.prank;
    dalloc(&c.prank_p[1], (size_t)c.Bmax * kMaxCentroids);
    dalloc(&c.q_eps_p[1], (size_t)c.Bmax);
    dalloc(&c.slice_cnt_p[1], (size_t)c.Bmax * kMaxSlices);
    dalloc(&c.cta_topk_p[1], (size_t)c.Bmax * kMaxSlices * kMaxTopK);
    dalloc(&c.cand_slot_p[1], (size_t)c.Bmax * kCandCap);
    dalloc(&c.cand_score_p[1], (size_t)c.Bmax * kCandCap);
    c.cur_par = 0;
}

// Batch i: prep + scoring on S, finish + align + noise on c.async_st. The buffers finish(i)
// reads alternate parity, so scoring(i + 1) on S overlaps finish(i) (the scoring kernel is
// capped at 4 ring stages, leaving shared memory for one finish CTA per SM) and align(i).
// Caller holds c.mu (shared) and c.scratch_mu. Returns the kernel count.
static int warmstart_async_impl(Ctx& c, const float* d_q, const sw_request* d_req, int B,
                                uint64_t seed, const sw_selector_config* sel, const sw_policy* pol,
                                const float* d_eps, uint64_t philox_seed, sw_choice* d_ch,
                                float* d_out, int t_out_max, cudaStream_t S) {
    ensure_async(c);
    const int par = c.async_par;
    if (c.async_used[par]) SW_CUDA(cudaStreamWaitEvent(S, c.async_done[par], 0));
    // the previous async call's prep + scoring may sit on another caller stream: the single-
    // buffered scoring scratch (bf16 queries, thresholds, slice bests) is reused right away
    if (c.async_used[par ^ 1]) SW_CUDA(cudaStreamWaitEvent(S, c.async_score_ev, 0));
    if (!c.last_user_async && c.scratch_ev) SW_CUDA(cudaStreamWaitEvent(S, c.scratch_ev, 0));
    set_par(c, par);
    const int kn = plan_impl(c, d_q, d_req, B, seed, sel, pol, d_ch, S, c.async_st);
    const int ka =
        launch_align_noise(c, d_ch, d_req, B, -1, d_eps, philox_seed, d_out, t_out_max, c.async_st);
    SW_CUDA(cudaEventRecord(c.async_done[par], c.async_st));
    if (c.scratch_ev) SW_CUDA(cudaEventRecord(c.scratch_ev, c.async_st));  // for later sync users
    c.async_used[par] = true;
    c.async_par = par ^ 1;
    c.last_user_async = true;
    return kn + ka;
}

int sw_plan(sw_ctx* ctx, const float* d_q, const sw_request* d_req, int32_t B, uint64_t seed,
            const sw_selector_config* sel, const sw_policy* pol, sw_choice* d_out, void* stream) {
    return guarded([&] {
        SW_REQUIRE(ctx && (B == 0 || (d_q && d_req && d_out)), "null argument");
        Ctx& c = ctx->c;
        HotGuard lk(c, as_stream(stream));
        SW_CUDA(cudaSetDevice(c.device));
        c.last_kernels = plan_impl(c, d_q, d_req, B, seed, sel, pol, d_out, as_stream(stream));
        return SW_OK;
    });
}

int sw_align_noise(sw_ctx* ctx, const sw_choice* d_ch, const sw_request* d_req, int32_t B,
                   const float* d_eps, uint64_t philox_seed, float* d_out, int32_t t_out_max,
                   void* stream) {
    return guarded([&] {
        SW_REQUIRE(ctx && (B == 0 || (d_ch && d_req && d_out)), "null argument");
        SW_REQUIRE(t_out_max >= 1, "t_out_max must be >= 1");
        Ctx& c = ctx->c;
        std::shared_lock lk(c.mu);
        SW_CUDA(cudaSetDevice(c.device));
        launch_align_noise(c, d_ch, d_req, B, -1, d_eps, philox_seed, d_out, t_out_max,
                           as_stream(stream));
        return SW_OK;
    });
}

int sw_align_noise_owned(sw_ctx* ctx, const sw_choice* d_ch, const sw_request* d_req, int32_t B,
                         int32_t rank, const float* d_eps, uint64_t philox_seed, float* d_out,
                         int32_t t_out_max, void* stream) {
    return guarded([&] {
        SW_REQUIRE(ctx && (B == 0 || (d_ch && d_req && d_out)), "null argument");
        Ctx& c = ctx->c;
        std::shared_lock lk(c.mu);
        SW_CUDA(cudaSetDevice(c.device));
        launch_align_noise(c, d_ch, d_req, B, rank, d_eps, philox_seed, d_out, t_out_max,
                           as_stream(stream));
        return SW_OK;
    });
}

int sw_warmstart(sw_ctx* ctx, const float* d_q, const sw_request* d_req, int32_t B, uint64_t seed,
                 const sw_selector_config* sel, const sw_policy* pol, const float* d_eps,
                 uint64_t philox_seed, sw_choice* d_ch, float* d_out, int32_t t_out_max,
                 void* stream) {
    return guarded([&] {
        SW_REQUIRE(ctx && (B == 0 || (d_q && d_req && d_ch && d_out)), "null argument");
        Ctx& c = ctx->c;
        HotGuard lk(c, as_stream(stream));
        SW_CUDA(cudaSetDevice(c.device));
        cudaStream_t st = as_stream(stream);
        int kn = plan_impl(c, d_q, d_req, B, seed, sel, pol, d_ch, st);
        kn += launch_align_noise(c, d_ch, d_req, B, -1, d_eps, philox_seed, d_out, t_out_max, st);
        c.last_kernels = kn;
        return SW_OK;
    });
}

// Pipelined host path: the same work as sw_warmstart_host, returned before it completes.
// Submission n uses staging slot n mod kPipe: its H2D runs on pipe_in once the slot's previous
// batch has consumed it, the kernels on the caller's stream after that H2D (and after the
// previous hot-path user, HotGuard), the D2H of the choices on pipe_out after the kernels. So
// batch n+1's prompts cross PCIe while batch n is being scored.
int sw_warmstart_host_submit(sw_ctx* ctx, const float* q, const sw_request* reqs, int32_t B,
                             uint64_t seed, const sw_selector_config* sel, const sw_policy* pol,
                             uint64_t philox_seed, sw_choice* choices, float* d_out,
                             int32_t t_out_max, void* stream, int64_t* ticket) {
    return guarded([&] {
        SW_REQUIRE(ctx && ticket && (B == 0 || (q && reqs && choices && d_out)), "null argument");
        Ctx& c = ctx->c;
        SW_REQUIRE(B <= c.Bmax, "batch exceeds the context's max_batch");
        std::lock_guard<std::mutex> pl(c.pipe_mu);
        SW_CUDA(cudaSetDevice(c.device));
        if (!c.pipe_in) {
            SW_CUDA(cudaStreamCreateWithFlags(&c.pipe_in, cudaStreamNonBlocking));
            SW_CUDA(cudaStreamCreateWithFlags(&c.pipe_out, cudaStreamNonBlocking));
            for (int i = 0; i < Ctx::kPipe; ++i) {
                SW_CUDA(cudaMalloc(&c.pipe_q[i], sizeof(float) * (size_t)c.Bmax * c.D));
                SW_CUDA(cudaMalloc(&c.pipe_req[i], sizeof(sw_request) * (size_t)c.Bmax));
                SW_CUDA(cudaMalloc(&c.pipe_ch[i], sizeof(sw_choice) * (size_t)c.Bmax));
                for (cudaEvent_t* e :
                     {&c.pipe_h2d[i], &c.pipe_used[i], &c.pipe_done[i], &c.pipe_planned[i]})
                    SW_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
                SW_CUDA(cudaEventRecord(c.pipe_used[i], c.pipe_in));
            }
        }
        const int slot = (int)(c.pipe_seq % Ctx::kPipe);
        cudaStream_t st = as_stream(stream);
        SW_CUDA(cudaStreamWaitEvent(c.pipe_in, c.pipe_used[slot], 0));
        SW_CUDA(cudaStreamWaitEvent(c.pipe_in, c.pipe_done[slot], 0));  // its choices are home
        SW_CUDA(cudaMemcpyAsync(c.pipe_q[slot], q, sizeof(float) * (size_t)B * c.D,
                                cudaMemcpyHostToDevice, c.pipe_in));
        SW_CUDA(cudaMemcpyAsync(c.pipe_req[slot], reqs, sizeof(sw_request) * (size_t)B,
                                cudaMemcpyHostToDevice, c.pipe_in));
        SW_CUDA(cudaEventRecord(c.pipe_h2d[slot], c.pipe_in));
        {
            // plan's prep + scoring on the caller's stream; finish, align + noise on the
            // context's async stream (under the next batch's scoring)
            std::shared_lock<std::shared_mutex> rd(c.mu);
            std::unique_lock<std::mutex> sc(c.scratch_mu);
            SW_CUDA(cudaStreamWaitEvent(st, c.pipe_h2d[slot], 0));
            const int par = c.async_st ? c.async_par : 0;
            c.last_kernels = warmstart_async_impl(c, c.pipe_q[slot], c.pipe_req[slot], B, seed,
                                                  sel, pol, nullptr, philox_seed,
                                                  c.pipe_ch[slot], d_out, t_out_max, st);
            const cudaEvent_t done = c.async_done[par];
            SW_CUDA(cudaEventRecord(c.pipe_used[slot], c.async_st ? c.async_st : st));
            SW_CUDA(cudaStreamWaitEvent(c.pipe_out, done, 0));
            if (c.async_st) SW_CUDA(cudaStreamWaitEvent(c.pipe_out, c.pipe_used[slot], 0));
        }
        SW_CUDA(cudaMemcpyAsync(choices, c.pipe_ch[slot], sizeof(sw_choice) * (size_t)B,
                                cudaMemcpyDeviceToHost, c.pipe_out));
        SW_CUDA(cudaEventRecord(c.pipe_done[slot], c.pipe_out));
        *ticket = c.pipe_seq++;
        return SW_OK;
    });
}

int sw_warmstart_host_wait(sw_ctx* ctx, int64_t ticket) {
    return guarded([&] {
        SW_REQUIRE(ctx, "null argument");
        Ctx& c = ctx->c;
        cudaEvent_t e;
        {
            std::lock_guard<std::mutex> pl(c.pipe_mu);
            SW_REQUIRE(ticket >= 0 && ticket < c.pipe_seq, "unknown ticket");
            // a slot's event is re-recorded by later submissions; waiting on the newer record
            // also covers the older batch (pipe_out runs the D2H copies in submission order)
            e = c.pipe_done[ticket % Ctx::kPipe];
        }
        SW_CUDA(cudaEventSynchronize(e));
        return SW_OK;
    });
}

int sw_warmstart_async(sw_ctx* ctx, const float* d_q, const sw_request* d_req, int32_t B,
                       uint64_t seed, const sw_selector_config* sel, const sw_policy* pol,
                       const float* d_eps, uint64_t philox_seed, sw_choice* d_ch, float* d_out,
                       int32_t t_out_max, void* stream) {
    return guarded([&] {
        SW_REQUIRE(ctx && (B == 0 || (d_q && d_req && d_ch && d_out)), "null argument");
        Ctx& c = ctx->c;
        std::shared_lock<std::shared_mutex> rd(c.mu);
        std::unique_lock<std::mutex> sc(c.scratch_mu);
        SW_CUDA(cudaSetDevice(c.device));
        cudaStream_t S = as_stream(stream);
        c.last_kernels = warmstart_async_impl(c, d_q, d_req, B, seed, sel, pol, d_eps,
                                              philox_seed, d_ch, d_out, t_out_max, S);
        return SW_OK;
    });
}

int sw_join(sw_ctx* ctx, void* stream) {
    return guarded([&] {
        SW_REQUIRE(ctx, "null argument");
        Ctx& c = ctx->c;
        std::unique_lock<std::mutex> sc(c.scratch_mu);
        SW_CUDA(cudaSetDevice(c.device));
        if (c.async_st) {
            SW_CUDA(cudaEventRecord(c.async_join_ev, c.async_st));
            SW_CUDA(cudaStreamWaitEvent(as_stream(stream), c.async_join_ev, 0));
        }
        return SW_OK;
    });
}

int sw_warmstart_host(sw_ctx* ctx, const float* q, const sw_request* reqs, int32_t B,
                      uint64_t seed, const sw_selector_config* sel, const sw_policy* pol,
                      uint64_t philox_seed, sw_choice* choices, float* d_out, int32_t t_out_max,
                      void* stream) {
    return guarded([&] {
        SW_REQUIRE(ctx && (B == 0 || (q && reqs && choices && d_out)), "null argument");
        Ctx& c = ctx->c;
        SW_REQUIRE(B <= c.Bmax, "batch exceeds the context's max_batch");
        HotGuard lk(c, as_stream(stream));
        SW_CUDA(cudaSetDevice(c.device));
        cudaStream_t st = as_stream(stream);
        SW_CUDA(cudaMemcpyAsync(c.d_q_stage, q, sizeof(float) * (size_t)B * c.D,
                                cudaMemcpyHostToDevice, st));
        SW_CUDA(cudaMemcpyAsync(c.d_req_stage, reqs, sizeof(sw_request) * (size_t)B,
                                cudaMemcpyHostToDevice, st));
        int kn = plan_impl(c, c.d_q_stage, c.d_req_stage, B, seed, sel, pol, c.d_choice_stage, st);
        kn += launch_align_noise(c, c.d_choice_stage, c.d_req_stage, B, -1, nullptr, philox_seed,
                                 d_out, t_out_max, st);
        SW_CUDA(cudaMemcpyAsync(choices, c.d_choice_stage, sizeof(sw_choice) * (size_t)B,
                                cudaMemcpyDeviceToHost, st));
        SW_CUDA(cudaStreamSynchronize(st));
        c.last_kernels = kn;
        return SW_OK;
    });
}

int sw_local_topk(sw_ctx* ctx, const float* d_q, int32_t B, int32_t k, int32_t rank,
                  void* d_records, int32_t* d_n, void* stream) {
    return guarded([&] {
        SW_REQUIRE(ctx && (B == 0 || (d_q && d_records && d_n)), "null argument");
        SW_REQUIRE(k >= 1 && k <= kMaxTopK, "k must be in [1, 32]");
        Ctx& c = ctx->c;
        HotGuard lk(c, as_stream(stream));
        SW_CUDA(cudaSetDevice(c.device));
        cudaStream_t st = as_stream(stream);
        int kn = launch_search(c, d_q, B, k, rank, st);
        // compact [B][32] records to [B][k]
        SW_CUDA(cudaMemcpy2DAsync(d_records, sizeof(HitRec) * k, c.hits, sizeof(HitRec) * kMaxTopK,
                                  sizeof(HitRec) * k, B, cudaMemcpyDeviceToDevice, st));
        SW_CUDA(cudaMemcpyAsync(d_n, c.nhits, sizeof(int32_t) * B, cudaMemcpyDeviceToDevice, st));
        c.last_kernels = kn;
        return SW_OK;
    });
}

// Sharded step, pipelined like sw_warmstart_async: prep + scoring on `stream`, the finish (local
// exact top-k, no select) and the record copies on the context's async stream, whose handle
// sw_async_stream returns — the caller enqueues the gather, sw_merge_select and
// sw_align_noise_owned there, and they overlap the next batch's scoring.
int sw_local_topk_async(sw_ctx* ctx, const float* d_q, int32_t B, int32_t k, int32_t rank,
                        void* d_records, int32_t* d_n, void* stream) {
    return guarded([&] {
        SW_REQUIRE(ctx && (B == 0 || (d_q && d_records && d_n)), "null argument");
        SW_REQUIRE(k >= 1 && k <= kMaxTopK, "k must be in [1, 32]");
        Ctx& c = ctx->c;
        std::shared_lock<std::shared_mutex> rd(c.mu);
        std::unique_lock<std::mutex> sc(c.scratch_mu);
        SW_CUDA(cudaSetDevice(c.device));
        cudaStream_t S = as_stream(stream);
        ensure_async(c);
        const int par = c.async_par;
        if (c.async_used[par]) SW_CUDA(cudaStreamWaitEvent(S, c.async_done[par], 0));
        if (c.async_used[par ^ 1]) SW_CUDA(cudaStreamWaitEvent(S, c.async_score_ev, 0));
        if (!c.last_user_async && c.scratch_ev) SW_CUDA(cudaStreamWaitEvent(S, c.scratch_ev, 0));
        set_par(c, par);
        const int kn = launch_search_fused(c, d_q, B, k, rank, nullptr, nullptr, nullptr, S,
                                           c.async_st);
        SW_CUDA(cudaMemcpy2DAsync(d_records, sizeof(HitRec) * k, c.hits, sizeof(HitRec) * kMaxTopK,
                                  sizeof(HitRec) * k, B, cudaMemcpyDeviceToDevice, c.async_st));
        SW_CUDA(cudaMemcpyAsync(d_n, c.nhits, sizeof(int32_t) * B, cudaMemcpyDeviceToDevice,
                                c.async_st));
        SW_CUDA(cudaEventRecord(c.async_done[par], c.async_st));
        if (c.scratch_ev) SW_CUDA(cudaEventRecord(c.scratch_ev, c.async_st));
        c.async_used[par] = true;
        c.async_par = par ^ 1;
        c.last_user_async = true;
        c.last_kernels = kn;
        return SW_OK;
    });
}

int sw_async_stream(sw_ctx* ctx, void** stream) {
    return guarded([&] {
        SW_REQUIRE(ctx && stream, "null argument");
        Ctx& c = ctx->c;
        std::unique_lock<std::mutex> sc(c.scratch_mu);
        SW_CUDA(cudaSetDevice(c.device));
        ensure_async(c);
        *stream = reinterpret_cast<void*>(c.async_st);
        return SW_OK;
    });
}

int sw_merge_select(sw_ctx* ctx, const void* d_gathered, const int32_t* d_gn, int32_t world,
                    const float* d_q, const sw_request* d_req, int32_t B, int32_t k,
                    uint64_t seed, const sw_selector_config* sel, const sw_policy* pol,
                    sw_choice* d_out, void* stream) {
    return guarded([&] {
        SW_REQUIRE(ctx && (B == 0 || (d_gathered && d_gn && d_req && d_out)), "null argument");
        check_sel(sel, pol);
        SW_REQUIRE(k == sel->top_k, "merge k must equal the selector top_k");
        Ctx& c = ctx->c;
        HotGuard lk(c, as_stream(stream));
        SW_CUDA(cudaSetDevice(c.device));
        cudaStream_t st = as_stream(stream);
        launch_merge(c, reinterpret_cast<const HitRec*>(d_gathered), d_gn, world, B, k, st);
        launch_select(c, c.hits, c.nhits, kMaxTopK, d_q, d_req, B, seed, *sel, *pol, d_out, 0, st);
        c.last_kernels = 2;
        return SW_OK;
    });
}

int sw_score_select_host(sw_ctx* ctx, int32_t n, const double* sims, const double* s_neg,
                         const double* durations, double L, const sw_selector_config* sel,
                         uint64_t rng_seed, double* scores_out, int32_t* pick) {
    return guarded([&] {
        SW_REQUIRE(ctx && sel && sims && s_neg && durations && scores_out && pick, "null argument");
        SW_REQUIRE(n >= 1, "score_candidates: empty candidate list");  // selector.cpp:28
        SW_REQUIRE(n <= kMaxTopK, "at most 32 candidates");
        SW_REQUIRE(L > 0.0, "requested duration must be positive");    // selector.cpp:29-31
        SW_REQUIRE(sel->temperature > 0.0, "selector temperature must be > 0");
        SW_REQUIRE(sel->quality_threshold >= 0.0 && sel->quality_threshold <= 1.0,
                   "selector quality threshold must be in [0, 1]");
        Ctx& c = ctx->c;
        SW_CUDA(cudaSetDevice(c.device));
        std::lock_guard<std::mutex> hl(c.host_mu);
        double* d_in = static_cast<double*>(host_stage(c, sizeof(double) * 8 * (size_t)n + 64));
        double* d_sc = d_in + 3 * n;
        int32_t* d_pick = reinterpret_cast<int32_t*>(d_in + 8 * n);
        cudaStream_t st = c.host_st;
        SW_CUDA(cudaMemcpyAsync(d_in, sims, sizeof(double) * n, cudaMemcpyHostToDevice, st));
        SW_CUDA(cudaMemcpyAsync(d_in + n, s_neg, sizeof(double) * n, cudaMemcpyHostToDevice, st));
        SW_CUDA(cudaMemcpyAsync(d_in + 2 * n, durations, sizeof(double) * n, cudaMemcpyHostToDevice, st));
        launch_score_select_one(c, n, d_in, d_in + n, d_in + 2 * n, L, *sel, rng_seed, d_sc,
                                d_pick, st);
        SW_CUDA(cudaMemcpyAsync(scores_out, d_sc, sizeof(double) * 5 * n, cudaMemcpyDeviceToHost, st));
        SW_CUDA(cudaMemcpyAsync(pick, d_pick, sizeof(int32_t) * 2, cudaMemcpyDeviceToHost, st));
        SW_CUDA(cudaStreamSynchronize(st));
        return SW_OK;
    });
}

int sw_score_candidates_host(sw_ctx* ctx, int32_t n, int32_t dim, const double* sims,
                             const float* audio, const double* durations, double L,
                             const float* negative, double* scores_out) {
    return guarded([&] {
        SW_REQUIRE(ctx && sims && audio && durations && scores_out, "null argument");
        SW_REQUIRE(n >= 1, "score_candidates: empty candidate list");  // selector.cpp:28
        SW_REQUIRE(n <= kMaxTopK, "at most 32 candidates");
        SW_REQUIRE(L > 0.0, "requested duration must be positive");    // selector.cpp:29-31
        SW_REQUIRE(dim >= 1, "dim must be >= 1");
        Ctx& c = ctx->c;
        SW_REQUIRE(negative || dim == c.D, "dot: dimension mismatch");
        SW_CUDA(cudaSetDevice(c.device));
        std::lock_guard<std::mutex> hl(c.host_mu);
        const size_t ab = sizeof(float) * (size_t)n * dim, nb = sizeof(float) * (size_t)dim;
        char* base = static_cast<char*>(host_stage(c, sizeof(double) * 7 * (size_t)n + ab + nb + 512));
        double* d_sims = reinterpret_cast<double*>(base);
        double* d_dur = d_sims + n;
        double* d_sc = d_dur + n;
        float* d_audio = reinterpret_cast<float*>(d_sc + 5 * n);
        float* d_neg = negative ? d_audio + (size_t)n * dim : c.neg;
        cudaStream_t st = c.host_st;
        SW_CUDA(cudaMemcpyAsync(d_sims, sims, sizeof(double) * n, cudaMemcpyHostToDevice, st));
        SW_CUDA(cudaMemcpyAsync(d_dur, durations, sizeof(double) * n, cudaMemcpyHostToDevice, st));
        SW_CUDA(cudaMemcpyAsync(d_audio, audio, ab, cudaMemcpyHostToDevice, st));
        if (negative) SW_CUDA(cudaMemcpyAsync(d_neg, negative, nb, cudaMemcpyHostToDevice, st));
        launch_score_candidates(n, dim, d_sims, d_audio, d_dur, d_neg, L, d_sc, st);
        SW_CUDA(cudaMemcpyAsync(scores_out, d_sc, sizeof(double) * 5 * n, cudaMemcpyDeviceToHost, st));
        SW_CUDA(cudaStreamSynchronize(st));
        return SW_OK;
    });
}

int sw_select_host(sw_ctx* ctx, int32_t n, const double* s_pos, const double* q,
                   double temperature, double threshold, double u, int32_t* pick,
                   uint32_t* flags) {
    return guarded([&] {
        SW_REQUIRE(ctx && s_pos && q && pick, "null argument");
        SW_REQUIRE(n >= 0 && n <= kMaxTopK, "at most 32 candidates");
        SW_REQUIRE(temperature > 0.0, "selector temperature must be > 0");  // selector.cpp:10
        SW_REQUIRE(threshold >= 0.0 && threshold <= 1.0,
                   "selector quality threshold must be in [0, 1]");
        Ctx& c = ctx->c;
        SW_CUDA(cudaSetDevice(c.device));
        std::lock_guard<std::mutex> hl(c.host_mu);
        double* d_in = static_cast<double*>(host_stage(c, sizeof(double) * (2 * (size_t)n + 2) + 64));
        int32_t* d_pick = reinterpret_cast<int32_t*>(d_in + 2 * n);
        cudaStream_t st = c.host_st;
        if (n > 0) {
            SW_CUDA(cudaMemcpyAsync(d_in, s_pos, sizeof(double) * n, cudaMemcpyHostToDevice, st));
            SW_CUDA(cudaMemcpyAsync(d_in + n, q, sizeof(double) * n, cudaMemcpyHostToDevice, st));
        }
        launch_select_draw(n, d_in, d_in + n, temperature, threshold, u, d_pick, st);
        int32_t h[2];
        SW_CUDA(cudaMemcpyAsync(h, d_pick, sizeof(h), cudaMemcpyDeviceToHost, st));
        SW_CUDA(cudaStreamSynchronize(st));
        *pick = h[0];
        if (flags) *flags = (uint32_t)h[1];
        return SW_OK;
    });
}

int sw_gater_host(sw_ctx* ctx, const float* prompts, const float* segs, const int32_t* T,
                  int32_t B, int32_t explore, double* phi_out, int32_t* arm_out) {
    return guarded([&] {
        SW_REQUIRE(ctx && prompts && segs && T && phi_out && arm_out, "null argument");
        Ctx& c = ctx->c;
        std::shared_lock lk(c.mu);
        SW_CUDA(cudaSetDevice(c.device));
        if (B <= 0) return SW_OK;
        std::lock_guard<std::mutex> hl(c.host_mu);
        const size_t fb = sizeof(float) * (size_t)B * c.D;
        char* base = static_cast<char*>(
            host_stage(c, 2 * fb + sizeof(double) * (size_t)B * kFeatureDim + 8 * (size_t)B + 1024));
        float* d_p = reinterpret_cast<float*>(base);
        float* d_s = reinterpret_cast<float*>(base + fb);
        double* d_phi = reinterpret_cast<double*>(base + (2 * fb + 255) / 256 * 256);
        int32_t* d_T = reinterpret_cast<int32_t*>(d_phi + (size_t)B * kFeatureDim);
        int32_t* d_arm = d_T + B;
        cudaStream_t st = c.host_st;
        SW_CUDA(cudaMemcpyAsync(d_p, prompts, fb, cudaMemcpyHostToDevice, st));
        SW_CUDA(cudaMemcpyAsync(d_s, segs, fb, cudaMemcpyHostToDevice, st));
        SW_CUDA(cudaMemcpyAsync(d_T, T, sizeof(int32_t) * B, cudaMemcpyHostToDevice, st));
        launch_gater(c, d_p, d_s, d_T, B, explore, d_phi, d_arm, st);
        SW_CUDA(cudaMemcpyAsync(phi_out, d_phi, sizeof(double) * B * kFeatureDim,
                                cudaMemcpyDeviceToHost, st));
        SW_CUDA(cudaMemcpyAsync(arm_out, d_arm, sizeof(int32_t) * B, cudaMemcpyDeviceToHost, st));
        SW_CUDA(cudaStreamSynchronize(st));
        return SW_OK;
    });
}

int sw_profile_enable(sw_ctx* ctx, int32_t on) {
    return guarded([&] {
        SW_REQUIRE(ctx, "null argument");
        ctx->c.prof = on != 0;
        // on = SW_PROFILE_MASK | stage bits: time only those stages (fewer events in a loop)
        ctx->c.prof_mask = (on & SW_PROFILE_MASK) ? (uint32_t)(on & 0xFF) : 0xFFu;
        return SW_OK;
    });
}

static void prof_collect(Ctx& c) {
    for (size_t i = 0; i < c.prof_used; ++i) {
        SW_CUDA(cudaEventSynchronize(c.prof_ev[2 * i + 1]));
        float ms = 0.0f;
        SW_CUDA(cudaEventElapsedTime(&ms, c.prof_ev[2 * i], c.prof_ev[2 * i + 1]));
        c.prof_ms[c.prof_stage[i]] += ms;
        c.prof_n[c.prof_stage[i]] += 1;
    }
    c.prof_used = 0;
}

int sw_profile_reset(sw_ctx* ctx) {
    return guarded([&] {
        SW_REQUIRE(ctx, "null argument");
        Ctx& c = ctx->c;
        SW_CUDA(cudaSetDevice(c.device));
        prof_collect(c);
        for (int s = 0; s < SW_NUM_STAGES; ++s) {
            c.prof_ms[s] = 0.0;
            c.prof_n[s] = 0;
        }
        return SW_OK;
    });
}

int sw_profile_read(sw_ctx* ctx, int32_t stage, double* total_ms, int64_t* launches) {
    return guarded([&] {
        SW_REQUIRE(ctx && stage >= 0 && stage < SW_NUM_STAGES, "bad argument");
        Ctx& c = ctx->c;
        SW_CUDA(cudaSetDevice(c.device));
        prof_collect(c);
        if (total_ms) *total_ms = c.prof_ms[stage];
        if (launches) *launches = c.prof_n[stage];
        return SW_OK;
    });
}

int sw_debug_query_stats(sw_ctx* ctx, int32_t B, int32_t* stats) {
    return guarded([&] {
        SW_REQUIRE(ctx && stats && B >= 0 && B <= ctx->c.Bmax, "bad argument");
        SW_CUDA(cudaSetDevice(ctx->c.device));
        SW_CUDA(cudaDeviceSynchronize());
        SW_CUDA(cudaMemcpy(stats, ctx->c.dbg, sizeof(int32_t) * 8 * B, cudaMemcpyDeviceToHost));
        return SW_OK;
    });
}

int sw_choice_rows(sw_ctx* ctx, const sw_choice* d_ch, int32_t B, float* d_rows, void* stream) {
    return guarded([&] {
        SW_REQUIRE(ctx && (B == 0 || (d_ch && d_rows)), "null argument");
        Ctx& c = ctx->c;
        HotGuard lk(c, as_stream(stream));
        launch_choice_rows(c, d_ch, B, d_rows, as_stream(stream));
        return SW_OK;
    });
}

int sw_overflow_stats(sw_ctx* ctx, int64_t* fallback_queries) {
    return guarded([&] {
        SW_REQUIRE(ctx && fallback_queries, "null argument");
        Ctx& c = ctx->c;
        SW_CUDA(cudaSetDevice(c.device));
        SW_CUDA(cudaDeviceSynchronize());
        unsigned long long v = 0;
        SW_CUDA(cudaMemcpy(&v, c.ovf_state + 2, sizeof(v), cudaMemcpyDeviceToHost));
        *fallback_queries = (int64_t)v;
        return SW_OK;
    });
}

int sw_last_launch_info(const sw_ctx* ctx, int32_t* kernels, int32_t* used_tc, int32_t* cand_max) {
    if (!ctx) return SW_EINVAL;
    if (kernels) *kernels = ctx->c.last_kernels;
    if (used_tc) *used_tc = ctx->c.last_tc;
    if (cand_max) *cand_max = ctx->c.last_cand_max;
    return SW_OK;
}

}  // extern "C"
