// Cache Manager trace replay with batched lookups — BASELINE config 5 ("1K-capacity
// quality-aware evict/refine churn interleaved with batched lookups").
//
// The reference replays a trace one request at a time (Pipeline::replay, pipeline.cpp:299-323):
// handle_request plans the request against the cache (search -> gate -> select -> gater -> t*),
// runs the simulated backend, records the reuse, admits the output (evicting past capacity),
// then run_maintenance refines entries whose recent reuses skipped too little. swr_replay keeps
// that loop and its decisions but plans `batch` consecutive requests in ONE device call (sw_plan
// over the snapshot the cache holds when the batch starts), then applies their
// mutations and the maintenance pass in request order. batch = 1 is the reference's replay
// exactly (tests check it against the unmodified Pipeline::replay).
//
// The simulated backend (generate, simgen.cpp:62-115) is the workload driver here, restated on
// the host: quality model, the output embedding normalize((1 - w) prompt + w reference) with
// w = 0.2 skip, and the nfe cost. Its latent payload is not produced (it never reaches a
// ServeOutcome field). The trace generator synth_workload (simgen.cpp:162-194) is
// restated bit-exactly (swr_synth_workload).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#include <cuda_runtime.h>

#include "host_policy.hpp"

using swh::HostRng;

namespace {

double clamp01(double v) { return std::min(1.0, std::max(0.0, v)); }

double expected_quality(const swr_config& c, double skip, double sigma) {  // simgen.cpp:11-16
    const double sigma_pos = std::max(0.0, sigma);
    const double excess = std::max(0.0, skip - c.skip_headroom * sigma_pos);
    const double q = c.q_max - c.penalty_slope * excess * excess;
    return std::min(1.0, std::max(0.0, q));
}

double cosine(const float* a, const float* b, int d) {  // core.cpp:26-37
    double s = 0.0;
    for (int i = 0; i < d; ++i) s += static_cast<double>(a[i]) * static_cast<double>(b[i]);
    return std::min(1.0, std::max(-1.0, s));
}

struct GenOut {
    std::vector<float> emb;
    double quality = 0.0, nfe = 0.0;
    int steps = 0;
};

// generate (simgen.cpp:62-115) without the latent payload. ref: the warm-start reference's
// embedding (the matched segment row), or nullptr for a cold run.
GenOut generate(const swr_config& c, const float* prompt, int dim, double L, int T, double skip,
                const float* ref, uint64_t seed) {
    if (!(L > 0.0)) throw std::invalid_argument("generate: duration must be positive");
    if (T < 1) throw std::invalid_argument("generate: total_steps must be >= 1");
    if (skip < 0.0 || skip > 0.65 + 1e-9)
        throw std::invalid_argument("generate: skip fraction outside the arm range");
    const int skipped = (int)std::llround(skip * T);
    GenOut g;
    g.steps = T - skipped;
    HostRng rng(swh::derive_seed(seed, 0x51554cULL));  // quality noise stream
    const double noise = c.noise_scale * rng.normal();
    if (skip == 0.0) {
        g.quality = std::min(1.0, std::max(0.0, c.q_max - std::fabs(noise)));
    } else {
        const double sigma = ref ? cosine(prompt, ref, dim) : 0.0;
        g.quality = std::min(1.0, std::max(0.0, expected_quality(c, skip, sigma) + noise));
    }
    const double w = 0.2 * skip;
    if (ref && w > 0.0) {
        std::vector<float> mix((size_t)dim);
        for (int i = 0; i < dim; ++i)
            mix[(size_t)i] = static_cast<float>((1.0 - w) * prompt[i] + w * ref[i]);
        g.emb = swh::normalize(mix);
    } else {
        g.emb = swh::normalize(std::vector<float>(prompt, prompt + dim));
    }
    g.nfe = g.steps * (c.step_time_s_per_10s * (L / 10.0));
    return g;
}

struct RegenCtx {
    const swr_config* cfg;
};

// RegenerateFn of run_maintenance (pipeline.cpp:286-291): a cold full-step generation
int regen_cb(void* user, const float* prompt, int32_t dim, double duration_s, uint64_t seed,
             float* emb_out, double* quality_out, float*, int32_t* t_src_out) {
    const RegenCtx* r = static_cast<const RegenCtx*>(user);
    if (!prompt) return SW_EINVAL;
    GenOut g = generate(*r->cfg, prompt, dim, duration_s, r->cfg->default_total_steps, 0.0,
                        nullptr, seed);
    std::memcpy(emb_out, g.emb.data(), sizeof(float) * dim);
    *quality_out = g.quality;
    *t_src_out = 0;
    return SW_OK;
}

#define CU(x)                                                                            \
    do {                                                                                 \
        cudaError_t e_ = (x);                                                            \
        if (e_ != cudaSuccess) throw std::runtime_error(std::string(#x) + ": " +         \
                                                        cudaGetErrorString(e_));         \
    } while (0)

struct DevBufs {
    float* q = nullptr;
    sw_request* r = nullptr;
    sw_choice* ch = nullptr;
    float* rows = nullptr;
    cudaStream_t st = nullptr;
    ~DevBufs() {
        cudaFree(q);
        cudaFree(r);
        cudaFree(ch);
        cudaFree(rows);
        if (st) cudaStreamDestroy(st);
    }
};

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

}  // namespace

extern "C" {

int sw_negative_embedding(int32_t dim, float* out) {  // make_negative_embedding (selector.cpp:16-20)
    if (dim < 1 || !out) return SW_EINVAL;
    HostRng rng(swh::derive_seed(0x4e454741ULL, (uint64_t)dim));
    const std::vector<float> v = swh::random_unit_vector((size_t)dim, rng);
    std::memcpy(out, v.data(), sizeof(float) * dim);
    return SW_OK;
}

int swr_synth_workload(const swr_workload* w, uint64_t seed, float* prompts, double* durations,
                       double* arrivals, int32_t* total_steps) {  // simgen.cpp:162-194
    if (!w || !prompts || !durations || !arrivals || !total_steps) return SW_EINVAL;
    if (w->near_duplicate_rate < 0.0 || w->near_duplicate_rate > 1.0) return SW_EINVAL;
    if (w->cluster_count < 1 || w->dim < 1 || w->n_prompts < 0) return SW_EINVAL;
    const size_t D = (size_t)w->dim;
    HostRng rng(seed);
    std::vector<std::vector<float>> centers((size_t)w->cluster_count);
    for (auto& c : centers) c = swh::random_unit_vector(D, rng);
    double clock = 0.0;
    for (int64_t i = 0; i < w->n_prompts; ++i) {
        const bool dup = i > 0 && rng.uniform() < w->near_duplicate_rate;
        std::vector<float> p;
        if (dup) {
            const uint64_t j = rng.uniform_int((uint64_t)i);
            p = swh::perturb(std::vector<float>(prompts + j * D, prompts + (j + 1) * D),
                             w->duplicate_perturbation, rng);
        } else {
            p = swh::perturb(centers[(size_t)(i % w->cluster_count)], w->cluster_perturbation, rng);
        }
        std::memcpy(prompts + (size_t)i * D, p.data(), sizeof(float) * D);
        durations[i] = rng.uniform(w->duration_lo_s, w->duration_hi_s);
        clock += rng.exponential(w->arrival_rate_hz);
        arrivals[i] = clock;
        total_steps[i] = w->total_steps;
    }
    return SW_OK;
}

int swr_replay(sw_ctx* ctx, swcm_cache* cm, const swr_config* cfg, int64_t n, const float* prompts,
               const double* durations, const double* arrivals, const int32_t* steps,
               swr_outcome* out, swr_stats* stats) {
    if (!ctx || !cm || !cfg || (n > 0 && (!prompts || !durations || !arrivals || !steps || !out)))
        return SW_EINVAL;
    if (cfg->batch < 1) return SW_EINVAL;
    try {
        int32_t dim = 0, max_batch = 0, device = 0;
        int rc = sw_ctx_info(ctx, &dim, nullptr, nullptr, nullptr, &max_batch, &device);
        if (rc < 0) return rc;
        if (dim != cm->dim) return SW_EINVAL;
        const int Bm = std::min<int>(cfg->batch, max_batch);
        CU(cudaSetDevice(device));
        DevBufs d;
        CU(cudaStreamCreateWithFlags(&d.st, cudaStreamNonBlocking));
        CU(cudaMalloc(&d.q, sizeof(float) * (size_t)Bm * dim));
        CU(cudaMalloc(&d.r, sizeof(sw_request) * (size_t)Bm));
        CU(cudaMalloc(&d.ch, sizeof(sw_choice) * (size_t)Bm));
        CU(cudaMalloc(&d.rows, sizeof(float) * (size_t)Bm * dim));
        std::vector<sw_request> hr((size_t)Bm);
        std::vector<sw_choice> hc((size_t)Bm);
        std::vector<float> hrows((size_t)Bm * dim);
        std::vector<uint8_t> fb((size_t)Bm);
        HostRng maint(swh::derive_seed(cfg->seed, 0x4d41494eULL));  // pipeline.cpp:70
        RegenCtx rg{cfg};
        swr_stats st{};
        double prev_arrival = 0.0, busy_until = 0.0;
        std::vector<double> lat;
        lat.reserve((size_t)n);
        double q_sum = 0.0, r_sum = 0.0, hits = 0.0;
        const double t_start = now_s();
        for (int64_t b0 = 0; b0 < n; b0 += Bm) {
            const int bn = (int)std::min<int64_t>(Bm, n - b0);
            // ---- batched lookups against the current cache snapshot
            const double t0 = now_s();
            for (int i = 0; i < bn; ++i) {
                const int64_t g = b0 + i;
                if (!(durations[g] > 0.0)) throw std::invalid_argument("request duration must be positive");
                if (steps[g] < 1) throw std::invalid_argument("request step budget must be >= 1");
                hr[(size_t)i] = sw_request{(uint64_t)(g + 1), durations[g], steps[g], 0};
            }
            CU(cudaMemcpyAsync(d.q, prompts + (size_t)b0 * dim, sizeof(float) * (size_t)bn * dim,
                               cudaMemcpyHostToDevice, d.st));
            CU(cudaMemcpyAsync(d.r, hr.data(), sizeof(sw_request) * bn, cudaMemcpyHostToDevice, d.st));
            rc = sw_plan(ctx, d.q, d.r, bn, cfg->seed, &cfg->selector, &cfg->policy, d.ch, d.st);
            if (rc < 0) return rc;
            rc = sw_choice_rows(ctx, d.ch, bn, d.rows, d.st);
            if (rc < 0) return rc;
            CU(cudaMemcpyAsync(hc.data(), d.ch, sizeof(sw_choice) * bn, cudaMemcpyDeviceToHost, d.st));
            CU(cudaMemcpyAsync(hrows.data(), d.rows, sizeof(float) * (size_t)bn * dim,
                               cudaMemcpyDeviceToHost, d.st));
            CU(cudaStreamSynchronize(d.st));
            // the retrieval stage's time_stretch (pipeline.cpp:164-169) runs at lookup time, on
            // the clip the cache held then: its hard bounds (vocoder.cpp:134-139) on the sliced
            // clip (slice_clip, simgen.cpp:113-128, over the entry's 200 Hz latent) send a
            // request to the cold fallback (pipeline.cpp:218-223)
            for (int i = 0; i < bn; ++i) {
                const sw_choice& c = hc[(size_t)i];
                fb[(size_t)i] = 0;
                if (!c.hit) continue;
                auto it = cm->entries.find(c.entry_id);
                const double rate = (double)cfg->latent_rate;
                double in_s = 0.0;
                if (it != cm->entries.end()) {
                    const int64_t total = std::llround(it->second.duration_s * rate);
                    if (c.segment.level == 0) {
                        in_s = (double)total / rate;
                    } else {
                        int64_t lo = std::llround(c.segment.start_s * rate);
                        int64_t hi = std::llround((c.segment.start_s + c.segment.length_s) * rate);
                        lo = std::min(lo, total);
                        hi = std::min(hi, total);
                        in_s = (double)(hi - lo) / rate;
                    }
                }
                const double r = in_s > 0.0 ? durations[b0 + i] / in_s : 0.0;
                fb[(size_t)i] = !(in_s > 0.0) || r < 0.4 || r > 2.5;
            }
            const double t1 = now_s();
            st.lookup_s += t1 - t0;
            st.batches += 1;
            st.lookups += bn;
            // ---- per request, in order: generate, record_reuse, admit (+ evict), maintenance
            for (int i = 0; i < bn; ++i) {
                const double tm0 = now_s();
                const int64_t g = b0 + i;
                const uint64_t id = (uint64_t)(g + 1);
                const float* prompt = prompts + (size_t)g * dim;
                const double L = durations[g];
                const int T = steps[g];
                if (arrivals[g] < prev_arrival)
                    throw std::runtime_error("trace arrival times must be monotone non-decreasing");
                prev_arrival = arrivals[g];
                const sw_choice& c = hc[(size_t)i];
                swr_outcome o{};
                o.request_id = id;
                const bool hit = c.hit != 0 && !fb[(size_t)i];
                int arm = c.arm;
                if (fb[(size_t)i]) {
                    o.fallback = 1;
                    arm = cfg->policy.kind == SW_POLICY_FIXED ? cfg->policy.fixed_arm : 0;
                }
                const double skip = 0.05 * arm;
                GenOut gen = generate(*cfg, prompt, dim, L, T, skip,
                                      hit ? hrows.data() + (size_t)i * dim : nullptr,
                                      swh::derive_seed(cfg->seed, id, 3));
                o.cache_hit = hit ? 1 : 0;
                o.entry_id = hit ? c.entry_id : 0;
                o.arm_index = arm;
                o.skip_fraction = skip;
                o.steps_skipped = T - gen.steps;
                o.quality = gen.quality;
                o.nfe_cost_s = gen.nfe;
                o.reference_similarity = hit ? c.similarity : 0.0;
                const double now_h = arrivals[g] / 3600.0;
                if (hit) {
                    // (an entry evicted since this batch's lookups: warn + no-op, cache.cpp:56-60)
                    rc = swcm_record_reuse(cm, c.entry_id, o.steps_skipped, L, now_h, skip);
                    if (rc < 0) return rc;
                    st.reuses += rc == SW_OK ? 1 : 0;
                }
                uint64_t adm = 0;
                rc = swcm_admit(cm, gen.emb.data(), L, prompt, gen.quality, now_h, nullptr, 0, &adm);
                if (rc < 0) return rc;
                if (rc == 1) {
                    o.admitted_entry_id = adm;
                    st.admits += 1;
                    st.evictions += (int64_t)cm->last_evicted.size();
                }
                const double start = std::max(arrivals[g], busy_until);
                const double finish = start + gen.nfe;
                busy_until = finish;
                o.sim_latency_s = finish - arrivals[g];
                st.total_nfe_s += gen.nfe;
                st.baseline_nfe_s += T * (cfg->step_time_s_per_10s * (L / 10.0));
                lat.push_back(o.sim_latency_s);
                q_sum += o.quality;
                r_sum += cfg->alpha * skip + (1.0 - cfg->alpha) * clamp01(o.quality);
                hits += hit ? 1.0 : 0.0;
                out[g] = o;
                const double tm1 = now_s();
                st.mutation_s += tm1 - tm0;
                // ---- run_maintenance (pipeline.cpp:280-297)
                if (cfg->refinement_enabled) {
                    const int nc = swcm_refinement_candidates(cm, nullptr, 0);
                    if (nc > 0) {
                        std::vector<uint64_t> cand((size_t)nc);
                        swcm_refinement_candidates(cm, cand.data(), nc);
                        for (uint64_t rid : cand) {
                            int32_t replaced = 0;
                            rc = cm->refine(rid, maint, &regen_cb, &rg, &replaced);
                            if (rc < 0) return rc;
                            st.refinements += 1;
                        }
                    }
                }
                st.maintenance_s += now_s() - tm1;
            }
        }
        st.total_s = now_s() - t_start;
        if (n > 0) {
            std::sort(lat.begin(), lat.end());
            auto pct = [&](double p) {
                const size_t idx = (size_t)std::ceil(p * (double)lat.size());
                return lat[std::min(lat.size() - 1, idx > 0 ? idx - 1 : 0)];
            };
            const double nn = (double)n;
            st.mean_quality = q_sum / nn;
            st.mean_reward = r_sum / nn;
            st.hit_rate = hits / nn;
            double ls = 0.0;
            for (double l : lat) ls += l;
            st.mean_latency_s = ls / nn;
            st.median_latency_s = pct(0.5);
            st.p95_latency_s = pct(0.95);
        }
        st.speedup = st.total_nfe_s > 0.0 ? st.baseline_nfe_s / st.total_nfe_s : 1.0;
        if (stats) *stats = st;
        return SW_OK;
    } catch (const std::invalid_argument& e) {
        return SW_EINVAL;
    } catch (const std::exception& e) {
        return SW_ERUNTIME;
    }
}

}  // extern "C"
