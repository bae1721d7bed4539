// Test infrastructure only (see oracle/Makefile): extern "C" shims that drive the UNMODIFIED
// reference implementation (/root/reference/proj/src, compiled in place) so Python tests and the
// bench's CPU-baseline leg can call it through ctypes. Nothing here re-implements the reference;
// every function forwards to the reference's own C++ API and copies values in/out.
//
// The per-request flow in ref_plan_batch mirrors Pipeline::plan_request + pick_arm
// (reference proj/src/pipeline.cpp:91-202) and the t* line of generate (simgen.cpp:70), with the
// cache's segment rows looked up from the caller-owned row buffer exactly as
// pipeline.cpp:113-131 looks them up through CacheManager::find.

#include <chrono>
#include <cmath>
#include <string>
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <optional>
#include <thread>
#include <vector>

#include "semwarm/cache.hpp"
#include "semwarm/core.hpp"
#include "semwarm/gater.hpp"
#include "semwarm/index.hpp"
#include "semwarm/vocoder.hpp"
#include "semwarm/selector.hpp"
#include "semwarm/simgen.hpp"
#include "semwarm/pipeline.hpp"

using namespace semwarm;

namespace {

struct EntryRows {
    const float* rows;  // caller-owned, n * dim floats, pyramid order (level-0 first)
    std::vector<PyramidDescriptor> segs;
};

struct RefIndex {
    IvfIndex idx;
    size_t dim = 0;
    std::map<uint64_t, EntryRows> entries;
};

EmbeddingVector vec(const float* p, size_t dim) {
    return EmbeddingVector(std::vector<float>(p, p + dim));
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------- core (core.cpp:58-124)
uint64_t ref_derive_seed(uint64_t base, uint64_t a, uint64_t b, uint64_t c) {
    return derive_seed(base, a, b, c);
}
uint64_t ref_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t ref_rng_first_u64(uint64_t seed) {
    Rng r(seed);
    return r.next_u64();
}
double ref_rng_first_uniform(uint64_t seed) {
    Rng r(seed);
    return r.uniform();
}
double ref_dot(const float* a, const float* b, int dim) { return dot(vec(a, dim), vec(b, dim)); }
double ref_cosine(const float* a, const float* b, int dim) {
    return cosine_similarity(vec(a, dim), vec(b, dim));
}
void ref_normalize(const float* raw, int dim, float* out) {
    EmbeddingVector v = normalize(std::vector<float>(raw, raw + dim));
    std::memcpy(out, v.values.data(), sizeof(float) * dim);
}
void ref_random_unit_vector(uint64_t seed, int dim, float* out) {
    Rng r(seed);
    EmbeddingVector v = random_unit_vector(dim, r);
    std::memcpy(out, v.values.data(), sizeof(float) * dim);
}
// n vectors from ONE sequential stream (as synth_workload draws its centres, simgen.cpp:169-170)
void ref_random_unit_vectors(uint64_t seed, int n, int dim, float* out) {
    Rng r(seed);
    for (int i = 0; i < n; ++i) {
        EmbeddingVector v = random_unit_vector(dim, r);
        std::memcpy(out + (size_t)i * dim, v.values.data(), sizeof(float) * dim);
    }
}
void ref_perturb(const float* v, int dim, double scale, uint64_t seed, float* out) {
    Rng r(seed);
    EmbeddingVector p = perturb(vec(v, dim), scale, r);
    std::memcpy(out, p.values.data(), sizeof(float) * dim);
}
void ref_make_negative(int dim, float* out) {
    EmbeddingVector v = make_negative_embedding(dim);
    std::memcpy(out, v.values.data(), sizeof(float) * dim);
}

// ---------------------------------------------------------------- pyramid (index.cpp:12-57)
int ref_pyramid_segments(double duration, double delta, int* levels, double* starts,
                         double* lengths, int cap) {
    auto segs = pyramid_segments(duration, delta);
    int n = (int)segs.size();
    for (int i = 0; i < n && i < cap; ++i) {
        levels[i] = segs[i].level;
        starts[i] = segs[i].start_s;
        lengths[i] = segs[i].length_s;
    }
    return n;
}
int ref_build_entry_vectors(uint64_t id, const float* full, int dim, double duration,
                            double delta, uint64_t seed_base, float* rows, int* levels,
                            double* starts, double* lengths, int cap) {
    auto v = build_entry_vectors(id, vec(full, dim), duration, delta, seed_base);
    int n = (int)v.size();
    for (int i = 0; i < n && i < cap; ++i) {
        std::memcpy(rows + (size_t)i * dim, v[i].embedding.values.data(), sizeof(float) * dim);
        levels[i] = v[i].segment.level;
        starts[i] = v[i].segment.start_s;
        lengths[i] = v[i].segment.length_s;
    }
    return n;
}

// ---------------------------------------------------------------- index (index.cpp:186-326)
void* ref_index_new(int dim) {
    auto* h = new RefIndex;
    h->dim = (size_t)dim;
    // exhaustive parity mode: a single list that is never re-clustered
    h->idx = IvfIndex::build({}, 1, 0, 1);
    h->idx.set_rebuild_interval(UINT64_MAX);
    return h;
}
void ref_index_free(void* p) { delete static_cast<RefIndex*>(p); }
// IVF mode exactly as CacheManager creates it (cache.cpp:17, pipeline.cpp:79-81):
// IvfIndex::build({}, C, seed, nprobe) + set_rebuild_interval.
void* ref_ivf_new(int dim, int centroids, uint64_t seed, int nprobe, uint64_t interval) {
    auto* h = new RefIndex;
    h->dim = (size_t)dim;
    h->idx = IvfIndex::build({}, (uint32_t)centroids, seed, (uint32_t)nprobe);
    h->idx.set_rebuild_interval(interval);
    return h;
}
// SWIX snapshot of the index (index.cpp:347-369): the only view of its centroids and lists.
int ref_index_save(void* p, const char* path) {
    try {
        static_cast<RefIndex*>(p)->idx.save(path);
    } catch (const std::exception&) {
        return -1;
    }
    return (int)static_cast<RefIndex*>(p)->idx.centroid_count();
}
void* ref_index_load(const char* path, int dim) {
    auto* h = new RefIndex;
    h->dim = (size_t)dim;
    try {
        h->idx = IvfIndex::load(path);
    } catch (const std::exception&) {
        delete h;
        return nullptr;
    }
    return h;
}
// IvfIndex::load(path) for the index, the caller's arena (kept alive) for candidate assembly:
// the CPU baseline of an IVF-mode cache whose lists were built elsewhere (a 1M-row k-means
// does not finish on the host in a bench run).
void* ref_index_new_loaded(const char* path, int dim, int n_entries, const uint64_t* ids,
                           const int64_t* off, const float* rows, const int* levels,
                           const double* starts, const double* lengths) {
    auto* h = static_cast<RefIndex*>(ref_index_load(path, dim));
    if (!h) return nullptr;
    for (int e = 0; e < n_entries; ++e) {
        EntryRows er;
        er.rows = rows + (size_t)off[e] * h->dim;
        for (int64_t r = off[e]; r < off[e + 1]; ++r)
            er.segs.push_back(PyramidDescriptor{levels[r], starts[r], lengths[r]});
        h->entries[ids[e]] = std::move(er);
    }
    return h;
}
// time_stretch (vocoder.cpp:128-207) of one 1-D clip; returns the output length, or -1 when
// the reference throws (empty clip, ratio outside [0.4, 2.5], bad config).
int ref_time_stretch(const float* in, int n, int rate, double target_s, int window, int hop,
                     float* out, int cap) {
    AudioClip c;
    c.samples.assign(in, in + n);
    c.sample_rate = rate;
    StftConfig cfg;
    cfg.window_size = window;
    cfg.analysis_hop = hop;
    try {
        AudioClip o = time_stretch(c, target_s, cfg);
        const int m = (int)o.samples.size();
        std::memcpy(out, o.samples.data(), sizeof(float) * (size_t)std::min(m, cap));
        return m;
    } catch (const std::exception&) {
        return -1;
    }
}
// synth_latent (simgen.cpp:19-50): the simulated backend's 1-D latent of an embedding.
int ref_synth_latent(const float* emb, int dim, double duration_s, int rate, float* out, int cap) {
    auto v = synth_latent(vec(emb, dim), duration_s, rate);
    std::memcpy(out, v.data(), sizeof(float) * (size_t)std::min<int>((int)v.size(), cap));
    return (int)v.size();
}
int ref_save_embeddings(const char* path, const float* v, int n, int dim) {
    std::vector<EmbeddingVector> vs;
    for (int i = 0; i < n; ++i) vs.push_back(vec(v + (size_t)i * dim, dim));
    try {
        save_embeddings(path, vs);
    } catch (const std::exception&) {
        return -1;
    }
    return 0;
}
int ref_index_check_consistent(void* p) {
    return static_cast<RefIndex*>(p)->idx.check_consistent() ? 1 : 0;
}

// Inserts n_entries entries; entry e owns rows [off[e], off[e+1]) of `rows` (caller keeps the
// buffer alive for the index lifetime: candidate assembly reads segment rows from it).
int ref_index_insert_many(void* p, int n_entries, const uint64_t* ids, const int64_t* off,
                          const float* rows, const int* levels, const double* starts,
                          const double* lengths) {
    auto* h = static_cast<RefIndex*>(p);
    try {
        for (int e = 0; e < n_entries; ++e) {
            std::vector<IndexedVector> vs;
            EntryRows er;
            er.rows = rows + (size_t)off[e] * h->dim;
            for (int64_t r = off[e]; r < off[e + 1]; ++r) {
                PyramidDescriptor d{levels[r], starts[r], lengths[r]};
                vs.push_back(IndexedVector{ids[e], d, vec(rows + (size_t)r * h->dim, h->dim)});
                er.segs.push_back(d);
            }
            h->idx.insert(std::move(vs));
            h->entries[ids[e]] = std::move(er);
        }
    } catch (const std::exception& ex) {
        return -1;
    }
    return 0;
}
void ref_index_remove(void* p, uint64_t id) {
    auto* h = static_cast<RefIndex*>(p);
    h->idx.remove(id);
    h->entries.erase(id);
}
int ref_index_search(void* p, const float* q, int k, uint64_t* ids, int* levels,
                     double* starts, double* lengths, double* sims) {
    auto* h = static_cast<RefIndex*>(p);
    auto hits = h->idx.search(vec(q, h->dim), (size_t)k);
    for (size_t i = 0; i < hits.size(); ++i) {
        ids[i] = hits[i].entry_id;
        levels[i] = hits[i].segment.level;
        starts[i] = hits[i].segment.start_s;
        lengths[i] = hits[i].segment.length_s;
        sims[i] = hits[i].similarity;
    }
    return (int)hits.size();
}

// ---------------------------------------------------------------- selector (selector.cpp:24-85)
// Raw score_candidates + select over caller-assembled candidates.
int ref_score_select(int n, const uint64_t* ids, const int* levels, const double* starts,
                     const double* lengths, const double* sims, const float* audio, int dim,
                     const float* neg, const float* prompt, double L, int top_k, double temp,
                     double thr, uint64_t rng_seed, double* s_pos, double* s_neg, double* a,
                     double* b, double* q) {
    SelectorConfig cfg;
    cfg.top_k = (size_t)top_k;
    cfg.temperature = temp;
    cfg.quality_threshold = thr;
    cfg.negative_embedding = vec(neg, dim);
    std::vector<CandidateInput> in(n);
    for (int i = 0; i < n; ++i) {
        in[i].entry_id = ids[i];
        in[i].segment = PyramidDescriptor{levels[i], starts[i], lengths[i]};
        in[i].prompt_similarity = sims[i];
        in[i].audio_embedding = vec(audio + (size_t)i * dim, dim);
        in[i].duration_s = lengths[i];
    }
    auto sc = score_candidates(in, vec(prompt, dim), L, cfg);
    for (int i = 0; i < n; ++i) {
        s_pos[i] = sc[i].s_pos;
        s_neg[i] = sc[i].s_neg;
        a[i] = sc[i].a;
        b[i] = sc[i].b;
        q[i] = sc[i].q;
    }
    Rng rng(rng_seed);
    auto pick = select(sc, cfg, rng);
    return pick ? (int)*pick : -1;
}

// ---------------------------------------------------------------- gater (gater.cpp:13-92)
void ref_context_features(const float* prompt, const float* cache, int dim, int T, double* phi) {
    BanditContext ctx{vec(prompt, dim), vec(cache, dim), T};
    auto f = context_features(ctx);
    for (size_t i = 0; i < f.size(); ++i) phi[i] = f[i];
}
int ref_choose_arm(const float* theta, const float* psi, int fd, double beta, const double* phi,
                   int explore) {
    BanditModel m = BanditModel::zeros((size_t)fd);
    std::memcpy(m.theta.data(), theta, sizeof(float) * kNumArms * fd);
    std::memcpy(m.psi.data(), psi, sizeof(float) * kNumArms * fd);
    m.beta = beta;
    std::vector<double> f(phi, phi + fd);
    return choose_arm(m, f, explore ? GaterMode::kExplore : GaterMode::kExploit);
}
double ref_arm_skip_fraction(int arm) { return arm_skip_fraction(arm); }

// ---------------------------------------------------------------- the warm-start plan
// Per request: search (index.cpp:289) -> candidate assembly (pipeline.cpp:113-131) ->
// score_candidates + select (pipeline.cpp:134-141) -> seg-emb lookup + similarity + features
// (pipeline.cpp:150-175) -> pick_arm (pipeline.cpp:180-202; a miss under the fixed policy keeps the
// fixed arm, pipeline.cpp:229-231) -> t* = llround(skip * T) (simgen.cpp:70).
// policy: 0 exploit, 1 explore, 2 rule, 3 fixed. The vocoder stretch (pipeline.cpp:164-169) is
// not run: its output never reaches any field computed here.
struct RefPlanOut {
    int32_t hit;
    int32_t arm;
    int32_t steps_skipped;
    int32_t n_hits;
    uint64_t entry_id;
    int32_t level;
    int32_t pick;
    double start_s;
    double length_s;
    double similarity;
};

static void plan_one(RefIndex* h, const SelectorConfig& cfg, const BanditModel& model, int policy,
                     double rule_thr, double rule_skip, int fixed_arm, const float* qp, double L,
                     uint64_t req_id, int T, uint64_t seed, RefPlanOut* out, uint64_t* hit_ids,
                     double* hit_sims) {
    std::memset(out, 0, sizeof(*out));
    out->pick = -1;
    EmbeddingVector q = vec(qp, h->dim);
    Rng selector_rng(derive_seed(seed, req_id, 2));
    auto hits = h->idx.search(q, cfg.top_k);
    out->n_hits = (int)hits.size();
    for (size_t i = 0; i < hits.size(); ++i) {
        if (hit_ids) hit_ids[i] = hits[i].entry_id;
        if (hit_sims) hit_sims[i] = hits[i].similarity;
    }
    bool hit = false;
    double similarity = 0.0;
    std::vector<double> features;
    if (!hits.empty()) {
        std::vector<CandidateInput> inputs;
        for (const auto& hh : hits) {
            auto it = h->entries.find(hh.entry_id);
            if (it == h->entries.end()) continue;
            CandidateInput in;
            in.entry_id = hh.entry_id;
            in.segment = hh.segment;
            in.prompt_similarity = hh.similarity;
            in.duration_s = hh.segment.length_s;
            const auto& er = it->second;
            for (size_t s = 0; s < er.segs.size(); ++s) {
                if (er.segs[s].level == hh.segment.level &&
                    std::fabs(er.segs[s].start_s - hh.segment.start_s) < 1e-9) {
                    in.audio_embedding = vec(er.rows + s * h->dim, h->dim);
                    break;
                }
            }
            if (in.audio_embedding.dim() == 0) continue;
            inputs.push_back(std::move(in));
        }
        if (!inputs.empty()) {
            auto scored = score_candidates(inputs, q, L, cfg);
            auto pick = select(scored, cfg, selector_rng);
            if (pick) {
                const auto& c = scored[*pick];
                const auto& er = h->entries.at(c.entry_id);
                EmbeddingVector seg_emb = vec(er.rows, h->dim);  // full embedding = level 0
                for (size_t s = 0; s < er.segs.size(); ++s) {
                    if (er.segs[s].level == c.segment.level &&
                        std::fabs(er.segs[s].start_s - c.segment.start_s) < 1e-9) {
                        seg_emb = vec(er.rows + s * h->dim, h->dim);
                        break;
                    }
                }
                hit = true;
                out->pick = (int)*pick;
                out->entry_id = c.entry_id;
                out->level = c.segment.level;
                out->start_s = c.segment.start_s;
                out->length_s = c.segment.length_s;
                similarity = cosine_similarity(q, seg_emb);
                features = context_features(BanditContext{q, seg_emb, T});
            }
        }
    }
    int arm = 0;
    if (hit) {
        switch (policy) {
            case 0: arm = choose_arm(model, features, GaterMode::kExploit); break;
            case 1: arm = choose_arm(model, features, GaterMode::kExplore); break;
            case 2:
                arm = similarity >= rule_thr ? (int)std::llround(rule_skip / 0.05) : 0;
                break;
            default: arm = fixed_arm; break;
        }
    } else if (policy == 3) {
        arm = fixed_arm;
    }
    double skip = arm_skip_fraction(arm);
    out->hit = hit ? 1 : 0;
    out->arm = arm;
    out->steps_skipped = (int)std::llround(skip * T);
    out->similarity = similarity;
}

int ref_plan_batch(void* p, const float* neg, int B, const float* queries, const double* L,
                   const uint64_t* req_ids, const int* T, uint64_t seed, int top_k, double temp,
                   double thr, int policy, const float* theta, const float* psi, int fd,
                   double beta, double rule_thr, double rule_skip, int fixed_arm, int nthreads,
                   RefPlanOut* out, uint64_t* hit_ids, double* hit_sims) {
    auto* h = static_cast<RefIndex*>(p);
    SelectorConfig cfg;
    cfg.top_k = (size_t)top_k;
    cfg.temperature = temp;
    cfg.quality_threshold = thr;
    cfg.negative_embedding = vec(neg, h->dim);
    BanditModel model = BanditModel::zeros((size_t)fd);
    if (theta) std::memcpy(model.theta.data(), theta, sizeof(float) * kNumArms * fd);
    if (psi) std::memcpy(model.psi.data(), psi, sizeof(float) * kNumArms * fd);
    model.beta = beta;
    auto work = [&](int lo, int hi) {
        for (int i = lo; i < hi; ++i) {
            plan_one(h, cfg, model, policy, rule_thr, rule_skip, fixed_arm,
                     queries + (size_t)i * h->dim, L[i], req_ids[i], T[i], seed, out + i,
                     hit_ids ? hit_ids + (size_t)i * top_k : nullptr,
                     hit_sims ? hit_sims + (size_t)i * top_k : nullptr);
        }
    };
    try {
        if (nthreads <= 1 || B <= 1) {
            work(0, B);
        } else {
            // disjoint query slices over one shared const index (reader model, pipeline.cpp:216)
            std::vector<std::thread> ts;
            int per = (B + nthreads - 1) / nthreads;
            for (int t = 0; t < nthreads; ++t) {
                int lo = t * per, hi = std::min(B, lo + per);
                if (lo >= hi) break;
                ts.emplace_back(work, lo, hi);
            }
            for (auto& t : ts) t.join();
        }
    } catch (const std::exception&) {
        return -1;
    }
    return 0;
}

// ---------------------------------------------------------------- cache manager (cache.cpp)
// Driven by the trace-replay parity test for the host-side Cache Manager policy.
struct RefCache {
    std::unique_ptr<CacheManager> cm;
};
void* ref_cache_new(uint64_t capacity, double decay, double grace, double floor_q, double delta,
                    uint64_t emb_seed) {
    CacheConfig c;
    c.capacity = capacity;
    c.decay_per_hour = decay;
    c.grace_hours = grace;
    c.quality_floor = floor_q;
    c.pyramid_delta = delta;
    c.embedding_seed = emb_seed;
    auto* r = new RefCache;
    r->cm = std::make_unique<CacheManager>(c, 1, 1, 0);
    r->cm->index().set_rebuild_interval(UINT64_MAX);
    return r;
}
// CacheManager in IVF mode exactly as Pipeline builds it (pipeline.cpp:79-81)
void* ref_cache_new_ivf(uint64_t capacity, double decay, double grace, double floor_q,
                        double delta, uint64_t emb_seed, int centroids, int nprobe,
                        uint64_t index_seed, uint64_t interval) {
    CacheConfig c;
    c.capacity = capacity;
    c.decay_per_hour = decay;
    c.grace_hours = grace;
    c.quality_floor = floor_q;
    c.pyramid_delta = delta;
    c.embedding_seed = emb_seed;
    auto* r = new RefCache;
    r->cm = std::make_unique<CacheManager>(c, (uint32_t)centroids, (uint32_t)nprobe, index_seed);
    r->cm->index().set_rebuild_interval(interval);
    return r;
}
void ref_cache_free(void* p) { delete static_cast<RefCache*>(p); }
int ref_cache_index_save(void* p, const char* path) {
    try {
        static_cast<RefCache*>(p)->cm->index().save(path);
    } catch (const std::exception&) {
        return -1;
    }
    return (int)static_cast<RefCache*>(p)->cm->index().centroid_count();
}
// admit a clip with the given embedding/duration (latent is irrelevant to every policy decision)
int64_t ref_cache_admit(void* p, const float* emb, int dim, double duration, double quality,
                        double now_h) {
    auto* r = static_cast<RefCache*>(p);
    SimClip clip;
    clip.duration_s = duration;
    clip.embedding = vec(emb, dim);
    auto id = r->cm->admit(std::move(clip), vec(emb, dim), quality, now_h);
    return id ? (int64_t)*id : -1;
}
void ref_cache_record_reuse(void* p, uint64_t id, int steps, double dur, double now_h,
                            double skip) {
    static_cast<RefCache*>(p)->cm->record_reuse(id, steps, dur, now_h, skip);
}
int ref_cache_evict(void* p, double now_h, uint64_t* out, int cap) {
    auto ev = static_cast<RefCache*>(p)->cm->evict_if_full(now_h);
    for (size_t i = 0; i < ev.size() && (int)i < cap; ++i) out[i] = ev[i];
    return (int)ev.size();
}
double ref_cache_importance(void* p, uint64_t id, double now_h) {
    return static_cast<RefCache*>(p)->cm->current_importance(id, now_h);
}
int ref_cache_size(void* p) { return (int)static_cast<RefCache*>(p)->cm->size(); }
int ref_cache_ids(void* p, uint64_t* out, int cap) {
    int n = 0;
    for (const auto& [id, e] : static_cast<RefCache*>(p)->cm->entries()) {
        if (n < cap) out[n] = id;
        ++n;
    }
    return n;
}
int ref_cache_refinement_candidates(void* p, uint64_t* out, int cap) {
    auto c = static_cast<RefCache*>(p)->cm->refinement_candidates();
    for (size_t i = 0; i < c.size() && (int)i < cap; ++i) out[i] = c[i];
    return (int)c.size();
}
// refine with regenerations whose (quality, embedding) come from the caller, in call order
struct RefRegen {
    const double* qualities;
    const float* embs;
    int dim;
    int n;
    int used;
};
int ref_cache_refine(void* p, uint64_t id, uint64_t rng_seed, const double* qualities,
                     const float* embs, int dim, int n, uint64_t* seeds_out) {
    auto* r = static_cast<RefCache*>(p);
    RefRegen rg{qualities, embs, dim, n, 0};
    Rng rng(rng_seed);
    RegenerateFn fn = [&](const EmbeddingVector&, double d, uint64_t seed) {
        if (seeds_out && rg.used < rg.n) seeds_out[rg.used] = seed;
        int i = rg.used < rg.n ? rg.used : rg.n - 1;
        rg.used++;
        SimClip c;
        c.duration_s = d;
        c.embedding = vec(rg.embs + (size_t)i * rg.dim, rg.dim);
        return std::make_pair(c, rg.qualities[i]);
    };
    return r->cm->refine(id, fn, rng) ? 1 : 0;
}
// search through the cache's own index (segment rows derived by the reference at admit time)
int ref_cache_search(void* p, const float* q, int dim, int k, uint64_t* ids, int* levels,
                     double* starts, double* lengths, double* sims) {
    auto* r = static_cast<RefCache*>(p);
    auto hits = r->cm->index().search(vec(q, dim), (size_t)k);
    for (size_t i = 0; i < hits.size(); ++i) {
        ids[i] = hits[i].entry_id;
        levels[i] = hits[i].segment.level;
        starts[i] = hits[i].segment.start_s;
        lengths[i] = hits[i].segment.length_s;
        sims[i] = hits[i].similarity;
    }
    return (int)hits.size();
}
// segment rows of one cached entry (pyramid order), as CacheManager::find exposes them
int ref_cache_entry_rows(void* p, uint64_t id, float* rows, int cap) {
    const CacheEntry* e = static_cast<RefCache*>(p)->cm->find(id);
    if (!e) return -1;
    int n = (int)e->segment_vectors.size();
    for (int i = 0; i < n && i < cap; ++i) {
        const auto& v = e->segment_vectors[i].embedding.values;
        std::memcpy(rows + (size_t)i * v.size(), v.data(), sizeof(float) * v.size());
    }
    return n;
}

// ---------------------------------------------------------------- snapshots (cache.cpp:211-295,
// gater.cpp:277-306): the reference's own directory snapshot and model file, for the
// interchange tests of the device-arena loaders
int ref_cache_save_snapshot(void* p, const char* dir) {
    try {
        static_cast<RefCache*>(p)->cm->save_snapshot(dir);
    } catch (const std::exception&) {
        return -1;
    }
    return 0;
}
int ref_cache_load_snapshot(void* p, const char* dir) {
    try {
        static_cast<RefCache*>(p)->cm->load_snapshot(dir);
    } catch (const std::exception&) {
        return -1;
    }
    return 0;
}
int ref_cache_check_consistent(void* p) {
    return static_cast<RefCache*>(p)->cm->check_consistent() ? 1 : 0;
}
// admit with a full SimClip payload (latent series, rate, seed, skip fraction)
int64_t ref_cache_admit_clip(void* p, const float* emb, const float* prompt, int dim,
                             double duration, double quality, double now_h, const float* latent,
                             int n_latent, int rate, uint64_t seed, double skip) {
    auto* r = static_cast<RefCache*>(p);
    SimClip clip;
    clip.duration_s = duration;
    clip.embedding = vec(emb, dim);
    clip.latent.assign(latent, latent + n_latent);
    clip.latent_rate = rate;
    clip.seed = seed;
    clip.skip_fraction_used = skip;
    auto id = r->cm->admit(std::move(clip), vec(prompt, dim), quality, now_h);
    return id ? (int64_t)*id : -1;
}
// ledger state of one entry: importance, last_update_h, admitted_h, quality, duration_s,
// attempts, reuse_count, then the recent skips (returns their count)
int ref_cache_entry_state(void* p, uint64_t id, double* out, double* skips, int cap) {
    const CacheEntry* e = static_cast<RefCache*>(p)->cm->find(id);
    if (!e) return -1;
    out[0] = e->importance;
    out[1] = e->last_update_h;
    out[2] = e->admitted_h;
    out[3] = e->quality;
    out[4] = e->duration_s;
    out[5] = e->refinement_attempts;
    out[6] = (double)e->reuse_count;
    int n = 0;
    for (double s : e->recent_skips) {
        if (n < cap) skips[n] = s;
        ++n;
    }
    return n;
}
int ref_cache_clip(void* p, uint64_t id, float* latent, int cap, int* rate, uint64_t* seed,
                   double* skip, float* emb) {
    const CacheEntry* e = static_cast<RefCache*>(p)->cm->find(id);
    if (!e) return -1;
    const int n = (int)e->clip.latent.size();
    for (int i = 0; i < n && i < cap; ++i) latent[i] = e->clip.latent[i];
    *rate = e->clip.latent_rate;
    *seed = e->clip.seed;
    *skip = e->clip.skip_fraction_used;
    std::memcpy(emb, e->full_embedding.values.data(), sizeof(float) * e->full_embedding.values.size());
    return n;
}
int ref_bandit_save(const char* path, const float* theta, const float* psi, int fd) {
    BanditModel m = BanditModel::zeros((size_t)fd);
    std::memcpy(m.theta.data(), theta, sizeof(float) * m.theta.size());
    std::memcpy(m.psi.data(), psi, sizeof(float) * m.psi.size());
    try {
        m.save(path);
    } catch (const std::exception&) {
        return -1;
    }
    return 0;
}
int ref_bandit_load(const char* path, float* theta, float* psi, int cap) {
    try {
        BanditModel m = BanditModel::load(path);
        if ((int)m.theta.size() > cap) return -2;
        std::memcpy(theta, m.theta.data(), sizeof(float) * m.theta.size());
        std::memcpy(psi, m.psi.data(), sizeof(float) * m.psi.size());
        return (int)m.feature_dim;
    } catch (const std::exception&) {
        return -1;
    }
}

// ---------------------------------------------------------------- simgen quality (simgen.cpp:12-17)
double ref_expected_quality(double skip, double sigma) {
    QualityModel m;
    return m.expected_quality(skip, sigma);
}


// ---------------------------------------------------------------- trace replay (config 5)
// synth_workload (simgen.cpp:162-194) with the reference defaults, n prompts of `dim`.
int ref_synth_workload(int64_t n, int dim, uint64_t seed, float* prompts, double* dur,
                       double* arr, int32_t* steps) {
    WorkloadConfig wc;
    wc.n_prompts = (size_t)n;
    wc.dim = (size_t)dim;
    auto tr = synth_workload(wc, seed);
    for (size_t i = 0; i < tr.size(); ++i) {
        std::memcpy(prompts + i * dim, tr[i].prompt_embedding.values.data(), sizeof(float) * dim);
        dur[i] = tr[i].duration_s;
        arr[i] = tr[i].arrival_time_s;
        steps[i] = tr[i].total_steps;
    }
    return (int)tr.size();
}

struct RefReplayOut {  // swr_outcome's layout
    uint64_t request_id;
    int32_t cache_hit, arm_index, steps_skipped, fallback;
    uint64_t entry_id, admitted_entry_id;
    double quality, nfe_cost_s, sim_latency_s, skip_fraction, reference_similarity;
};

static PipelineConfig replay_cfg(int dim, uint64_t capacity, int policy, const float* theta,
                                 const float* psi, double beta, int fixed_arm, uint64_t seed) {
    ConfigMap cm;
    cm.set("dim", std::to_string(dim));
    cm.set("seed", std::to_string(seed));
    cm.set("cache.capacity", std::to_string(capacity));
    const char* pol[] = {"exploit", "explore", "rule", "fixed"};
    cm.set("gater.policy", pol[policy]);
    cm.set("fixed.arm", std::to_string(fixed_arm));
    PipelineConfig cfg = PipelineConfig::from_config(cm);
    if (theta) std::memcpy(cfg.gater.theta.data(), theta, sizeof(float) * kNumArms * kFeatureDim);
    if (psi) std::memcpy(cfg.gater.psi.data(), psi, sizeof(float) * kNumArms * kFeatureDim);
    cfg.gater.beta = beta;
    return cfg;
}

static void copy_out(const ServeOutcome& o, RefReplayOut* r) {
    std::memset(r, 0, sizeof(*r));
    r->request_id = o.request_id;
    r->cache_hit = o.cache_hit;
    r->arm_index = o.arm_index;
    r->steps_skipped = o.steps_skipped;
    r->fallback = o.fallback;
    r->entry_id = o.entry_id ? *o.entry_id : 0;
    r->admitted_entry_id = o.admitted_entry_id ? *o.admitted_entry_id : 0;
    r->quality = o.quality;
    r->nfe_cost_s = o.nfe_cost_s;
    r->sim_latency_s = o.sim_latency_s;
    r->skip_fraction = o.skip_fraction;
    r->reference_similarity = o.reference_similarity;
}

static std::vector<GenerationRequest> make_trace(int64_t n, int dim, const float* prompts,
                                                 const double* dur, const double* arr,
                                                 const int32_t* steps) {
    std::vector<GenerationRequest> tr((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        tr[i].id = (uint64_t)(i + 1);
        tr[i].prompt_embedding = vec(prompts + (size_t)i * dim, dim);
        tr[i].duration_s = dur[i];
        tr[i].arrival_time_s = arr[i];
        tr[i].total_steps = steps[i];
    }
    return tr;
}

// batch <= 0: the reference's own Pipeline::replay (pipeline.cpp:299-323), untouched.
// batch >= 1: the same decisions with the lookups of `batch` consecutive requests planned
// against the cache as it stands when the batch starts (plan_request, pipeline.cpp:91-178, incl.
// slice_clip + time_stretch), then per request: pick_arm, generate, record_reuse, admit and the
// maintenance pass (pipeline.cpp:180-297) — through the reference's public API on the
// Pipeline's own CacheManager. batch = 1 must equal batch <= 0 (tests check it).
int ref_replay(int64_t n, int dim, const float* prompts, const double* dur, const double* arr,
               const int32_t* steps, uint64_t capacity, int policy, const float* theta,
               const float* psi, double beta, int fixed_arm, uint64_t seed, int batch,
               RefReplayOut* out, double* summary /* [total_nfe, baseline, speedup, mean_q,
               mean_reward, hit_rate, mean_lat, median_lat, p95_lat, refinements] */,
               double* wall_s) {
    try {
        PipelineConfig cfg = replay_cfg(dim, capacity, policy, theta, psi, beta, fixed_arm, seed);
        auto trace = make_trace(n, dim, prompts, dur, arr, steps);
        Pipeline pipe(cfg);
        const auto t0 = std::chrono::steady_clock::now();
        RunReport rep;
        if (batch <= 0) {
            rep = pipe.replay(trace);
        } else {
            const PipelineConfig& pc = pipe.config();
            CacheManager& cache = pipe.cache();
            Rng maint(derive_seed(pc.seed, 0x4d41494eULL));
            double prev = 0.0, busy = 0.0;
            for (int64_t b0 = 0; b0 < n; b0 += batch) {
                const int64_t b1 = std::min<int64_t>(n, b0 + batch);
                struct Plan {
                    bool hit = false, fallback = false;
                    uint64_t entry_id = 0;
                    double similarity = 0.0;
                    std::optional<SimClip> reference;
                    std::vector<double> features;
                };
                std::vector<Plan> plans((size_t)(b1 - b0));
                for (int64_t g = b0; g < b1; ++g) {  // lookups against the frozen snapshot
                    const GenerationRequest& req = trace[(size_t)g];
                    Plan& pl = plans[(size_t)(g - b0)];
                    Rng sel_rng(derive_seed(pc.seed, req.id, 2));
                    try {
                        auto hits = cache.index().search(req.prompt_embedding, pc.selector.top_k);
                        std::optional<SearchHit> chosen;
                        std::vector<CandidateInput> inputs;
                        for (const auto& h : hits) {
                            const CacheEntry* e = cache.find(h.entry_id);
                            if (!e) continue;
                            CandidateInput in;
                            in.entry_id = h.entry_id;
                            in.segment = h.segment;
                            in.prompt_similarity = h.similarity;
                            in.duration_s = h.segment.length_s;
                            for (const auto& v : e->segment_vectors)
                                if (v.segment.level == h.segment.level &&
                                    std::fabs(v.segment.start_s - h.segment.start_s) < 1e-9) {
                                    in.audio_embedding = v.embedding;
                                    break;
                                }
                            if (in.audio_embedding.dim() == 0) continue;
                            inputs.push_back(std::move(in));
                        }
                        if (!inputs.empty()) {
                            auto scored = score_candidates(inputs, req.prompt_embedding,
                                                           req.duration_s, pc.selector);
                            auto pick = select(scored, pc.selector, sel_rng);
                            if (pick)
                                chosen = SearchHit{scored[*pick].entry_id, scored[*pick].segment,
                                                   scored[*pick].s_pos};
                        }
                        if (chosen) {
                            const CacheEntry* entry = cache.find(chosen->entry_id);
                            EmbeddingVector seg_emb = entry->full_embedding;
                            for (const auto& v : entry->segment_vectors)
                                if (v.segment.level == chosen->segment.level &&
                                    std::fabs(v.segment.start_s - chosen->segment.start_s) < 1e-9) {
                                    seg_emb = v.embedding;
                                    break;
                                }
                            SimClip ref = chosen->segment.level == 0
                                              ? entry->clip
                                              : slice_clip(entry->clip, chosen->segment.start_s,
                                                           chosen->segment.length_s, seg_emb);
                            ref.embedding = seg_emb;
                            AudioClip view;
                            view.samples = std::move(ref.latent);
                            view.sample_rate = ref.latent_rate;
                            AudioClip st = time_stretch(view, req.duration_s, pc.stft);
                            ref.latent = std::move(st.samples);
                            ref.duration_s = req.duration_s;
                            pl.hit = true;
                            pl.entry_id = chosen->entry_id;
                            pl.similarity = cosine_similarity(req.prompt_embedding, seg_emb);
                            pl.features = context_features(
                                BanditContext{req.prompt_embedding, seg_emb, req.total_steps});
                            pl.reference = std::move(ref);
                        }
                    } catch (const std::exception&) {
                        pl = Plan{};
                        pl.fallback = true;
                    }
                }
                for (int64_t g = b0; g < b1; ++g) {
                    const GenerationRequest& req = trace[(size_t)g];
                    Plan& pl = plans[(size_t)(g - b0)];
                    if (req.arrival_time_s < prev) return -2;
                    prev = req.arrival_time_s;
                    ServeOutcome o;
                    o.request_id = req.id;
                    o.fallback = pl.fallback;
                    int arm = 0;
                    if (pl.hit) {
                        switch (pc.skip_policy) {
                            case SkipPolicy::kModelExploit:
                                arm = choose_arm(pc.gater, pl.features, GaterMode::kExploit);
                                break;
                            case SkipPolicy::kModelExplore:
                                arm = choose_arm(pc.gater, pl.features, GaterMode::kExplore);
                                break;
                            case SkipPolicy::kRuleBased:
                                arm = pl.similarity >= pc.rule_similarity_threshold
                                          ? (int)std::llround(pc.rule_skip_fraction / 0.05) : 0;
                                break;
                            case SkipPolicy::kFixedArm: arm = pc.fixed_arm; break;
                        }
                    } else if (pc.skip_policy == SkipPolicy::kFixedArm) {
                        arm = pc.fixed_arm;
                    }
                    double skip = arm_skip_fraction(arm);
                    const uint64_t gen_seed = derive_seed(pc.seed, req.id, 3);
                    GenerationResult res = generate(req.prompt_embedding, req.duration_s,
                                                    req.total_steps, skip,
                                                    pl.hit ? pl.reference : std::nullopt,
                                                    gen_seed, pc.sim);
                    o.cache_hit = pl.hit;
                    if (pl.hit) o.entry_id = pl.entry_id;
                    o.arm_index = arm;
                    o.skip_fraction = skip;
                    o.steps_skipped = req.total_steps - res.steps_executed;
                    o.quality = res.quality;
                    o.nfe_cost_s = res.nfe_cost_s;
                    o.reference_similarity = pl.similarity;
                    const double now_h = req.arrival_time_s / 3600.0;
                    if (pl.hit)
                        cache.record_reuse(pl.entry_id, o.steps_skipped, req.duration_s, now_h, skip);
                    o.admitted_entry_id = cache.admit(std::move(res.clip), req.prompt_embedding,
                                                      res.quality, now_h);
                    const double start = std::max(req.arrival_time_s, busy);
                    busy = start + o.nfe_cost_s;
                    o.sim_latency_s = busy - req.arrival_time_s;
                    rep.total_nfe_s += o.nfe_cost_s;
                    rep.baseline_nfe_s += pc.sim.nfe_time_s(req.total_steps, req.duration_s);
                    rep.outcomes.push_back(o);
                    // run_maintenance (pipeline.cpp:280-297)
                    for (uint64_t id : cache.refinement_candidates()) {
                        RegenerateFn regen = [&](const EmbeddingVector& prompt, double d,
                                                 uint64_t sd) {
                            auto r = generate(prompt, d, pc.default_total_steps, 0.0,
                                              std::nullopt, sd, pc.sim);
                            return std::make_pair(std::move(r.clip), r.quality);
                        };
                        cache.refine(id, regen, maint);
                        rep.refinements++;
                    }
                }
            }
            std::vector<double> lat;
            double q = 0.0, r = 0.0, h = 0.0;
            for (const auto& o : rep.outcomes) {
                lat.push_back(o.sim_latency_s);
                q += o.quality;
                r += reward(o.arm_index, o.quality, pc.gater.alpha);
                h += o.cache_hit ? 1.0 : 0.0;
            }
            std::sort(lat.begin(), lat.end());
            const double nn = (double)rep.outcomes.size();
            if (nn > 0) {
                auto pct = [&](double p) {
                    size_t idx = (size_t)std::ceil(p * lat.size());
                    return lat[std::min(lat.size() - 1, idx > 0 ? idx - 1 : 0)];
                };
                rep.mean_quality = q / nn;
                rep.mean_reward = r / nn;
                rep.hit_rate = h / nn;
                double ls = 0.0;
                for (double l : lat) ls += l;
                rep.mean_latency_s = ls / nn;
                rep.median_latency_s = pct(0.5);
                rep.p95_latency_s = pct(0.95);
            }
            rep.speedup = rep.total_nfe_s > 0.0 ? rep.baseline_nfe_s / rep.total_nfe_s : 1.0;
        }
        if (wall_s)
            *wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (size_t i = 0; i < rep.outcomes.size(); ++i) copy_out(rep.outcomes[i], out + i);
        if (summary) {
            const double v[10] = {rep.total_nfe_s, rep.baseline_nfe_s, rep.speedup,
                                  rep.mean_quality, rep.mean_reward, rep.hit_rate,
                                  rep.mean_latency_s, rep.median_latency_s, rep.p95_latency_s,
                                  (double)rep.refinements};
            std::memcpy(summary, v, sizeof(v));
        }
        return (int)rep.outcomes.size();
    } catch (const std::exception&) {
        return -1;
    }
}

}  // extern "C"
