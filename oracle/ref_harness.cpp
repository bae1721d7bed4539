// Test infrastructure only (see oracle/Makefile): extern "C" shims that drive the UNMODIFIED
// reference implementation (/root/reference/proj/src, compiled in place) so Python tests and the
// bench's CPU-baseline leg can call it through ctypes. Nothing here re-implements the reference;
// every function forwards to the reference's own C++ API and copies values in/out.
//
// The per-request flow in ref_plan_batch mirrors Pipeline::plan_request + pick_arm
// (reference proj/src/pipeline.cpp:91-202) and the t* line of generate (simgen.cpp:70), with the
// cache's segment rows looked up from the caller-owned row buffer exactly as
// pipeline.cpp:113-131 looks them up through CacheManager::find.

#include <cmath>
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

// ---------------------------------------------------------------- simgen quality (simgen.cpp:12-17)
double ref_expected_quality(double skip, double sigma) {
    QualityModel m;
    return m.expected_quality(skip, sigma);
}

}  // extern "C"
