// semwarm_b200.hpp — header-only C++ adapters that put the C-ABI (semwarm_b200.h) behind the
// reference's C++ signatures, so the reference's own CacheManager / Pipeline keep calling
//     IvfIndex::build / insert / remove / search / set_rebuild_interval / check_consistent /
//     entry_count / contains / save / load                                 (index.hpp:47-101)
//     score_candidates / select                                            (selector.hpp:50-58)
//     choose_arm (batched)                                                 (gater.hpp:56-57)
// unchanged. The adapters are templates over the caller's own types (the reference's
// semwarm::EmbeddingVector / IndexedVector / SearchHit / CandidateInput / CandidateScore /
// SelectorConfig / Rng), so they are instantiated against the reference headers without copying
// them:
//
//     using GpuIvfIndex = semwarm_b200::IvfIndexT<semwarm::EmbeddingVector,
//                                                 semwarm::IndexedVector, semwarm::SearchHit>;
//
// and the reference's CacheManager then holds a GpuIvfIndex where it held an IvfIndex (a type
// swap in cache.hpp / cache.cpp). tools/dropin/ builds exactly that swap against
// the unmodified reference sources and replays a workload through the reference Pipeline.
//
// Error conventions follow the reference: SW_EINVAL -> std::invalid_argument, other negative
// codes -> std::runtime_error, SW_WARN_UNKNOWN_ID -> a warning (stderr or a callback) + no-op.
#pragma once

#include <cstdint>
#include <cstring>
#include <fstream>
#include <functional>
#include <iostream>
#include <iterator>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "semwarm_b200.h"

namespace semwarm_b200 {

inline int check(int rc, const char* what) {
    if (rc == SW_EINVAL) throw std::invalid_argument(std::string(what) + ": " + sw_last_error());
    if (rc < 0) throw std::runtime_error(std::string(what) + ": " + sw_last_error());
    return rc;
}

inline void default_warn(const std::string& m) { std::cerr << "[semwarm] warning: " << m << "\n"; }

// Owns one device arena (one cache shard). Movable, not copyable.
class Context {
public:
    Context(int dim, int rows_per_entry, int64_t max_entries, int max_batch = 1024,
            int latent_c = 8, int latent_t_max = 256, int latent_f = 16, uint32_t flags = 0,
            int device = 0, int64_t latent_slots = 0) {
        sw_config cfg{};
        cfg.dim = dim;
        cfg.rows_per_entry = rows_per_entry;
        cfg.max_entries = max_entries;
        cfg.latent_c = latent_c;
        cfg.latent_t_max = latent_t_max;
        cfg.latent_f = latent_f;
        cfg.max_batch = max_batch;
        cfg.latent_slots = latent_slots;
        cfg.latent_fps = 25.0;
        cfg.flags = flags;
        check(sw_ctx_create(&cfg, device, &ctx_), "sw_ctx_create");
        dim_ = dim;
    }
    ~Context() {
        if (ctx_) sw_ctx_destroy(ctx_);
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    Context(Context&& o) noexcept : ctx_(o.ctx_), dim_(o.dim_) { o.ctx_ = nullptr; }
    sw_ctx* get() const { return ctx_; }
    int dim() const { return dim_; }

private:
    sw_ctx* ctx_ = nullptr;
    int dim_ = 0;
};

// Geometry of the arenas IvfIndexT creates lazily (the reference IvfIndex has no capacity or
// shape: it learns the dimension from the first vector and grows without bound). rows_per_entry
// 0 = the largest row count among the first inserted entries (7 at the reference's delta 1/4);
// capacity is the initial entry count — the arena grows (doubling) past it.
struct ArenaDefaults {
    int rows_per_entry = 0;
    int64_t capacity = 1024;
    int max_batch = 1024;
    int device = 0;
    uint32_t flags = 0;
};
inline ArenaDefaults& arena_defaults() {
    static ArenaDefaults d;
    return d;
}

// Drop-in for semwarm::IvfIndex (index.hpp:47-101) on the B200 arena: the same static build,
// insert / remove / search (exhaustive or IVF: probe ranking, list-restricted scan, mutation-
// counted k-means rebuilds — bit-identical to the reference), the same accessors and the SWIX
// snapshot. Value semantics as far as the reference uses them: default-constructible and
// movable (CacheManager::load_snapshot move-assigns a fresh build); not copyable (the arena lives
// in HBM).
template <class EmbeddingVector, class IndexedVector, class SearchHit>
class IvfIndexT {
public:
    using Warn = std::function<void(const std::string&)>;

    IvfIndexT() = default;

    // Explicit geometry (exhaustive mode). Capacity is the initial entry count (grows).
    IvfIndexT(int dim, int rows_per_entry, int64_t capacity, int max_batch = 1024,
              int device = 0, uint32_t flags = 0) {
        ctx_ = std::make_unique<Context>(dim, rows_per_entry, capacity, max_batch, 0, 0, 0,
                                         flags | SW_FLAG_GROW, device);
        configured_ = true;
    }

    IvfIndexT(IvfIndexT&&) noexcept = default;
    IvfIndexT& operator=(IvfIndexT&&) noexcept = default;
    IvfIndexT(const IvfIndexT&) = delete;
    IvfIndexT& operator=(const IvfIndexT&) = delete;

    // IvfIndex::build (index.cpp:186-208): C target centroids, k-means seed, nprobe. An empty
    // `vecs` (CacheManager's constructor, cache.cpp:17) only records the configuration.
    static IvfIndexT build(std::vector<IndexedVector> vecs, uint32_t c, uint64_t seed,
                           uint32_t nprobe = 8) {
        if (c < 1) throw std::invalid_argument("centroid count must be >= 1");
        IvfIndexT idx;
        idx.ivf_ = true;
        idx.target_ = c;
        idx.seed_ = seed;
        idx.nprobe_ = nprobe;
        if (!vecs.empty()) {
            if (vecs.size() < c)
                idx.warn_("fewer vectors (" + std::to_string(vecs.size()) + ") than centroids (" +
                          std::to_string(c) + "); reducing C");
            idx.ensure_ctx(vecs);
            Packed p = pack(vecs, idx.ctx_->dim());
            check(sw_ivf_build(idx.ctx_->get(), (int64_t)p.ids.size(), p.ids.data(), p.off.data(),
                               p.rows.data(), p.segs.data()),
                  "IvfIndex::build");
        }
        return idx;
    }

    void set_warn(Warn w) { warn_ = std::move(w); }

    // IvfIndex::insert (index.cpp:224-234): rows grouped by consecutive entry id, order kept
    void insert(std::vector<IndexedVector> vecs) {
        if (vecs.empty()) return;
        ensure_ctx(vecs);
        Packed p = pack(vecs, ctx_->dim());
        check(sw_arena_insert_batch(ctx_->get(), (int64_t)p.ids.size(), p.ids.data(),
                                    p.off.data(), p.rows.data(), p.segs.data(), nullptr, nullptr,
                                    nullptr, 0),
              "IvfIndex::insert");
    }

    // IvfIndex::remove (index.cpp:236-255): unknown ids are a warning no-op
    void remove(uint64_t entry_id) {
        const int rc = ctx_ ? check(sw_arena_remove(ctx_->get(), entry_id), "IvfIndex::remove")
                            : SW_WARN_UNKNOWN_ID;
        if (rc == SW_WARN_UNKNOWN_ID) warn_("remove of unknown entry id " + std::to_string(entry_id));
    }

    // IvfIndex::search (index.cpp:285-326)
    std::vector<SearchHit> search(const EmbeddingVector& query, size_t k) const {
        return search(query, k, 0);
    }
    std::vector<SearchHit> search(const EmbeddingVector& query, size_t k, uint32_t nprobe) const {
        if (k < 1) throw std::invalid_argument("search k must be >= 1");  // index.cpp:291
        if (!ctx_) return {};  // no centroids yet (index.cpp:292)
        return search_batch_impl({query}, k, nprobe).front();
    }

    // B queries in one device pass (the batched form sw_plan builds on)
    std::vector<std::vector<SearchHit>> search_batch(const std::vector<EmbeddingVector>& qs,
                                                     size_t k) const {
        if (k < 1) throw std::invalid_argument("search k must be >= 1");
        if (!ctx_) return std::vector<std::vector<SearchHit>>(qs.size());
        return search_batch_impl(qs, k, 0);
    }

    size_t centroid_count() const {
        if (!ctx_) return 0;
        int32_t n = 0;
        check(sw_ivf_info(ctx_->get(), &n, nullptr, nullptr), "centroid_count");
        return (size_t)n;
    }
    size_t total_vectors() const { return ctx_ ? (size_t)sw_arena_row_count(ctx_->get()) : 0; }
    size_t entry_count() const { return ctx_ ? (size_t)sw_arena_entry_count(ctx_->get()) : 0; }
    bool contains(uint64_t id) const { return ctx_ && sw_arena_contains(ctx_->get(), id) != 0; }
    uint32_t nprobe() const { return nprobe_; }
    void set_nprobe(uint32_t n) {
        nprobe_ = n;
        if (ctx_ && ivf_) check(sw_ivf_set_nprobe(ctx_->get(), (int32_t)n), "set_nprobe");
    }
    void set_rebuild_interval(uint64_t n) {
        interval_ = n;
        if (ctx_ && ivf_) check(sw_ivf_set_rebuild_interval(ctx_->get(), n), "set_rebuild_interval");
    }

    // IvfIndex::check_consistent (index.cpp:334-343), recomputed on the device
    bool check_consistent() const { return !ctx_ || sw_index_check_consistent(ctx_->get()) == 1; }

    // IvfIndex::save / load (index.cpp:347-406): the SWIX snapshot, read and written by the
    // device arena directly
    void save(const std::string& path) const {
        if (ctx_) {
            check(sw_swix_save(ctx_->get(), path.c_str()), "IvfIndex::save");
            return;
        }
        std::string out("SWIX", 4);  // an index that never saw a vector: no centroids
        const uint32_t hdr[3] = {0u, nprobe_, 0u};
        out.append(reinterpret_cast<const char*>(hdr), sizeof(hdr));
        std::ofstream f(path, std::ios::binary | std::ios::trunc);
        if (!f) throw std::runtime_error("cannot write " + path);
        f.write(out.data(), (std::streamsize)out.size());
    }
    static IvfIndexT load(const std::string& path) {
        uint32_t C = 0, nprobe = 8, dim = 0;
        int max_rows = 1;
        scan_swix(path, &C, &nprobe, &dim, &max_rows);
        IvfIndexT idx;
        idx.ivf_ = true;
        idx.target_ = C > 0 ? C : 1;
        idx.nprobe_ = nprobe;
        idx.seed_ = 0;  // IvfIndex::load leaves seed 0 and no rebuilds
        if (C == 0) return idx;
        const ArenaDefaults& d = arena_defaults();
        int64_t entries = 0;
        scan_swix(path, nullptr, nullptr, nullptr, nullptr, &entries);
        idx.ctx_ = std::make_unique<Context>((int)dim, std::max(max_rows, d.rows_per_entry),
                                             std::max<int64_t>(d.capacity, entries), d.max_batch,
                                             0, 0, 0, d.flags | SW_FLAG_GROW, d.device);
        check(sw_swix_load(idx.ctx_->get(), path.c_str()), "IvfIndex::load");
        idx.configured_ = true;
        return idx;
    }

    sw_ctx* context() const { return ctx_ ? ctx_->get() : nullptr; }

private:
    struct Packed {
        std::vector<uint64_t> ids;
        std::vector<int64_t> off{0};
        std::vector<float> rows;
        std::vector<sw_segment> segs;
    };

    static Packed pack(const std::vector<IndexedVector>& vecs, int dim) {
        Packed p;
        p.rows.reserve(vecs.size() * (size_t)dim);
        for (const auto& v : vecs) {
            if ((int)v.embedding.dim() != dim)
                throw std::invalid_argument("dot: dimension mismatch");  // core.cpp:22-25
            if (p.ids.empty() || p.ids.back() != v.entry_id) {
                if (!p.ids.empty()) p.off.push_back((int64_t)p.segs.size());
                p.ids.push_back(v.entry_id);
            }
            p.rows.insert(p.rows.end(), v.embedding.values.begin(), v.embedding.values.end());
            p.segs.push_back(sw_segment{v.segment.level, 0, v.segment.start_s, v.segment.length_s});
        }
        p.off.push_back((int64_t)p.segs.size());
        return p;
    }

    // the first vectors fix the arena's dimension and rows per entry (lazy, like IvfIndex)
    void ensure_ctx(const std::vector<IndexedVector>& vecs) {
        if (ctx_) return;
        const ArenaDefaults& d = arena_defaults();
        int rows = d.rows_per_entry;
        if (rows <= 0) {
            std::map<uint64_t, int> cnt;
            for (const auto& v : vecs) rows = std::max(rows, ++cnt[v.entry_id]);
        }
        ctx_ = std::make_unique<Context>((int)vecs.front().embedding.dim(), rows, d.capacity,
                                         d.max_batch, 0, 0, 0, d.flags | SW_FLAG_GROW, d.device);
        if (ivf_)
            check(sw_ivf_configure(ctx_->get(), (int32_t)target_, (int32_t)nprobe_, interval_, seed_),
                  "IvfIndex::build");
        configured_ = true;
    }

    std::vector<std::vector<SearchHit>> search_batch_impl(const std::vector<EmbeddingVector>& qs,
                                                          size_t k, uint32_t nprobe) const {
        const int B = (int)qs.size();
        const int D = ctx_->dim();
        std::vector<float> q((size_t)B * D);
        for (int b = 0; b < B; ++b) {
            if ((int)qs[b].dim() != D) throw std::invalid_argument("dot: dimension mismatch");
            std::copy(qs[b].values.begin(), qs[b].values.end(), q.begin() + (size_t)b * D);
        }
        std::vector<sw_hit> hits((size_t)B * k);
        std::vector<int32_t> n(B);
        check(sw_search_host_ex(ctx_->get(), q.data(), B, (int32_t)k, (int32_t)nprobe,
                                hits.data(), n.data()),
              "IvfIndex::search");
        std::vector<std::vector<SearchHit>> out(B);
        for (int b = 0; b < B; ++b) {
            out[b].reserve(n[b]);
            for (int i = 0; i < n[b]; ++i) {
                const sw_hit& h = hits[(size_t)b * k + i];
                SearchHit s;
                s.entry_id = h.entry_id;
                s.segment.level = h.segment.level;
                s.segment.start_s = h.segment.start_s;
                s.segment.length_s = h.segment.length_s;
                s.similarity = h.similarity;
                out[b].push_back(s);
            }
        }
        return out;
    }

    // SWIX header and shape (index.cpp:347-369): C, nprobe, D, the largest row count of an
    // entry and the entry count
    static void scan_swix(const std::string& path, uint32_t* C, uint32_t* nprobe, uint32_t* dim,
                          int* max_rows, int64_t* entries = nullptr) {
        std::ifstream f(path, std::ios::binary);
        if (!f) throw std::runtime_error("cannot open index snapshot: " + path);
        const std::string b((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
        if (b.size() < 16 || std::memcmp(b.data(), "SWIX", 4) != 0)
            throw std::runtime_error("not an index snapshot (bad magic): " + path);
        uint32_t h[3];
        std::memcpy(h, b.data() + 4, 12);
        if (C) *C = h[0];
        if (nprobe) *nprobe = h[1];
        if (dim) *dim = h[2];
        if (!max_rows && !entries) return;
        size_t p = 16 + (size_t)h[0] * h[2] * 4;
        const size_t rec = 8 + 1 + 4 + 4 + (size_t)h[2] * 4;
        std::map<uint64_t, int> cnt;
        for (uint32_t j = 0; j < h[0]; ++j) {
            if (p + 8 > b.size()) throw std::runtime_error("index snapshot truncated: " + path);
            uint64_t n;
            std::memcpy(&n, b.data() + p, 8);
            p += 8;
            for (uint64_t i = 0; i < n; ++i, p += rec) {
                if (p + rec > b.size()) throw std::runtime_error("index snapshot truncated: " + path);
                uint64_t id;
                std::memcpy(&id, b.data() + p, 8);
                ++cnt[id];
            }
        }
        int m = 1;
        for (auto& kv : cnt) m = std::max(m, kv.second);
        if (max_rows) *max_rows = m;
        if (entries) *entries = (int64_t)cnt.size();
    }

    std::unique_ptr<Context> ctx_;
    bool configured_ = false;
    bool ivf_ = false;        // built through build()/load(): IVF bookkeeping like IvfIndex
    uint32_t target_ = 1;     // target_centroids_
    uint32_t nprobe_ = 8;     // nprobe_
    uint64_t seed_ = 0;       // seed_
    uint64_t interval_ = 1024;  // rebuild_interval_
    Warn warn_ = default_warn;
};

// ---------------------------------------------------------------- selector
// score_candidates + select (selector.cpp:24-85) on the device, templated on the reference's
// CandidateInput / CandidateScore / SelectorConfig / Rng. s_neg = clamp01(cos(audio embedding,
// cfg.negative_embedding)) and the gate run on the device in the reference's fp64 operation
// order; select draws rng.uniform() on the host exactly when the reference does (some candidate
// survives the gate), so the caller's RNG stream advances identically.
template <class CandidateScore, class CandidateInput, class EmbeddingVector, class SelectorConfig>
std::vector<CandidateScore> score_candidates(sw_ctx* ctx, const std::vector<CandidateInput>& cands,
                                             const EmbeddingVector& prompt, double L,
                                             const SelectorConfig& cfg) {
    (void)prompt;  // s_pos arrives precomputed from index search (selector.cpp:36)
    const int n = (int)cands.size();
    if (n == 0) throw std::invalid_argument("score_candidates: empty candidate list");
    if (!(L > 0.0)) throw std::invalid_argument("requested duration must be positive");
    const int D = (int)cfg.negative_embedding.dim();
    std::vector<double> sims(n), dur(n), sc((size_t)n * 5);
    std::vector<float> audio((size_t)n * D);
    for (int i = 0; i < n; ++i) {
        sims[i] = cands[i].prompt_similarity;
        dur[i] = cands[i].duration_s;
        if ((int)cands[i].audio_embedding.dim() != D)
            throw std::invalid_argument("dot: dimension mismatch");
        std::copy(cands[i].audio_embedding.values.begin(), cands[i].audio_embedding.values.end(),
                  audio.begin() + (size_t)i * D);
    }
    check(sw_score_candidates_host(ctx, n, D, sims.data(), audio.data(), dur.data(), L,
                                   cfg.negative_embedding.values.data(), sc.data()),
          "score_candidates");
    std::vector<CandidateScore> out(n);
    for (int i = 0; i < n; ++i) {
        CandidateScore& s = out[i];
        s.entry_id = cands[i].entry_id;
        s.segment = cands[i].segment;
        s.duration_s = cands[i].duration_s;
        s.s_pos = sc[(size_t)i * 5 + 0];
        s.s_neg = sc[(size_t)i * 5 + 1];
        s.a = sc[(size_t)i * 5 + 2];
        s.b = sc[(size_t)i * 5 + 3];
        s.q = sc[(size_t)i * 5 + 4];
    }
    return out;
}

template <class CandidateScore, class SelectorConfig, class Rng>
std::optional<size_t> select(sw_ctx* ctx, const std::vector<CandidateScore>& scored,
                             const SelectorConfig& cfg, Rng& rng) {
    if (cfg.top_k < 1) throw std::invalid_argument("selector top_k must be >= 1");
    if (!(cfg.temperature > 0.0)) throw std::invalid_argument("selector temperature must be > 0");
    if (cfg.quality_threshold < 0.0 || cfg.quality_threshold > 1.0)
        throw std::invalid_argument("selector quality threshold must be in [0, 1]");
    const int n = (int)scored.size();
    bool any = false;
    std::vector<double> s_pos(n), q(n);
    for (int i = 0; i < n; ++i) {
        s_pos[i] = scored[i].s_pos;
        q[i] = scored[i].q;
        any = any || q[i] >= cfg.quality_threshold;
    }
    if (!any) return std::nullopt;  // no survivor: no draw (selector.cpp:67)
    const double u = rng.uniform();
    int32_t pick = -1;
    uint32_t flags = 0;
    check(sw_select_host(ctx, n, s_pos.data(), q.data(), cfg.temperature, cfg.quality_threshold,
                         u, &pick, &flags),
          "select");
    if (pick < 0) return std::nullopt;
    return (size_t)pick;
}

// ---------------------------------------------------------------- gater
// context_features + choose_arm (gater.cpp:13-92) for a batch of (prompt, segment) contexts,
// evaluated on the device with the reference's operation order. Returns arms; fills phi.
template <class EmbeddingVector>
std::vector<int> choose_arms(sw_ctx* ctx, const std::vector<EmbeddingVector>& prompts,
                             const std::vector<EmbeddingVector>& segments,
                             const std::vector<int>& total_steps, bool explore,
                             std::vector<double>* phi = nullptr) {
    const int B = (int)prompts.size();
    if (B == 0) return {};
    const size_t D = prompts[0].dim();
    std::vector<float> p((size_t)B * D), s((size_t)B * D);
    for (int b = 0; b < B; ++b) {
        std::copy(prompts[b].values.begin(), prompts[b].values.end(), p.begin() + b * D);
        std::copy(segments[b].values.begin(), segments[b].values.end(), s.begin() + b * D);
    }
    std::vector<double> f((size_t)B * 11);
    std::vector<int32_t> arms(B);
    std::vector<int32_t> T(total_steps.begin(), total_steps.end());
    check(sw_gater_host(ctx, p.data(), s.data(), T.data(), B, explore ? 1 : 0, f.data(),
                        arms.data()),
          "choose_arm");
    if (phi) *phi = f;
    return std::vector<int>(arms.begin(), arms.end());
}

}  // namespace semwarm_b200
