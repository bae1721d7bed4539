// semwarm_b200.hpp — header-only C++ adapters that put the C-ABI (semwarm_b200.h) behind the
// reference's C++ signatures, so Pipeline-side code keeps calling
//     index.search(query, k) / index.insert(vecs) / index.remove(id)      (index.hpp:59-67)
//     choose_arm(model, ctx, mode)                                         (gater.hpp:56-57)
// unchanged. The adapters are templates over the caller's own types (the reference's
// semwarm::EmbeddingVector / IndexedVector / SearchHit / PyramidDescriptor / BanditContext), so
// they are instantiated against the reference headers without copying them:
//
//     using GpuIndex = semwarm_b200::IvfIndexT<semwarm::EmbeddingVector, semwarm::IndexedVector,
//                                              semwarm::SearchHit>;
//
// Error conventions follow the reference: SW_EINVAL -> std::invalid_argument, other negative
// codes -> std::runtime_error, SW_WARN_UNKNOWN_ID -> a warning callback + no-op.
#pragma once

#include <cstdint>
#include <functional>
#include <iostream>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "semwarm_b200.h"

namespace semwarm_b200 {

inline int check(int rc, const char* what) {
    if (rc == SW_EINVAL) throw std::invalid_argument(std::string(what) + ": " + sw_last_error());
    if (rc < 0) throw std::runtime_error(std::string(what) + ": " + sw_last_error());
    return rc;
}

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

// Drop-in for IvfIndex in exhaustive mode (nprobe >= C): insert / remove / search with the
// reference's exact semantics (fp64 sequential cosine, best segment per entry by strict '>',
// (sim desc, id asc), truncate to k; unknown-id remove warns and is a no-op).
template <class EmbeddingVector, class IndexedVector, class SearchHit>
class IvfIndexT {
public:
    using Warn = std::function<void(const std::string&)>;

    IvfIndexT(int dim, int rows_per_entry, int64_t capacity, int max_batch = 1024,
              int device = 0, uint32_t flags = 0)
        : ctx_(dim, rows_per_entry, capacity, max_batch, 0, 0, 0, flags, device) {}

    void set_warn(Warn w) { warn_ = std::move(w); }

    // IvfIndex::insert (index.cpp:226-239): rows grouped by entry id, pyramid order kept
    void insert(const std::vector<IndexedVector>& vecs) {
        if (vecs.empty()) return;
        std::vector<uint64_t> ids;
        std::vector<int64_t> off{0};
        std::vector<float> rows;
        std::vector<sw_segment> segs;
        for (size_t i = 0; i < vecs.size(); ++i) {
            const auto& v = vecs[i];
            if ((int)v.embedding.dim() != ctx_.dim())
                throw std::invalid_argument("embedding dimension mismatch");
            if (ids.empty() || ids.back() != v.entry_id) {
                if (!ids.empty()) off.push_back((int64_t)segs.size());
                ids.push_back(v.entry_id);
            }
            rows.insert(rows.end(), v.embedding.values.begin(), v.embedding.values.end());
            segs.push_back(sw_segment{v.segment.level, 0, v.segment.start_s, v.segment.length_s});
        }
        off.push_back((int64_t)segs.size());
        check(sw_arena_insert_batch(ctx_.get(), (int64_t)ids.size(), ids.data(), off.data(),
                                    rows.data(), segs.data(), nullptr, nullptr, nullptr, 0),
              "insert");
    }

    // IvfIndex::remove (index.cpp:241-255)
    void remove(uint64_t entry_id) {
        if (check(sw_arena_remove(ctx_.get(), entry_id), "remove") == SW_WARN_UNKNOWN_ID) {
            const std::string m = "remove of unknown entry id " + std::to_string(entry_id);
            if (warn_) warn_(m); else std::cerr << "[semwarm_b200] warning: " << m << "\n";
        }
    }

    // IvfIndex::search (index.cpp:289-326), one query
    std::vector<SearchHit> search(const EmbeddingVector& query, size_t k) const {
        return search_batch({query}, k).front();
    }

    // B queries in one device pass
    std::vector<std::vector<SearchHit>> search_batch(const std::vector<EmbeddingVector>& qs,
                                                     size_t k) const {
        if (k < 1) throw std::invalid_argument("search k must be >= 1");  // index.cpp:291
        const int B = (int)qs.size();
        std::vector<float> q((size_t)B * ctx_.dim());
        for (int b = 0; b < B; ++b) {
            if ((int)qs[b].dim() != ctx_.dim())
                throw std::invalid_argument("embedding dimension mismatch");
            std::copy(qs[b].values.begin(), qs[b].values.end(), q.begin() + (size_t)b * ctx_.dim());
        }
        std::vector<sw_hit> hits((size_t)B * k);
        std::vector<int32_t> n(B);
        check(sw_search_host(ctx_.get(), q.data(), B, (int32_t)k, hits.data(), n.data()),
              "search");
        std::vector<std::vector<SearchHit>> out(B);
        for (int b = 0; b < B; ++b) {
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

    size_t entry_count() const { return (size_t)sw_arena_entry_count(ctx_.get()); }
    bool contains(uint64_t id) const { return sw_arena_contains(ctx_.get(), id) != 0; }
    sw_ctx* context() const { return ctx_.get(); }

private:
    Context ctx_;
    Warn warn_;
};

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
