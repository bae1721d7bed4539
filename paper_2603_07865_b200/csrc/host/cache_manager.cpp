// Cache Manager host policy over the device arena (reference cache.hpp / cache.cpp).
//
// The policy — quality-floor admission, the reuse ledger with lazy gamma^dt decay, grace-aware
// lowest-importance eviction, best-of-N refinement with an attempt cap, the refine trigger —
// stays on the host exactly as in the reference (its decisions are sequential, libm pow-based and
// tiny). Every data-plane effect goes to the device arena through the C-ABI: admit ->
// sw_arena_insert (rows, bf16 shadow, s_neg, latent slot), evict -> sw_arena_remove, refine ->
// sw_arena_replace. Segment embeddings are derived on the host with the reference's own
// algorithm (derive_segment_embedding, index.cpp:33-46: mt19937_64 + Box-Muller through libm),
// as SURVEY §8a A4 prescribes, so the rows the arena holds are bit-identical to the reference's.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "semwarm_b200.h"

namespace {

// ---- core.cpp:58-124 (seeding, Rng::uniform/normal, normalize, random_unit_vector)
uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
uint64_t derive_seed(uint64_t base, uint64_t a, uint64_t b = 0, uint64_t c = 0) {
    uint64_t s = splitmix64(base ^ 0x53454d5741524dULL);
    s = splitmix64(s ^ a);
    s = splitmix64(s ^ b);
    return splitmix64(s ^ c);
}

class HostRng {
public:
    explicit HostRng(uint64_t seed) : gen_(seed) {}
    uint64_t next_u64() { return gen_(); }
    double uniform() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
    double normal() {  // Box-Muller with the cached spare (core.cpp:85-100)
        if (have_spare_) {
            have_spare_ = false;
            return spare_;
        }
        double u1, u2;
        do {
            u1 = uniform();
        } while (u1 <= 0.0);
        u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double theta = 2.0 * M_PI * u2;
        spare_ = r * std::sin(theta);
        have_spare_ = true;
        return r * std::cos(theta);
    }

private:
    std::mt19937_64 gen_;
    bool have_spare_ = false;
    double spare_ = 0.0;
};

std::vector<float> normalize(const std::vector<float>& raw) {  // core.cpp:40-52
    double s = 0.0;
    for (float v : raw) s += static_cast<double>(v) * v;
    const double n = std::sqrt(s);
    std::vector<float> out(raw.size());
    for (size_t i = 0; i < raw.size(); ++i) out[i] = static_cast<float>(raw[i] / n);
    return out;
}

std::vector<float> random_unit_vector(size_t dim, HostRng& rng) {  // core.cpp:110-114
    std::vector<float> v(dim);
    for (size_t i = 0; i < dim; ++i) v[i] = static_cast<float>(rng.normal());
    return normalize(v);
}

struct Seg {
    int level;
    double start, length;
};

// pyramid_segments (index.cpp:12-31)
std::vector<Seg> pyramid_segments(double duration, double delta) {
    if (delta < 1.0 / 16.0) delta = 1.0 / 16.0;
    const int max_level = static_cast<int>(std::floor(std::log2(1.0 / delta) + 1e-9));
    std::vector<Seg> out;
    for (int level = 0; level <= max_level; ++level) {
        const int tiles = 1 << level;
        const double len = duration / tiles;
        for (int i = 0; i < tiles; ++i) out.push_back(Seg{level, i * len, len});
    }
    return out;
}

// derive_segment_embedding (index.cpp:33-46)
std::vector<float> segment_embedding(const std::vector<float>& full, uint64_t id, const Seg& s,
                                     uint64_t seed_base) {
    if (s.level == 0) return full;
    const uint64_t tile = s.length > 0.0 ? static_cast<uint64_t>(std::llround(s.start / s.length)) : 0;
    HostRng rng(derive_seed(seed_base, id, static_cast<uint64_t>(s.level), tile));
    const std::vector<float> dir = random_unit_vector(full.size(), rng);
    std::vector<float> v(full.size());
    for (size_t i = 0; i < full.size(); ++i) v[i] = static_cast<float>(full[i] + 0.1 * dir[i]);
    return normalize(v);
}

struct Entry {
    uint64_t id = 0;
    double duration_s = 0.0;
    std::vector<float> prompt;
    double quality = 0.0;
    double importance = 0.0;
    double last_update_h = 0.0;
    double admitted_h = 0.0;
    int refinement_attempts = 0;
    size_t reuse_count = 0;
    std::deque<double> recent_skips;
};

}  // namespace

struct swcm_cache {
    sw_ctx* ctx = nullptr;
    int dim = 0;
    swcm_config cfg{};
    std::map<uint64_t, Entry> entries;  // ordered by id, like the reference's std::map
    uint64_t next_id = 1;
    std::vector<uint64_t> last_evicted;

    double decayed(const Entry& e, double now_h) const {  // cache.cpp:24-28
        const double dt = now_h - e.last_update_h;
        if (dt <= 0.0) return e.importance;
        return e.importance * std::pow(cfg.decay_per_hour, dt);
    }

    int write_rows(bool replace, uint64_t id, const std::vector<float>& full, double duration,
                   const float* latent, int t_src) {
        const std::vector<Seg> segs = pyramid_segments(duration, cfg.pyramid_delta);
        std::vector<float> rows;
        std::vector<sw_segment> ss;
        for (const Seg& s : segs) {
            const std::vector<float> v = segment_embedding(full, id, s, cfg.embedding_seed);
            rows.insert(rows.end(), v.begin(), v.end());
            ss.push_back(sw_segment{s.level, 0, s.start, s.length});
        }
        return replace ? sw_arena_replace(ctx, id, (int32_t)segs.size(), rows.data(), ss.data(),
                                          latent, t_src)
                       : sw_arena_insert(ctx, id, (int32_t)segs.size(), rows.data(), ss.data(),
                                         latent, t_src);
    }

    int evict_if_full(double now_h, std::vector<uint64_t>& evicted) {  // cache.cpp:70-105
        while (entries.size() > cfg.capacity) {
            const Entry* victim = nullptr;
            double victim_imp = 0.0;
            bool victim_graced = true;
            for (const auto& kv : entries) {
                const Entry& e = kv.second;
                const bool graced = now_h - e.admitted_h < cfg.grace_hours;
                const double imp = decayed(e, now_h);
                bool better;
                if (victim == nullptr) better = true;
                else if (graced != victim_graced) better = !graced;
                else if (imp != victim_imp) better = imp < victim_imp;
                else if (e.last_update_h != victim->last_update_h)
                    better = e.last_update_h < victim->last_update_h;
                else better = e.id < victim->id;
                if (better) {
                    victim = &e;
                    victim_imp = imp;
                    victim_graced = graced;
                }
            }
            const uint64_t id = victim->id;
            const int rc = sw_arena_remove(ctx, id);
            if (rc < 0) return rc;
            entries.erase(id);
            evicted.push_back(id);
        }
        return SW_OK;
    }
};

extern "C" {

int swcm_create(sw_ctx* ctx, int32_t dim, const swcm_config* cfg, swcm_cache** out) {
    if (!ctx || !cfg || !out || dim < 1 || cfg->capacity < 1) return SW_EINVAL;
    // admit inserts before it evicts (cache.cpp:30-52): the arena must hold capacity + 1 entries
    if (sw_arena_capacity(ctx) < (int64_t)cfg->capacity + 1) return SW_ENOMEM;
    auto* h = new swcm_cache;
    h->ctx = ctx;
    h->dim = dim;
    h->cfg = *cfg;
    *out = h;
    return SW_OK;
}

int swcm_destroy(swcm_cache* h) {
    delete h;
    return SW_OK;
}

int swcm_admit(swcm_cache* h, const float* clip_embedding, double duration_s,
               const float* prompt_embedding, double quality, double now_h, const float* latent,
               int32_t t_src, uint64_t* id_out) {  // cache.cpp:30-52
    if (!h || !clip_embedding || !id_out) return SW_EINVAL;
    h->last_evicted.clear();
    *id_out = 0;
    if (quality < h->cfg.quality_floor) return 0;  // rejected: not an error
    if (!(duration_s > 0.0)) return SW_EINVAL;     // pyramid_segments (index.cpp:17-19)
    Entry e;
    e.id = h->next_id;
    e.duration_s = duration_s;
    if (prompt_embedding) e.prompt.assign(prompt_embedding, prompt_embedding + h->dim);
    e.quality = quality;
    e.importance = 0.0;
    e.last_update_h = now_h;
    e.admitted_h = now_h;
    const std::vector<float> full(clip_embedding, clip_embedding + h->dim);
    int rc = h->write_rows(false, e.id, full, duration_s, latent, t_src);
    if (rc < 0) return rc;  // nothing stored: the id is not consumed
    ++h->next_id;
    const uint64_t id = e.id;
    h->entries.emplace(id, std::move(e));
    rc = h->evict_if_full(now_h, h->last_evicted);
    if (rc < 0) return rc;
    *id_out = id;
    return 1;
}

int swcm_last_evicted(const swcm_cache* h, uint64_t* out, int32_t cap) {
    if (!h) return SW_EINVAL;
    const int n = (int)h->last_evicted.size();
    for (int i = 0; i < n && i < cap; ++i) out[i] = h->last_evicted[i];
    return n;
}

int swcm_record_reuse(swcm_cache* h, uint64_t id, int32_t steps_skipped, double duration_s,
                      double now_h, double skip_fraction) {  // cache.cpp:54-68
    if (!h) return SW_EINVAL;
    auto it = h->entries.find(id);
    if (it == h->entries.end()) return SW_WARN_UNKNOWN_ID;
    Entry& e = it->second;
    e.importance = h->decayed(e, now_h);
    e.importance += static_cast<double>(steps_skipped) * duration_s;
    e.last_update_h = now_h;
    e.reuse_count++;
    e.recent_skips.push_back(skip_fraction);
    while (e.recent_skips.size() > (size_t)h->cfg.refine_window) e.recent_skips.pop_front();
    return SW_OK;
}

int swcm_evict_if_full(swcm_cache* h, double now_h, uint64_t* out, int32_t cap) {
    if (!h) return SW_EINVAL;
    std::vector<uint64_t> ev;
    const int rc = h->evict_if_full(now_h, ev);
    if (rc < 0) return rc;
    for (size_t i = 0; i < ev.size() && (int)i < cap; ++i) out[i] = ev[i];
    return (int)ev.size();
}

int swcm_refinement_candidates(const swcm_cache* h, uint64_t* out, int32_t cap) {
    if (!h) return SW_EINVAL;  // cache.cpp:142-154
    int n = 0;
    for (const auto& kv : h->entries) {
        const Entry& e = kv.second;
        if (e.refinement_attempts >= h->cfg.refine_attempt_cap) continue;
        if (e.reuse_count < (size_t)h->cfg.refine_window) continue;
        if (e.recent_skips.size() < (size_t)h->cfg.refine_window) continue;
        double mean = 0.0;
        for (double s : e.recent_skips) mean += s;
        mean /= static_cast<double>(e.recent_skips.size());
        if (mean < h->cfg.refine_skip_threshold) {
            if (n < cap) out[n] = kv.first;
            ++n;
        }
    }
    return n;
}

int swcm_refine(swcm_cache* h, uint64_t id, uint64_t rng_seed, swcm_regenerate_fn regen,
                void* user, int32_t* replaced) {  // cache.cpp:107-140
    if (!h || !regen || !replaced) return SW_EINVAL;
    *replaced = 0;
    auto it = h->entries.find(id);
    if (it == h->entries.end()) return SW_WARN_UNKNOWN_ID;
    Entry& e = it->second;
    if (e.refinement_attempts >= h->cfg.refine_attempt_cap) return SW_OK;  // warn + no-op
    e.refinement_attempts++;
    HostRng rng(rng_seed);
    std::vector<float> best_emb(h->dim), emb(h->dim);
    std::vector<float> lat;
    double best_q = -1.0;
    int best_t = 0;
    const size_t lat_cap = (size_t)h->cfg.latent_capacity;
    std::vector<float> cur_lat(lat_cap);
    std::vector<float> best_lat(lat_cap);
    for (int i = 0; i < h->cfg.refine_regenerations; ++i) {
        double q = 0.0;
        int32_t t = 0;
        const int rc = regen(user, e.prompt.empty() ? nullptr : e.prompt.data(), h->dim,
                             e.duration_s, rng.next_u64(), emb.data(), &q,
                             lat_cap ? cur_lat.data() : nullptr, &t);
        if (rc < 0) return rc;
        if (q > best_q) {
            best_q = q;
            best_emb = emb;
            best_t = t;
            if (lat_cap) best_lat = cur_lat;
        }
    }
    if (best_q <= e.quality) return SW_OK;
    const int rc = h->write_rows(true, e.id, best_emb, e.duration_s,
                                 lat_cap && best_t > 0 ? best_lat.data() : nullptr, best_t);
    if (rc < 0) return rc;  // the ledger keeps the quality the arena still holds
    e.quality = best_q;
    e.recent_skips.clear();
    *replaced = 1;
    return SW_OK;
}

int swcm_importance(const swcm_cache* h, uint64_t id, double now_h, double* out) {
    if (!h || !out) return SW_EINVAL;
    auto it = h->entries.find(id);
    if (it == h->entries.end()) return SW_EINVAL;  // cache.cpp:158 throws invalid_argument
    *out = h->decayed(it->second, now_h);
    return SW_OK;
}

int swcm_size(const swcm_cache* h) { return h ? (int)h->entries.size() : 0; }

int swcm_ids(const swcm_cache* h, uint64_t* out, int32_t cap) {
    if (!h) return SW_EINVAL;
    int n = 0;
    for (const auto& kv : h->entries) {
        if (n < cap) out[n] = kv.first;
        ++n;
    }
    return n;
}

// Ledger and arena reference the same entry-id set (CacheManager::check_consistent).
int swcm_check_consistent(const swcm_cache* h) {
    if (!h) return 0;
    if ((int64_t)h->entries.size() != sw_arena_entry_count(h->ctx)) return 0;
    for (const auto& kv : h->entries)
        if (!sw_arena_contains(h->ctx, kv.first)) return 0;
    return 1;
}

}  // extern "C"
