// Host-side restatements shared by the Cache Manager policy (cache_manager.cpp) and the
// trace-replay driver (replay.cpp): the reference's seeding and RNG (core.cpp:58-124,
// core.hpp:75-93), normalisation, pyramid segments and segment-embedding derivation
// (index.cpp:12-46), and the host ledger of the Cache Manager (cache.hpp:16-43). Everything
// that reaches the device arena goes through the C-ABI.
#pragma once
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

namespace swh {

// ---- core.cpp:58-124 (seeding, Rng::uniform/normal, normalize, random_unit_vector)
inline uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
inline uint64_t derive_seed(uint64_t base, uint64_t a, uint64_t b = 0, uint64_t c = 0) {
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
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    uint64_t uniform_int(uint64_t n) {  // rejection sampling (core.cpp:73-82)
        const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
        uint64_t x;
        do {
            x = gen_();
        } while (x >= limit);
        return x % n;
    }
    double exponential(double rate) {  // core.cpp:102-108
        double u;
        do {
            u = uniform();
        } while (u <= 0.0);
        return -std::log(u) / rate;
    }
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

inline std::vector<float> normalize(const std::vector<float>& raw) {  // core.cpp:40-52
    double s = 0.0;
    for (float v : raw) s += static_cast<double>(v) * v;
    const double n = std::sqrt(s);
    std::vector<float> out(raw.size());
    for (size_t i = 0; i < raw.size(); ++i) out[i] = static_cast<float>(raw[i] / n);
    return out;
}

inline std::vector<float> random_unit_vector(size_t dim, HostRng& rng) {  // core.cpp:110-114
    std::vector<float> v(dim);
    for (size_t i = 0; i < dim; ++i) v[i] = static_cast<float>(rng.normal());
    return normalize(v);
}

// perturb (core.cpp:116-124): normalize(v + scale * g), g a random unit vector
inline std::vector<float> perturb(const std::vector<float>& v, double scale, HostRng& rng) {
    if (scale == 0.0) return normalize(v);
    const std::vector<float> g = random_unit_vector(v.size(), rng);
    std::vector<float> out(v.size());
    for (size_t i = 0; i < v.size(); ++i) out[i] = static_cast<float>(v[i] + scale * g[i]);
    return normalize(out);
}

struct Seg {
    int level;
    double start, length;
};

// pyramid_segments (index.cpp:12-31)
inline std::vector<Seg> pyramid_segments(double duration, double delta) {
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
inline std::vector<float> segment_embedding(const std::vector<float>& full, uint64_t id, const Seg& s,
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
    // what the directory snapshot (cache.cpp:211-295) carries beyond the policy ledger: the
    // segments of the stored rows (the rows themselves live in the device arena), and the
    // SimClip payload (simgen.hpp:13-20) — its embedding is the entry's full embedding
    std::vector<Seg> segs;
    std::vector<float> clip_embedding;
    std::vector<float> clip_latent;
    int latent_rate = 200;
    uint64_t clip_seed = 0;
    double clip_skip = 0.0;
};

}  // namespace swh

struct swcm_cache {
    using Entry = swh::Entry;
    using Seg = swh::Seg;
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
                   const float* latent, int t_src, std::vector<Seg>* segs_out = nullptr) {
        const std::vector<Seg> segs = swh::pyramid_segments(duration, cfg.pyramid_delta);
        if (segs_out) *segs_out = segs;
        std::vector<float> rows;
        std::vector<sw_segment> ss;
        for (const Seg& s : segs) {
            const std::vector<float> v = swh::segment_embedding(full, id, s, cfg.embedding_seed);
            rows.insert(rows.end(), v.begin(), v.end());
            ss.push_back(sw_segment{s.level, 0, s.start, s.length});
        }
        return replace ? sw_arena_replace(ctx, id, (int32_t)segs.size(), rows.data(), ss.data(),
                                          latent, t_src)
                       : sw_arena_insert(ctx, id, (int32_t)segs.size(), rows.data(), ss.data(),
                                         latent, t_src);
    }

    // A context whose latent slots are [1][T][1] stores the reference's 1-D SimClip latent
    // (simgen.hpp:14) as is; the host copy is what a directory snapshot writes back.
    bool latent_1d() const {
        int32_t d = 0, lc = 0, lt = 0, lf = 0, mb = 0, dev = 0;
        return sw_ctx_info(ctx, &d, &lc, &lt, &lf, &mb, &dev) == SW_OK && lc == 1 && lf == 1;
    }
    void keep_clip_latent(Entry& e, const float* latent, int t_src) const {
        if (latent && t_src > 0 && latent_1d()) e.clip_latent.assign(latent, latent + t_src);
        else e.clip_latent.clear();
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

    // CacheManager::refine (cache.cpp:107-140) drawing its regeneration seeds from `rng` (the
    // Pipeline's maintenance_rng_, pipeline.cpp:283-296, or a per-call Rng)
    int refine(uint64_t id, swh::HostRng& rng, swcm_regenerate_fn regen, void* user,
               int32_t* replaced);
};

