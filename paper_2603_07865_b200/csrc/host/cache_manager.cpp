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
#include "host_policy.hpp"

using swh::HostRng;
using swh::Entry;

int swcm_cache::refine(uint64_t id, HostRng& rng, swcm_regenerate_fn regen, void* user,
                       int32_t* replaced) {  // cache.cpp:107-140
    if (!regen || !replaced) return SW_EINVAL;
    swcm_cache* h = this;
    *replaced = 0;
    auto it = h->entries.find(id);
    if (it == h->entries.end()) return SW_WARN_UNKNOWN_ID;
    Entry& e = it->second;
    if (e.refinement_attempts >= h->cfg.refine_attempt_cap) return SW_OK;  // warn + no-op
    e.refinement_attempts++;
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
    std::vector<swh::Seg> segs;
    const int rc = h->write_rows(true, e.id, best_emb, e.duration_s,
                                 lat_cap && best_t > 0 ? best_lat.data() : nullptr, best_t, &segs);
    if (rc < 0) return rc;  // the ledger keeps the quality the arena still holds
    e.segs = std::move(segs);
    e.clip_embedding = best_emb;  // e.clip = best_clip; full_embedding = clip.embedding
    h->keep_clip_latent(e, lat_cap && best_t > 0 ? best_lat.data() : nullptr, best_t);
    e.quality = best_q;
    e.recent_skips.clear();
    *replaced = 1;
    return SW_OK;
}


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
    int rc = h->write_rows(false, e.id, full, duration_s, latent, t_src, &e.segs);
    if (rc < 0) return rc;  // nothing stored: the id is not consumed
    e.clip_embedding = full;
    h->keep_clip_latent(e, latent, t_src);
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
    HostRng rng(rng_seed);
    return h->refine(id, rng, regen, user, replaced);
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
