/* semwarm_b200 — C-ABI of the B200-native SoundWeaver warm-start path.
 *
 * This is the drop-in boundary: plain pointers and sizes, no C++ or torch types. Every entry
 * point names the reference interface it replaces (file:line under /root/reference/proj).
 * The reference has no FFI of its own; its boundary is the C++ class API of
 * include/semwarm/{index,selector,gater,cache}.hpp called by Pipeline (pipeline.cpp:91-297).
 * The C++ shim in paper_2603_07865_b200/csrc/host/semwarm_b200.hpp re-exposes those C++
 * signatures on top of this ABI; INTEGRATION.md shows the binding a maintainer adds.
 *
 * Conventions
 *  - Every function returns int: SW_OK (0), a negative error, or a positive soft warning
 *    (the reference's warn()-and-no-op cases). No exception crosses the ABI.
 *  - sw_last_error() returns a thread-local message for the last failing call.
 *  - "d_" arguments are device pointers; calls taking a `stream` are stream-ordered and
 *    asynchronous. "_host" variants take host pointers and return synchronously.
 *  - Readers (search/plan/align) may run concurrently; arena mutations are exclusive and
 *    synchronous, mirroring the shared/unique locks of pipeline.cpp:216,264,282.
 */
#ifndef SEMWARM_B200_H
#define SEMWARM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SW_OK 0
#define SW_EINVAL (-1)        /* std::invalid_argument in the reference */
#define SW_ERUNTIME (-2)      /* std::runtime_error */
#define SW_ECUDA (-3)         /* CUDA / driver failure */
#define SW_ENOMEM (-4)        /* arena or device memory exhausted */
#define SW_WARN_UNKNOWN_ID 1  /* warn("... unknown entry id") + no-op (index.cpp:243-245) */

/* sw_config.flags */
#define SW_FLAG_EXACT_ONLY 0x1u   /* never use the tcgen05 pre-filter: fp64 brute force only */
#define SW_FLAG_TC_ALWAYS 0x2u    /* tcgen05 pre-filter at any size (now the default; kept so
                                     callers that set it keep compiling) */
#define SW_FLAG_GROW 0x4u         /* inserts grow a full arena (capacity doubles) instead of
                                     failing — the unbounded IvfIndex the C++ adapter mirrors */

/* sw_choice.flags */
#define SW_CHOICE_AMBIGUOUS_DRAW 0x1u  /* never set: the device exp is glibc's, bit for bit, so
                                          every softmax draw is the reference's */
#define SW_CHOICE_NONFINITE_PHI 0x2u   /* non-finite features -> arm 0 (gater.cpp:71-76) */
#define SW_CHOICE_INCOMPLETE 0x4u      /* search not certified (never set: overflowing queries
                                          are re-searched exactly, see sw_overflow_stats) */
#define SW_CHOICE_AMBIGUOUS_ARM 0x8u   /* never set: explore-mode softplus uses glibc's exp and
                                          log1p restated bit for bit */

typedef struct sw_ctx sw_ctx;

/* Arena geometry. One context = one device-resident cache shard. */
typedef struct sw_config {
    int32_t dim;             /* embedding dimension D (EmbeddingVector::dim, core.hpp:15-24) */
    int32_t rows_per_entry;  /* max pyramid rows per entry (7 at delta=1/4, index.cpp:12-31) */
    int64_t max_entries;     /* entry capacity (CacheConfig::capacity, cache.hpp:33) */
    int32_t latent_c;        /* latent slot shape [C][T_max][F], fp32 (8 x 256 x 16) */
    int32_t latent_t_max;
    int32_t latent_f;
    int32_t max_batch;       /* largest B any batched call will pass */
    int64_t latent_slots;    /* 0 -> max_entries; fewer -> slot = entry_slot % latent_slots */
    double latent_fps;       /* latent frame rate (25 frames/s = 256 frames per 10.24 s) */
    uint32_t flags;          /* SW_FLAG_* */
    int32_t reserved;
} sw_config;

/* PyramidDescriptor (index.hpp:13-17) */
typedef struct sw_segment {
    int32_t level;
    int32_t reserved;
    double start_s;
    double length_s;
} sw_segment;

/* SearchHit (index.hpp:25-29) */
typedef struct sw_hit {
    uint64_t entry_id;
    sw_segment segment;
    double similarity;
} sw_hit;

/* SelectorConfig (selector.hpp:25-33); the negative embedding is set with sw_set_negative */
typedef struct sw_selector_config {
    int32_t top_k;
    int32_t reserved;
    double temperature;
    double quality_threshold;
} sw_selector_config;

/* SkipPolicy + its parameters (pipeline.hpp:17-22, 37-41) */
#define SW_POLICY_EXPLOIT 0
#define SW_POLICY_EXPLORE 1
#define SW_POLICY_RULE 2
#define SW_POLICY_FIXED 3
typedef struct sw_policy {
    int32_t kind;
    int32_t fixed_arm;
    double rule_similarity_threshold;
    double rule_skip_fraction;
} sw_policy;

/* GenerationRequest (core.hpp:45-51) minus the prompt, which travels as a B x D fp32 matrix */
typedef struct sw_request {
    uint64_t id;
    double duration_s;
    int32_t total_steps;
    int32_t reserved;
} sw_request;

/* Result of plan_request + pick_arm + t* (pipeline.cpp:91-202, simgen.cpp:70): the
 * ServeOutcome fields cache_hit, entry_id, arm_index, steps_skipped, reference_similarity
 * (core.hpp:54-67) plus the chosen segment and where its latent lives. */
typedef struct sw_choice {
    int32_t hit;
    int32_t arm;
    int32_t steps_skipped;
    int32_t n_hits;
    uint64_t entry_id;
    sw_segment segment;  /* the matched segment; segment.reserved = its pyramid row in the entry */
    double similarity;
    double skip_fraction;
    int32_t pick;    /* index of the chosen candidate in the top-k list, -1 on a miss */
    uint32_t flags;  /* SW_CHOICE_* */
    int32_t t_out;   /* aligned latent frames written by sw_align_noise (0 on a miss) */
    int32_t owner;   /* shard rank that owns the chosen entry */
    int64_t slot;    /* arena slot of the chosen entry on its owner shard */
} sw_choice;

/* Per-shard top-k record exchanged by the multi-GPU all-gather (128 bytes). */
#define SW_HIT_RECORD_BYTES 128

/* ---------------------------------------------------------------- context */
int sw_ctx_create(const sw_config* cfg, int device, sw_ctx** out);
int sw_ctx_destroy(sw_ctx* ctx);
const char* sw_last_error(void);
int sw_version(void);
/* Shape of a context: embedding dim, latent C / T_max / F (C = 0 without a latent arena),
 * max batch, CUDA device. Any output may be NULL. */
int sw_ctx_info(sw_ctx* ctx, int32_t* dim, int32_t* latent_c, int32_t* latent_t_max,
                int32_t* latent_f, int32_t* max_batch, int32_t* device);

/* SelectorConfig::negative_embedding (selector.hpp:31, make_negative_embedding selector.cpp:16-20).
 * Host pointer, D floats. Recomputes every stored row's s_neg. */
int sw_set_negative(sw_ctx* ctx, const float* neg);
/* BanditModel theta/psi/beta (gater.hpp:35-52), host pointers, 14 x feature_dim fp32 each. */
int sw_set_gater(sw_ctx* ctx, const float* theta, const float* psi, int32_t feature_dim,
                 double beta);
/* Forward-noising schedule abar[0..n-1] (fp64, abar[0] = 1). Default: scaled-linear
 * 0.00085..0.012 over 1000 DDPM steps. Index used: llround((T - t*) * (n-1) / T). */
int sw_set_schedule(sw_ctx* ctx, const double* abar, int32_t n);

/* ---------------------------------------------------------------- arena (Cache Manager data plane)
 * IvfIndex::insert (index.cpp:226-239) + the latent payload CacheManager::admit stores
 * (cache.cpp:30-52). rows: n_rows x D fp32 in pyramid order (level 0 first); segs: n_rows;
 * latent: C x t_src x F fp32 or NULL. Host pointers. Inserting an id that already exists
 * appends its rows (IvfIndex keeps per-entry counts, index.cpp:234-235). */
int sw_arena_insert(sw_ctx* ctx, uint64_t entry_id, int32_t n_rows, const float* rows,
                    const sw_segment* segs, const float* latent, int32_t t_src);
/* Bulk insert of n entries; entry e owns rows [row_off[e], row_off[e+1]). If src_on_device,
 * rows/segs/latents are device pointers (latents: n x C x t_src[e] x F packed at lat_off[e]). */
int sw_arena_insert_batch(sw_ctx* ctx, int64_t n, const uint64_t* ids, const int64_t* row_off,
                          const float* rows, const sw_segment* segs, const float* latents,
                          const int64_t* lat_off, const int32_t* t_src, int32_t src_on_device);
/* IvfIndex::remove (index.cpp:241-255): SW_WARN_UNKNOWN_ID for an unknown id. */
int sw_arena_remove(sw_ctx* ctx, uint64_t entry_id);
/* CacheManager::refine's re-index (cache.cpp:129-139): replace rows/latent of an entry in place. */
int sw_arena_replace(sw_ctx* ctx, uint64_t entry_id, int32_t n_rows, const float* rows,
                     const sw_segment* segs, const float* latent, int32_t t_src);
int64_t sw_arena_entry_count(const sw_ctx* ctx);  /* IvfIndex::entry_count (index.hpp:74) */
int sw_arena_contains(const sw_ctx* ctx, uint64_t entry_id); /* index.hpp:75 */
/* Entry slots the arena holds: max_entries + 1 (CacheManager::admit inserts before it evicts,
 * cache.cpp:30-52) rounded up to whole 256-row tiles. */
int64_t sw_arena_capacity(const sw_ctx* ctx);
/* Grows the arena to at least max_entries (+1 spare) entry slots, keeping every entry. */
int sw_arena_reserve(sw_ctx* ctx, int64_t max_entries);
/* IvfIndex::total_vectors (index.hpp:70): stored rows over all entries. */
int64_t sw_arena_row_count(const sw_ctx* ctx);
/* Host copy of `count` live entries starting at the first-th in slot order: ids, row counts,
 * and (if non-NULL) rows [count][rows_per_entry_pad][D] fp32 and segs [count][pad]. Returns the
 * number copied. For checkers and re-layouts; synchronous. */
int64_t sw_arena_export(sw_ctx* ctx, int64_t first, int64_t count, uint64_t* ids,
                        int32_t* nrows, float* rows, sw_segment* segs);
/* IvfIndex::check_consistent (index.cpp:334-343) + the arena bookkeeping: 1 if every stored row
 * is in exactly the list of its nearest centroid (recomputed on the device in fp64), per-entry
 * row counts match the index ledger and the validity flags match the id map, else 0. */
int sw_index_check_consistent(sw_ctx* ctx);
/* Benchmark fill: n entries with ids first_id.. of seeded iid unit rows generated on the
 * device (Philox normals, fp64 normalise, fp32 round), durations U[4,12] s, pyramid rows per
 * the context's rows_per_entry, latents N(0,1). Deterministic in seed. */
int sw_arena_fill_synthetic(sw_ctx* ctx, int64_t n, uint64_t first_id, uint64_t seed,
                            double delta);
/* Copy stored fp32 rows of an entry back to host (n_rows_cap x D); returns rows copied. */
int sw_arena_read_rows(sw_ctx* ctx, uint64_t entry_id, float* rows, int32_t n_rows_cap);

/* ---------------------------------------------------------------- IVF coarse quantiser
 * IvfIndex (index.hpp:47-101) in its reference-default mode (pipeline.cpp:28-31: 64 centroids,
 * nprobe 8, rebuild every 1024 mutations). Without sw_ivf_configure a context is in exhaustive
 * parity mode (one list). */
/* IvfIndex::build({}, centroids, seed, nprobe) + set_rebuild_interval (index.cpp:186-208).
 * Empty arena only. centroids < 1 -> SW_EINVAL (index.cpp:191); at most 256 lists. */
int sw_ivf_configure(sw_ctx* ctx, int32_t centroids, int32_t nprobe, uint64_t rebuild_interval,
                     uint64_t seed);
/* IvfIndex::set_rebuild_interval (index.hpp:76; pipeline.cpp:81). */
int sw_ivf_set_rebuild_interval(sw_ctx* ctx, uint64_t rebuild_interval);
/* The configuration sw_ivf_configure installed (target centroids, nprobe, interval, seed);
 * enabled = 0 for the exhaustive (parity) mode. */
int sw_ivf_config(sw_ctx* ctx, int32_t* enabled, int32_t* centroids, int32_t* nprobe,
                  uint64_t* rebuild_interval, uint64_t* seed);
/* IvfIndex::build(vecs, C, seed, nprobe) with non-empty vecs (index.cpp:186-208) on a configured,
 * empty arena: bulk-inserts the entries (no mutation counting), then k-means over the rows in
 * the given order with the configured seed itself; C is reduced to the row count. */
int sw_ivf_build(sw_ctx* ctx, int64_t n, const uint64_t* ids, const int64_t* row_off,
                 const float* rows, const sw_segment* segs);
/* IvfIndex::set_nprobe (index.hpp:74). */
int sw_ivf_set_nprobe(sw_ctx* ctx, int32_t nprobe);
/* IvfIndex::rebuild (index.cpp:257-283): k-means++ and Lloyd over every stored row in
 * (id, level, start) order with seed derive_seed(seed, ++rebuild_count), bit-identical to the
 * reference; dot products, member sums and reseeding searches run on the GPU. Also the bulk
 * path after sw_arena_fill_synthetic. */
int sw_ivf_rebuild(sw_ctx* ctx);
/* centroid_count() (index.hpp:69), mutations since the last rebuild, rebuild count. */
int sw_ivf_info(sw_ctx* ctx, int32_t* n_centroids, uint64_t* mutations, uint64_t* rebuilds);
/* Host copy of the centroids (C x D fp32); returns C. */
int sw_ivf_centroids(sw_ctx* ctx, float* centroids_out, int32_t cap);
/* Installs centroids (e.g. from a SWIX snapshot, index.cpp:345-408) and reassigns every stored
 * row to its nearest one. */
int sw_ivf_set_centroids(sw_ctx* ctx, const float* centroids, int32_t n_centroids);
/* The list of each of an entry's rows (test / debug); returns the row count. */
int sw_ivf_entry_lists(sw_ctx* ctx, uint64_t entry_id, int16_t* lists, int32_t cap);

/* ---------------------------------------------------------------- phase vocoder
 * time_stretch (vocoder.cpp:128-207; StftConfig{window, hop}, pipeline.hpp:36 uses {128, 32})
 * of B 1-D clips on the GPU, one CTA per clip. d_in: device, clip b = d_in[in_off[b] ..
 * + in_len[b]) at sample_rate; target_s[b] host. Outputs are packed into d_out (out_cap floats)
 * at out_off[b] (host, written), out_len[b] = llround(target_s * rate) samples. status[b]
 * (host): 0, or SW_EINVAL where the reference throws (empty clip, target <= 0, stretch ratio
 * outside [0.4, 2.5]). A bad window / hop fails the call with SW_EINVAL (StftConfig::validate).
 * Stream-ordered; host arrays may be reused once the call returns. */
/* Alignment used by sw_align_noise / sw_warmstart: SW_ALIGN_CROP_TILE (default; crop or tile
 * cyclically, the north-star definition) or SW_ALIGN_VOCODER — the reference's own alignment
 * (slice_clip + time_stretch{window, hop}, pipeline.cpp:158-169) applied to every latent channel
 * (c, f) at the latent frame rate, then the same forward noising. A request whose stretch ratio
 * leaves [0.4, 2.5] (where the reference throws and serves cold) keeps an untouched output. */
#define SW_ALIGN_CROP_TILE 0
#define SW_ALIGN_VOCODER 1
int sw_set_align_mode(sw_ctx* ctx, int32_t mode, int32_t window, int32_t hop);
int sw_time_stretch(const float* d_in, const int64_t* in_off, const int32_t* in_len, int32_t B,
                    int32_t sample_rate, const double* target_s, int32_t window, int32_t hop,
                    float* d_out, int64_t out_cap, int64_t* out_off, int32_t* out_len,
                    int32_t* status, void* stream);

/* ---------------------------------------------------------------- request batching (§8f)
 * Aggregates concurrent single-request callers (the reference's per-connection
 * Pipeline::handle_request, server.cpp:83,149) into device batches. swb_submit is thread-safe
 * and blocks until its request's batch has run; a worker takes up to max_batch queued requests,
 * waiting at most max_wait_us after the oldest for the batch to fill. Results equal one sw_plan
 * (or sw_warmstart) over the same requests: draws and noise are keyed by request id. latent
 * (optional, C x t_out_max x F floats) receives the aligned + noised latent when the batcher was
 * created with_latent. */
typedef struct swb_batcher swb_batcher;
int swb_create(sw_ctx* ctx, int32_t max_batch, int32_t max_wait_us, uint64_t seed,
               const sw_selector_config* sel, const sw_policy* policy, uint64_t philox_seed,
               int32_t t_out_max, int32_t with_latent, swb_batcher** out);
int swb_destroy(swb_batcher* b);
int swb_submit(swb_batcher* b, const float* prompt, const sw_request* req, sw_choice* choice,
               float* latent);
int swb_stats(swb_batcher* b, int64_t* batches, int64_t* requests);
/* Native load generator (measurement): `clients` threads each submit `per_client` blocking
 * requests drawn round-robin from the n prompts / requests (ids first_id, first_id + 1, ...);
 * reports wall-clock requests/s, p50 / p99 latency and the mean device batch. */
int swb_load_test(swb_batcher* b, const float* prompts, const sw_request* reqs, int32_t n,
                  int32_t clients, int32_t per_client, uint64_t first_id, double* req_per_s,
                  double* p50_ms, double* p99_ms, double* mean_batch);

/* ---------------------------------------------------------------- snapshots
 * IvfIndex::load (index.cpp:371-406) straight into an EMPTY context's device arena: entries,
 * centroids, nprobe and every row's stored list; the context switches to IVF mode. Malformed
 * files -> SW_ERUNTIME (the reference throws std::runtime_error). */
int sw_swix_load(sw_ctx* ctx, const char* path);
/* IvfIndex::save (index.cpp:347-369) of the context's index; rows inside a list in rebuild
 * order (id, level, start). */
int sw_swix_save(sw_ctx* ctx, const char* path);
/* BanditModel::load / save (gater.cpp:277-306, "SWMB"): the Skip Gater's theta / psi straight
 * into (out of) the context's device-resident gater; beta is GaterConfig's (not in the file). */
int sw_gater_load_swmb(sw_ctx* ctx, const char* path, double beta);
int sw_gater_save_swmb(sw_ctx* ctx, const char* path);
/* load_embeddings (core.cpp:201-220): reads a SWEM file into `out` (up to cap floats); returns
 * count * dim and the shape, or a negative status. */
int64_t sw_swem_read(const char* path, float* out, int64_t cap_floats, int32_t* count,
                     int32_t* dim);

/* ---------------------------------------------------------------- batched hot path
 * IvfIndex::search (index.cpp:289-326) in exhaustive mode for B queries: exact fp64 cosine,
 * best segment per entry, (sim desc, id asc), truncated to k. d_out: B x k, d_n: B. Always
 * certified: queries whose tcgen05 candidate slices overflow are re-searched by exact brute
 * force on the device. (A negative d_n[b] = -n - 1 would flag an uncertified result;
 * sw_search_host turns it into SW_ERUNTIME.) */
int sw_search(sw_ctx* ctx, const float* d_queries, int32_t B, int32_t k, sw_hit* d_out,
              int32_t* d_n, void* stream);
int sw_search_host(sw_ctx* ctx, const float* queries, int32_t B, int32_t k, sw_hit* out,
                   int32_t* n);
/* IvfIndex::search(q, k, nprobe) (index.hpp:67): nprobe > 0 overrides the index's nprobe for
 * this call (0: the index's own). Host buffers, synchronous, no allocation per call. */
int sw_search_host_ex(sw_ctx* ctx, const float* queries, int32_t B, int32_t k, int32_t nprobe,
                      sw_hit* out, int32_t* n);

/* Pipeline::plan_request + pick_arm + t* (pipeline.cpp:91-202, simgen.cpp:70) for B requests:
 * search -> score_candidates -> select (Rng(derive_seed(seed, id, 2)), pipeline.cpp:211) ->
 * context_features -> choose_arm / rule / fixed -> steps_skipped = llround(0.05 arm T). */
int sw_plan(sw_ctx* ctx, const float* d_queries, const sw_request* d_reqs, int32_t B,
            uint64_t seed, const sw_selector_config* sel, const sw_policy* pol,
            sw_choice* d_out, void* stream);

/* Temporal alignment of the chosen cached latent to the request (crop / tile cyclically along
 * T, slice_clip frame math simgen.cpp:113-128) fused with forward noising
 * x_t = sqrt(abar)*x0 + sqrt(1-abar)*eps. d_eps: B x C x t_out_max x F, or NULL for Philox
 * noise keyed by (philox_seed, request id). d_out: B x C x t_out_max x F. Misses untouched. */
int sw_align_noise(sw_ctx* ctx, const sw_choice* d_choices, const sw_request* d_reqs,
                   int32_t B, const float* d_eps, uint64_t philox_seed, float* d_out,
                   int32_t t_out_max, void* stream);

/* plan + align_noise in one stream-ordered call (the whole warm-start path). */
int sw_warmstart(sw_ctx* ctx, const float* d_queries, const sw_request* d_reqs, int32_t B,
                 uint64_t seed, const sw_selector_config* sel, const sw_policy* pol,
                 const float* d_eps, uint64_t philox_seed, sw_choice* d_choices, float* d_out,
                 int32_t t_out_max, void* stream);
/* Cross-batch pipelined sw_warmstart: prep + scoring of this batch on `stream`, its finish
 * (filter, exact rescoring, top-k, gate, select, gater) and align + noise on the context's
 * own stream, so they run under the NEXT call's scoring kernel. d_choices and d_out are
 * complete, and d_queries / d_reqs / d_eps may be reused, once sw_join(ctx, s) has been
 * enqueued on a stream s and s reached that point. Results are identical to sw_warmstart's,
 * in exhaustive and IVF mode. */
int sw_warmstart_async(sw_ctx* ctx, const float* d_queries, const sw_request* d_reqs, int32_t B,
                       uint64_t seed, const sw_selector_config* sel, const sw_policy* pol,
                       const float* d_eps, uint64_t philox_seed, sw_choice* d_choices,
                       float* d_out, int32_t t_out_max, void* stream);
/* Makes `stream` wait for every sw_warmstart_async enqueued so far. */
int sw_join(sw_ctx* ctx, void* stream);
/* End-to-end from host buffers (pinned or pageable): H2D prompts+requests, warm start,
 * D2H choices; the noised latents stay on the device in d_out. Synchronous. */
int sw_warmstart_host(sw_ctx* ctx, const float* queries, const sw_request* reqs, int32_t B,
                      uint64_t seed, const sw_selector_config* sel, const sw_policy* pol,
                      uint64_t philox_seed, sw_choice* choices, float* d_out,
                      int32_t t_out_max, void* stream);
/* Pipelined form of sw_warmstart_host for serving loops: enqueues the H2D copies (own copy
 * stream), the plan (on `stream`), the align + noise (the context's align stream, so it runs
 * under the next batch's scoring kernel) and the D2H of the choices (own copy stream), and
 * returns a ticket at once; sw_warmstart_host_wait(ticket) blocks until `choices` has landed
 * and `d_out` is written. Up to three submissions are in flight; `queries`, `reqs` and
 * `choices` must
 * stay valid (and should be pinned) until the wait returns. Results are identical to
 * sw_warmstart_host's. */
int sw_warmstart_host_submit(sw_ctx* ctx, const float* queries, const sw_request* reqs,
                             int32_t B, uint64_t seed, const sw_selector_config* sel,
                             const sw_policy* pol, uint64_t philox_seed, sw_choice* choices,
                             float* d_out, int32_t t_out_max, void* stream, int64_t* ticket);
int sw_warmstart_host_wait(sw_ctx* ctx, int64_t ticket);

/* ---------------------------------------------------------------- multi-GPU (entry-sharded)
 * Per-shard top-k records for the all-gather: B x k records of SW_HIT_RECORD_BYTES plus a
 * count per query. `rank` is stamped into each record. */
int sw_local_topk(sw_ctx* ctx, const float* d_queries, int32_t B, int32_t k, int32_t rank,
                  void* d_records, int32_t* d_n, void* stream);
/* Deterministic merge of world x (B x k) gathered records (sim desc, id asc) followed by
 * score_candidates / select / gater / t* (replicated on every rank; no broadcast needed). */
/* Pipelined sw_local_topk: prep + scoring on `stream`; the finish and the record copies on the
 * context's async stream (sw_async_stream), where the caller also enqueues the all-gather,
 * sw_merge_select and sw_align_noise_owned of the same batch — they then overlap the next
 * batch's scoring. sw_join closes the pipeline. */
int sw_local_topk_async(sw_ctx* ctx, const float* d_queries, int32_t B, int32_t k, int32_t rank,
                        void* d_records, int32_t* d_n, void* stream);
int sw_async_stream(sw_ctx* ctx, void** stream);
int sw_merge_select(sw_ctx* ctx, const void* d_gathered, const int32_t* d_gathered_n,
                    int32_t world, const float* d_queries, const sw_request* d_reqs, int32_t B,
                    int32_t k, uint64_t seed, const sw_selector_config* sel,
                    const sw_policy* pol, sw_choice* d_out, void* stream);
/* Owner-computes alignment: only requests whose chosen entry has owner == rank are written. */
int sw_align_noise_owned(sw_ctx* ctx, const sw_choice* d_choices, const sw_request* d_reqs,
                         int32_t B, int32_t rank, const float* d_eps, uint64_t philox_seed,
                         float* d_out, int32_t t_out_max, void* stream);

/* In-library sharding over the GPUs of one process (no torch): a group owns one context per
 * shard and runs sw_local_topk -> all-gather -> sw_merge_select -> sw_align_noise_owned on every
 * shard's stream. The all-gather is NCCL (ncclCommInitAll + ncclAllGather over NVLink, libnccl
 * opened at run time) when every shard has its own device, or peer copies (cudaMemcpyPeerAsync)
 * when shards share a device. Entries are placed by id mod n_shards (sw_group_insert) or
 * directly through sw_group_shard. Replaces the N-way fan-out of IvfIndex::search
 * (index.cpp:289-326) + plan_request (pipeline.cpp:91-202) of BASELINE config 4. */
#define SW_GROUP_TRANSPORT_AUTO 0  /* NCCL if all devices differ (and N > 1), else COPY */
#define SW_GROUP_TRANSPORT_NCCL 1
#define SW_GROUP_TRANSPORT_COPY 2
typedef struct sw_group sw_group;
int sw_group_create(const sw_config* cfg, int32_t n_shards, const int32_t* devices,
                    int32_t transport, sw_group** out);
int sw_group_destroy(sw_group* g);
int sw_group_info(sw_group* g, int32_t* n_shards, int32_t* transport);
int sw_group_shard(sw_group* g, int32_t shard, sw_ctx** ctx);
int32_t sw_group_owner(sw_group* g, uint64_t entry_id);
int sw_group_insert(sw_group* g, uint64_t entry_id, int32_t n_rows, const float* rows,
                    const sw_segment* segs, const float* latent, int32_t t_src);
int sw_group_remove(sw_group* g, uint64_t entry_id);
int sw_group_set_negative(sw_group* g, const float* neg);
int sw_group_set_gater(sw_group* g, const float* theta, const float* psi, int32_t feature_dim,
                       double beta);
/* One batch from host prompts/requests: choices (identical on every shard) come back in
 * h_choices; d_out[s] (optional, on shard s's device, B x C x t_out_max x F) receives the
 * aligned + noised latents of the requests whose chosen entry shard s owns. Synchronous. */
int sw_group_warmstart_host(sw_group* g, const float* h_queries, const sw_request* h_reqs,
                            int32_t B, uint64_t seed, const sw_selector_config* sel,
                            const sw_policy* pol, uint64_t philox_seed, sw_choice* h_choices,
                            float* const* d_out, int32_t t_out_max);
/* The choices shard `shard` computed in the last batch (the replicated merge, for checks). */
int sw_group_shard_choices(sw_group* g, int32_t shard, int32_t B, sw_choice* h_choices);

/* ---------------------------------------------------------------- component entry points
 * score_candidates + select (selector.cpp:24-85) on one explicit candidate set, evaluated by
 * the same device code the batched path uses. Outputs n x {s_pos,s_neg,a,b,q} and the pick. */
int sw_score_select_host(sw_ctx* ctx, int32_t n, const double* sims, const double* s_neg,
                         const double* durations, double L, const sw_selector_config* sel,
                         uint64_t rng_seed, double* scores_out, int32_t* pick);
/* score_candidates (selector.cpp:24-58) alone: n <= 32 candidates with their index similarity,
 * matched-segment embedding (n x dim) and duration; s_neg = clamp01(cos(audio, negative)) with
 * `negative` (dim floats) or, if NULL, the context's negative embedding. Writes n x {s_pos,
 * s_neg, a, b, q}. */
int sw_score_candidates_host(sw_ctx* ctx, int32_t n, int32_t dim, const double* sims,
                             const float* audio, const double* durations, double L,
                             const float* negative, double* scores_out);
/* select (selector.cpp:60-85) alone, given the gate scores and the caller's draw
 * u = rng.uniform() (a caller draws it only when some q >= threshold, as the reference does).
 * *pick = chosen index or -1; *flags = SW_CHOICE_AMBIGUOUS_DRAW if the cumulative weight lands
 * within exp()'s ulp slack of the target. */
int sw_select_host(sw_ctx* ctx, int32_t n, const double* s_pos, const double* q,
                   double temperature, double threshold, double u, int32_t* pick,
                   uint32_t* flags);
/* context_features + choose_arm (gater.cpp:13-92) for B (prompt, segment) pairs. */
int sw_gater_host(sw_ctx* ctx, const float* prompts, const float* segs, const int32_t* T,
                  int32_t B, int32_t explore, double* phi_out, int32_t* arm_out);
/* Stage profiling with CUDA events recorded on the launching stream around every kernel of the
 * hot path (no host sync while enabled). Stages: SW_STAGE_*. sw_profile_read synchronizes the
 * recorded events and returns the summed device time and launch count of one stage. */
#define SW_STAGE_PREP 0      /* queries -> bf16, |q| */
#define SW_STAGE_SCORE_TC 1  /* tcgen05 scoring + certified candidate emission */
#define SW_STAGE_FINISH 2    /* candidate filter + fp64 rescoring + top-k (+ select) */
#define SW_STAGE_SELECT 3    /* standalone select (multi-GPU merge path) */
#define SW_STAGE_ALIGN 4     /* align + noise */
#define SW_STAGE_MERGE 5     /* multi-GPU record merge */
#define SW_STAGE_ALIGN_GEOM 6 /* per-request align geometry (the pre-pass of align + noise) */
#define SW_NUM_STAGES 7
/* on: 0 off, 1 every stage, SW_PROFILE_MASK | (1 << stage) | ... only the listed stages */
#define SW_PROFILE_MASK 0x100
int sw_profile_enable(sw_ctx* ctx, int32_t on);
int sw_profile_reset(sw_ctx* ctx);
int sw_profile_read(sw_ctx* ctx, int32_t stage, double* total_ms, int64_t* launches);
/* Per-query statistics of the last search/plan (B x 8 int32): emitted candidates, certified
 * candidates rescored, then device clock cycles of the finish phases (filter, rescore, top-k +
 * enrichment, select). Synchronizes the device. */
int sw_debug_query_stats(sw_ctx* ctx, int32_t B, int32_t* stats);
/* Launch statistics of the last sw_plan/sw_search on this context (kernels launched; scoring
 * mode: 0 exact fp64 only, 1 tcgen05 single CTAs, 2 tcgen05 CTA pairs (cta_group::2), 3 CTA
 * pairs with the queries resident in TMEM). */
int sw_last_launch_info(const sw_ctx* ctx, int32_t* kernels, int32_t* used_tensor_cores,
                        int32_t* candidates_max);
/* Queries so far whose tcgen05 candidate slices overflowed and that the certified fallback (an
 * exact fp64 brute-force IvfIndex::search of the whole arena) answered instead. Results are
 * exact either way; this counts how often the slow path ran. Synchronizes the device. */
int sw_overflow_stats(sw_ctx* ctx, int64_t* fallback_queries);

/* ---------------------------------------------------------------- Cache Manager (host policy)
 * CacheManager (cache.hpp:45-106) over a context's arena: the policy stays on the host exactly
 * as in the reference; admit / evict / refine land in the arena through sw_arena_*. */
typedef struct swcm_cache swcm_cache;
typedef struct swcm_config { /* CacheConfig (cache.hpp:31-42) */
    uint64_t capacity;
    double decay_per_hour;
    double grace_hours;
    double quality_floor;
    double pyramid_delta;
    uint64_t embedding_seed;  /* derive_seed(seed, "SEGM") in the reference (pipeline.cpp:76-78) */
    int32_t refine_regenerations;
    int32_t refine_attempt_cap;
    int32_t refine_window;
    int32_t reserved;
    double refine_skip_threshold;
    int64_t latent_capacity;  /* floats the regenerate callback may write (0: no latents) */
} swcm_config;
/* RegenerateFn (cache.hpp:47-49): fill embedding (dim floats), quality, optional latent. */
typedef int (*swcm_regenerate_fn)(void* user, const float* prompt, int32_t dim, double duration_s,
                                  uint64_t seed, float* embedding_out, double* quality_out,
                                  float* latent_out, int32_t* t_src_out);
int swcm_create(sw_ctx* ctx, int32_t dim, const swcm_config* cfg, swcm_cache** out);
int swcm_destroy(swcm_cache* cache);
/* CacheManager::admit (cache.cpp:30-52): returns 1 admitted (*id_out set), 0 rejected. */
int swcm_admit(swcm_cache* cache, const float* clip_embedding, double duration_s,
               const float* prompt_embedding, double quality, double now_h, const float* latent,
               int32_t t_src, uint64_t* id_out);
int swcm_last_evicted(const swcm_cache* cache, uint64_t* out, int32_t cap);
/* CacheManager::record_reuse (cache.cpp:54-68) */
int swcm_record_reuse(swcm_cache* cache, uint64_t entry_id, int32_t steps_skipped,
                      double duration_s, double now_h, double skip_fraction);
/* CacheManager::evict_if_full (cache.cpp:70-105): returns the number evicted */
int swcm_evict_if_full(swcm_cache* cache, double now_h, uint64_t* out, int32_t cap);
/* CacheManager::refinement_candidates (cache.cpp:142-154) */
int swcm_refinement_candidates(const swcm_cache* cache, uint64_t* out, int32_t cap);
/* CacheManager::refine (cache.cpp:107-140) with Rng(rng_seed); *replaced = 1 if the stored
 * entry was replaced. SW_WARN_UNKNOWN_ID for an unknown id (warn + no-op). */
int swcm_refine(swcm_cache* cache, uint64_t entry_id, uint64_t rng_seed, swcm_regenerate_fn regen,
                void* user, int32_t* replaced);
int swcm_importance(const swcm_cache* cache, uint64_t entry_id, double now_h, double* out);
int swcm_size(const swcm_cache* cache);
int swcm_ids(const swcm_cache* cache, uint64_t* out, int32_t cap);
int swcm_check_consistent(const swcm_cache* cache);
/* CacheManager::save_snapshot / load_snapshot (cache.cpp:211-295): manifest.jsonl + <id>.emb
 * (SWEM) + <id>.clip (SWSC). Load replaces the ledger, re-creates the index with the context's
 * IVF configuration and inserts every entry's stored segment rows in ascending id order straight
 * into the device arena (the SimClip latent into its slot when slots are [1][T][1]); save reads
 * the rows back from the arena. Files are interchangeable with the reference's. */
int swcm_save_snapshot(const swcm_cache* cache, const char* dir);
int swcm_load_snapshot(swcm_cache* cache, const char* dir);

/* ---------------------------------------------------------------- trace replay (config 5)
 * WorkloadConfig (simgen.hpp:87-98). */
typedef struct swr_workload {
    int64_t n_prompts;
    int32_t cluster_count;
    int32_t dim;
    double near_duplicate_rate;
    double cluster_perturbation;
    double duplicate_perturbation;
    double duration_lo_s;
    double duration_hi_s;
    double arrival_rate_hz;
    int32_t total_steps;
    int32_t reserved;
} swr_workload;
/* synth_workload (simgen.cpp:162-194), bit-identical for the same seed: request i (id i + 1)
 * gets prompts[i * dim ..], durations[i], arrivals[i] (s) and total_steps[i]. */
int swr_synth_workload(const swr_workload* cfg, uint64_t seed, float* prompts, double* durations,
                       double* arrivals, int32_t* total_steps);

/* make_negative_embedding (selector.cpp:16-20): the fixed seeded negative reference of `dim`. */
int sw_negative_embedding(int32_t dim, float* out);

/* The PipelineConfig fields a replay uses (pipeline.hpp:24-51) plus the lookup batch size. */
typedef struct swr_config {
    uint64_t seed;                   /* PipelineConfig::seed */
    sw_selector_config selector;
    sw_policy policy;
    double q_max;                    /* QualityModel (simgen.hpp:27-31) */
    double penalty_slope;
    double noise_scale;
    double skip_headroom;
    double step_time_s_per_10s;      /* SimGenConfig */
    double alpha;                    /* BanditModel::alpha (the reward's trade-off) */
    int32_t latent_rate;
    int32_t default_total_steps;
    int32_t refinement_enabled;
    int32_t batch;                   /* lookups per device batch; 1 = Pipeline::replay exactly */
} swr_config;

/* ServeOutcome (core.hpp:54-67); entry ids 0 = none. */
typedef struct swr_outcome {
    uint64_t request_id;
    int32_t cache_hit;
    int32_t arm_index;
    int32_t steps_skipped;
    int32_t fallback;
    uint64_t entry_id;
    uint64_t admitted_entry_id;
    double quality;
    double nfe_cost_s;
    double sim_latency_s;
    double skip_fraction;
    double reference_similarity;
} swr_outcome;

/* RunReport's summary (pipeline.hpp:53-68) + wall-clock split of the replay. */
typedef struct swr_stats {
    double total_s;         /* wall time of the whole replay */
    double lookup_s;        /* batched sw_plan + segment-row gather + D2H */
    double mutation_s;      /* generate + record_reuse + admit (+ evictions), per request */
    double maintenance_s;   /* refinement_candidates + refine, after every request */
    int64_t batches, lookups, admits, evictions, refinements, reuses;
    double total_nfe_s, baseline_nfe_s, speedup, mean_quality, mean_reward, hit_rate;
    double mean_latency_s, median_latency_s, p95_latency_s;
} swr_stats;

/* Pipeline::replay (pipeline.cpp:299-323) over a warm-start context + Cache Manager, with the
 * lookups of `batch` consecutive requests planned in one sw_plan against the cache as it stands
 * when the batch starts; mutations (simulated generate, record_reuse, admit + evict)
 * and run_maintenance (refine with the pipeline's maintenance RNG, pipeline.cpp:70,280-297) follow
 * per request, in order. The context must hold the cache's embedding arena (IVF configured as
 * the pipeline's index), the negative embedding and the gater; out: n outcomes. */
int swr_replay(sw_ctx* ctx, swcm_cache* cache, const swr_config* cfg, int64_t n,
               const float* prompts, const double* durations, const double* arrivals,
               const int32_t* total_steps, swr_outcome* out, swr_stats* stats);

/* Device gather of each chosen segment row (slot, segment.reserved) of B choices into
 * d_rows (B x dim fp32; misses zero-filled). Stream-ordered. */
int sw_choice_rows(sw_ctx* ctx, const sw_choice* d_choices, int32_t B, float* d_rows,
                   void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SEMWARM_B200_H */
