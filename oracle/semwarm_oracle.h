/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the SoundWeaver warm-start path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this. It is the
 * checker, never the product: the product path is paper_2603_07865_b200/libsemwarm_b200.so.
 *
 * Every function cites the reference file:line it restates (/root/reference/proj/...). The
 * restatement is pinned against the compiled reference (oracle/_ref/libsemwarm_ref.so) by
 * tests/test_oracle_pinning.py and against committed golden vectors (tests/golden/).
 * Exception: so_align_noise / so_philox_normals restate OUR definition of crop/tile/pad + forward
 * noising, which the reference does not have — parity there is unpinned by the
 * reference and pinned only by our own known-answer tests.
 */
#ifndef SEMWARM_ORACLE_H
#define SEMWARM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

uint64_t so_splitmix64(uint64_t x);                                       /* core.cpp:58-63 */
uint64_t so_derive_seed(uint64_t base, uint64_t a, uint64_t b, uint64_t c); /* core.cpp:65-71 */
uint64_t so_mt64_first(uint64_t seed);    /* first output of std::mt19937_64(seed), core.hpp:80 */
double so_uniform_first(uint64_t seed);   /* Rng::uniform, core.hpp:83 */
double so_dot(const float* a, const float* b, int dim);    /* core.cpp:21-31 */
double so_cosine(const float* a, const float* b, int dim); /* core.cpp:33-38 */
int so_pyramid_segments(double duration, double delta, int* levels, double* starts,
                        double* lengths, int cap);         /* index.cpp:12-31 */

/* Arena view of a cache: entry e owns rows [off[e], off[e+1]) in pyramid (list) order. */
typedef struct {
    int dim;
    int n_entries;
    const uint64_t* ids;
    const int64_t* off;
    const float* rows;
    const int* levels;
    const double* starts;
    const double* lengths;
} so_arena;

typedef struct {
    uint64_t entry_id;
    int32_t level;
    int32_t row; /* absolute row index of the winning segment */
    double start_s;
    double length_s;
    double similarity;
} so_hit;

/* Exhaustive IvfIndex::search (index.cpp:289-326 with nprobe >= C): per-entry best segment by
 * strict '>' in list order, sort (sim desc, id asc), truncate to k. Returns hit count. */
int so_search(const so_arena* ar, const float* q, int k, so_hit* out);

/* score_candidates + select (selector.cpp:24-85). s_neg rows are given directly.
 * Returns the picked index or -1. Writes the CandidateScore fields. */
int so_score_select(int n, const double* sims, const double* durations, const float* audio,
                    int dim, const float* neg, double L, double temp, double thr,
                    uint64_t rng_seed, double* s_pos, double* s_neg, double* a, double* b,
                    double* q);

void so_context_features(const float* prompt, const float* cache, int dim, int T,
                         double* phi); /* gater.cpp:13-30 */
int so_choose_arm(const float* theta, const float* psi, int fd, double beta, const double* phi,
                  int explore);        /* gater.cpp:52-92 */

typedef struct {
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
} so_plan; /* same layout as RefPlanOut in ref_harness.cpp */

/* plan_request + pick_arm + t* for a batch (pipeline.cpp:91-202, simgen.cpp:70).
 * policy: 0 exploit, 1 explore, 2 rule, 3 fixed. */
int so_plan_batch(const so_arena* ar, const float* neg, int B, const float* queries,
                  const double* L, const uint64_t* req_ids, const int* T, uint64_t seed,
                  int top_k, double temp, double thr, int policy, const float* theta,
                  const float* psi, int fd, double beta, double rule_thr, int rule_arm,
                  int fixed_arm, int nthreads, so_plan* out, so_hit* hits_out);

/* ---- our align + noise definition (no reference counterpart) ---- */
void so_philox4x32_r(const uint32_t ctr[4], const uint32_t key[2], int rounds, uint32_t out[4]);
void so_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* glibc 2.39 exp (FMA build), restated op for op (the reference's std::exp). */
double so_ref_exp(double x);
void so_exp_pair(const double* x, int64_t n, double* ours, double* lib);
/* glibc 2.39 log1p (FMA build), restated op for op (explore-mode softplus). */
double so_ref_log1p(double x);
void so_log1p_pair(const double* x, int64_t n, double* ours, double* lib);
/* The normal transform of each 32-bit word. */
void so_icdf_normals(const uint32_t* words, int64_t n, float* out);
/* n standard normals for (seed, request_id), element i from Philox4x32-7 counter (i/4, rid). */
void so_philox_normals(uint64_t seed, uint64_t request_id, int64_t n, float* out);
/* x_t[c][t][f] = fmaf(s1, eps, s0 * x0[c][lo + t mod T_seg][f]), t < T_out = llround(L*fps).
 * eps == NULL -> Philox normals (seed, request_id). Returns T_out. */
int so_align_noise(const float* latent, int C, int t_src, int F, double start_s,
                   double length_s, double L, double fps, double abar, const float* eps,
                   uint64_t philox_seed, uint64_t request_id, float* out);
/* default DDPM schedule: scaled-linear betas 0.00085..0.012 over 1000 steps, abar[0] = 1 */
void so_abar_table(double* abar /* 1001 */);
int so_abar_index(int total_steps, int steps_skipped); /* llround((T - S) * 1000 / T) */

#ifdef __cplusplus
}
#endif
#endif
