/* TEST INFRASTRUCTURE ONLY — see semwarm_oracle.h. Plain-C restatement of the reference
 * warm-start path; built with -ffp-contract=off so no FMA changes a rounding. */
#define _GNU_SOURCE
#include "semwarm_oracle.h"
/* the segment table of the noise definition and glibc exp's 2^(k/128) table (shared
 * constants, not code) */
#include "noise_table.h"
#include "exp_table.h"
#include "noise_def.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ seeding (core.cpp:58-71) */
uint64_t so_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

uint64_t so_derive_seed(uint64_t base, uint64_t a, uint64_t b, uint64_t c) {
    uint64_t s = so_splitmix64(base ^ 0x53454d5741524dULL); /* "SEMWARM" */
    s = so_splitmix64(s ^ a);
    s = so_splitmix64(s ^ b);
    return so_splitmix64(s ^ c);
}

/* First output of std::mt19937_64 seeded with `seed` (the engine behind Rng, core.hpp:94).
 * Seeding: x[0] = seed, x[i] = f * (x[i-1] ^ (x[i-1] >> 62)) + i. The first refill only needs
 * x[0], x[1] and x[156] for its first word: y = upper(x0) | lower(x1);
 * x0' = x156 ^ (y >> 1) ^ (odd(y) ? a : 0), then the standard tempering. */
uint64_t so_mt64_first(uint64_t seed) {
    const uint64_t f = 6364136223846793005ULL;
    uint64_t x = seed, x0 = seed, x1 = 0, x156 = 0;
    for (uint64_t i = 1; i <= 156; ++i) {
        x = f * (x ^ (x >> 62)) + i;
        if (i == 1) x1 = x;
    }
    x156 = x;
    uint64_t y = (x0 & 0xFFFFFFFF80000000ULL) | (x1 & 0x7FFFFFFFULL);
    uint64_t z = x156 ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

double so_uniform_first(uint64_t seed) { /* core.hpp:83 */
    return (double)(so_mt64_first(seed) >> 11) * 0x1.0p-53;
}

/* ------------------------------------------------------------------ similarity (core.cpp:21-38) */
double so_dot(const float* a, const float* b, int dim) {
    double s = 0.0;
    for (int i = 0; i < dim; ++i) s += (double)a[i] * (double)b[i];
    return s;
}

double so_cosine(const float* a, const float* b, int dim) {
    double s = so_dot(a, b, dim);
    if (s > 1.0) s = 1.0;
    if (s < -1.0) s = -1.0;
    return s;
}

/* ------------------------------------------------------------------ pyramid (index.cpp:12-31) */
int so_pyramid_segments(double duration, double delta, int* levels, double* starts,
                        double* lengths, int cap) {
    if (!(delta > 0.0) || delta > 1.0 || !(duration > 0.0)) return -1;
    if (delta < 1.0 / 16.0) delta = 1.0 / 16.0;
    int max_level = (int)floor(log2(1.0 / delta) + 1e-9);
    int n = 0;
    for (int level = 0; level <= max_level; ++level) {
        int tiles = 1 << level;
        double len = duration / tiles;
        for (int i = 0; i < tiles; ++i, ++n) {
            if (n < cap) {
                levels[n] = level;
                starts[n] = i * len;
                lengths[n] = len;
            }
        }
    }
    return n;
}

/* ------------------------------------------------------------------ search (index.cpp:289-326) */
/* (sim desc, id asc) ordering of index.cpp:320-323 */
static int hit_before(const so_hit* a, const so_hit* b) {
    if (a->similarity != b->similarity) return a->similarity > b->similarity;
    return a->entry_id < b->entry_id;
}

int so_search(const so_arena* ar, const float* q, int k, so_hit* out) {
    if (k < 1) return -1;
    int n = 0;
    for (int e = 0; e < ar->n_entries; ++e) {
        int64_t lo = ar->off[e], hi = ar->off[e + 1];
        if (hi <= lo) continue;
        so_hit best;
        best.entry_id = ar->ids[e];
        best.row = -1;
        best.similarity = 0.0;
        for (int64_t r = lo; r < hi; ++r) {
            double sim = so_cosine(q, ar->rows + r * ar->dim, ar->dim);
            if (best.row < 0 || sim > best.similarity) { /* strict '>', index.cpp:311 */
                best.similarity = sim;
                best.row = (int32_t)r;
            }
        }
        best.level = ar->levels[best.row];
        best.start_s = ar->starts[best.row];
        best.length_s = ar->lengths[best.row];
        /* insertion into the running top-k (equivalent to full sort + truncate) */
        int pos = n < k ? n : k;
        if (n >= k && !hit_before(&best, &out[k - 1])) continue;
        while (pos > 0 && hit_before(&best, &out[pos - 1])) {
            if (pos < k) out[pos] = out[pos - 1];
            --pos;
        }
        out[pos] = best;
        if (n < k) ++n;
    }
    return n;
}

/* ------------------------------------------------------------------ selector (selector.cpp:24-85) */
static double clamp01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

int so_score_select(int n, const double* sims, const double* durations, const float* audio,
                    int dim, const float* neg, double L, double temp, double thr,
                    uint64_t rng_seed, double* s_pos, double* s_neg, double* a, double* b,
                    double* q) {
    double max_pos = 0.0, max_neg_dis = 0.0;
    for (int i = 0; i < n; ++i) {
        s_pos[i] = clamp01(sims[i]);
        s_neg[i] = clamp01(so_cosine(audio + (size_t)i * dim, neg, dim));
        if (s_pos[i] > max_pos) max_pos = s_pos[i];
        if (1.0 - s_neg[i] > max_neg_dis) max_neg_dis = 1.0 - s_neg[i];
    }
    const double lo = 0.5 * L, hi = 1.5 * L;
    for (int i = 0; i < n; ++i) {
        a[i] = max_pos > 0.0 ? s_pos[i] / max_pos : 0.0;
        b[i] = max_neg_dis > 0.0 ? (1.0 - s_neg[i]) / max_neg_dis : 0.0;
        int ok = durations[i] >= lo && durations[i] <= hi;
        q[i] = ok ? (a[i] < b[i] ? a[i] : b[i]) : 0.0;
    }
    /* select: survivors q >= thr, stable softmax over s_pos, one uniform() draw */
    int surv[64], ns = 0;
    for (int i = 0; i < n && ns < 64; ++i)
        if (q[i] >= thr) surv[ns++] = i;
    if (ns == 0) return -1;
    double max_s = s_pos[surv[0]];
    for (int j = 0; j < ns; ++j)
        if (s_pos[surv[j]] > max_s) max_s = s_pos[surv[j]];
    double w[64], total = 0.0;
    for (int j = 0; j < ns; ++j) {
        w[j] = exp((s_pos[surv[j]] - max_s) / temp);
        total += w[j];
    }
    double target = so_uniform_first(rng_seed) * total;
    double acc = 0.0;
    for (int j = 0; j < ns; ++j) {
        acc += w[j];
        if (acc >= target) return surv[j];
    }
    return surv[ns - 1];
}

/* ------------------------------------------------------------------ gater (gater.cpp:13-92) */
void so_context_features(const float* p, const float* c, int dim, int T, double* phi) {
    phi[0] = so_cosine(p, c, dim);
    for (int j = 0; j < 8; ++j) {
        size_t lo = (size_t)j * dim / 8, hi = (size_t)(j + 1) * dim / 8;
        double s = 0.0;
        for (size_t i = lo; i < hi; ++i) s += (double)p[i] * c[i];
        phi[1 + j] = s;
    }
    phi[9] = (double)T / 200.0;
    phi[10] = 1.0;
}

static double softplus(double x) { /* gater.cpp:32-36 */
    if (x > 30.0) return x;
    if (x < -30.0) return exp(x);
    return log1p(exp(x));
}

int so_choose_arm(const float* theta, const float* psi, int fd, double beta, const double* phi,
                  int explore) {
    for (int i = 0; i < fd; ++i)
        if (!isfinite(phi[i])) return 0;
    int best = 0;
    double best_score = -INFINITY;
    for (int a = 0; a < 14; ++a) {
        double s = 0.0;
        for (int i = 0; i < fd; ++i) s += (double)theta[a * fd + i] * phi[i];
        if (explore) {
            double u = 0.0;
            for (int i = 0; i < fd; ++i) u += (double)psi[a * fd + i] * phi[i];
            s += beta * softplus(u);
        }
        if (s >= best_score) { /* ties to the larger skip fraction, gater.cpp:85 */
            best_score = s;
            best = a;
        }
    }
    return best;
}

/* ------------------------------------------------------------------ plan (pipeline.cpp:91-202) */
typedef struct {
    const so_arena* ar;
    const float* neg;
    const float* queries;
    const double* L;
    const uint64_t* req_ids;
    const int* T;
    uint64_t seed;
    int top_k;
    double temp, thr;
    int policy;
    const float* theta;
    const float* psi;
    int fd;
    double beta, rule_thr;
    int rule_arm, fixed_arm;
    so_plan* out;
    so_hit* hits_out;
    int lo, hi;
} plan_job;

static void plan_one(const plan_job* j, int i) {
    const so_arena* ar = j->ar;
    const int dim = ar->dim;
    const float* q = j->queries + (size_t)i * dim;
    so_plan* o = j->out + i;
    memset(o, 0, sizeof(*o));
    o->pick = -1;
    so_hit hits[64];
    int nh = so_search(ar, q, j->top_k, hits);
    o->n_hits = nh;
    if (j->hits_out)
        for (int h = 0; h < nh; ++h) j->hits_out[(size_t)i * j->top_k + h] = hits[h];
    int hit = 0;
    double sim = 0.0, phi[11];
    if (nh > 0) {
        double sims[64], dur[64], sp[64], sn[64], a[64], b[64], qq[64];
        float* audio = (float*)malloc(sizeof(float) * (size_t)nh * dim);
        for (int h = 0; h < nh; ++h) {
            sims[h] = hits[h].similarity;
            dur[h] = hits[h].length_s; /* matched segment length, pipeline.cpp:122 */
            memcpy(audio + (size_t)h * dim, ar->rows + (size_t)hits[h].row * dim,
                   sizeof(float) * dim);
        }
        uint64_t rs = so_derive_seed(j->seed, j->req_ids[i], 2, 0); /* pipeline.cpp:211 */
        int pick = so_score_select(nh, sims, dur, audio, dim, j->neg, j->L[i], j->temp, j->thr, rs,
                                   sp, sn, a, b, qq);
        free(audio);
        if (pick >= 0) {
            const so_hit* c = &hits[pick];
            const float* seg = ar->rows + (size_t)c->row * dim;
            hit = 1;
            o->pick = pick;
            o->entry_id = c->entry_id;
            o->level = c->level;
            o->start_s = c->start_s;
            o->length_s = c->length_s;
            sim = so_cosine(q, seg, dim);                  /* pipeline.cpp:173 */
            so_context_features(q, seg, dim, j->T[i], phi); /* pipeline.cpp:174 */
        }
    }
    int arm = 0;
    if (hit) {
        if (j->policy == 0 || j->policy == 1)
            arm = so_choose_arm(j->theta, j->psi, j->fd, j->beta, phi, j->policy == 1);
        else if (j->policy == 2)
            arm = sim >= j->rule_thr ? j->rule_arm : 0;
        else
            arm = j->fixed_arm;
    } else if (j->policy == 3) {
        arm = j->fixed_arm;
    }
    o->hit = hit;
    o->arm = arm;
    o->steps_skipped = (int)llround(0.05 * arm * j->T[i]); /* gater.hpp:18, simgen.cpp:70 */
    o->similarity = sim;
}

static void* plan_worker(void* arg) {
    const plan_job* j = (const plan_job*)arg;
    for (int i = j->lo; i < j->hi; ++i) plan_one(j, i);
    return NULL;
}

int so_plan_batch(const so_arena* ar, const float* neg, int B, const float* queries,
                  const double* L, const uint64_t* req_ids, const int* T, uint64_t seed,
                  int top_k, double temp, double thr, int policy, const float* theta,
                  const float* psi, int fd, double beta, double rule_thr, int rule_arm,
                  int fixed_arm, int nthreads, so_plan* out, so_hit* hits_out) {
    if (top_k < 1 || top_k > 64) return -1;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    plan_job jobs[256];
    pthread_t th[256];
    int per = (B + nthreads - 1) / nthreads, nt = 0;
    for (int t = 0; t < nthreads; ++t) {
        plan_job* j = &jobs[t];
        j->ar = ar; j->neg = neg; j->queries = queries; j->L = L; j->req_ids = req_ids;
        j->T = T; j->seed = seed; j->top_k = top_k; j->temp = temp; j->thr = thr;
        j->policy = policy; j->theta = theta; j->psi = psi; j->fd = fd; j->beta = beta;
        j->rule_thr = rule_thr; j->rule_arm = rule_arm; j->fixed_arm = fixed_arm;
        j->out = out; j->hits_out = hits_out;
        j->lo = t * per;
        j->hi = j->lo + per < B ? j->lo + per : B;
        if (j->lo >= j->hi) break;
        if (nthreads == 1) {
            plan_worker(j);
        } else {
            pthread_create(&th[t], NULL, plan_worker, j);
        }
        ++nt;
    }
    if (nthreads > 1)
        for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
    return 0;
}

/* ------------------------------------------------------------ glibc exp, restated */
/* The reference's std::exp is glibc 2.39's exp; on an x86-64 CPU with FMA + AVX2 its ifunc picks
 * the FMA build of sysdeps/ieee754/dbl-64/e_exp.c (ARM optimized-routines, 128-entry table).
 * This is that object code's operation sequence (objdump of libm.so.6, __exp_fma), every fma
 * where the binary has one, so it is bit-identical to the library on every input; the device
 * copy (csrc/select_dev.cuh ref_exp) repeats it with __fma_rn / __dmul_rn / __dadd_rn.
 * tests/test_oracle_pinning.py checks this function against the libm exp. */
static double u2d(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
static uint64_t d2u(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }

double so_ref_exp(double x) {
    const double InvLn2N = 0x1.71547652b82fep7, Shift = 0x1.8p52;
    const double NegLn2hiN = -0x1.62e42fefa0000p-8, NegLn2loN = -0x1.cf79abc9e3b3ap-47;
    const double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3;
    const double C4 = 0x1.55555cf172b91p-5, C5 = 0x1.1111167a4d017p-7;
    const uint64_t ix = d2u(x);
    const uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ff;
    int special = 0;
    if (abstop - 0x3c9u > 0x3eu) {
        if ((int32_t)(abstop - 0x3c9u) < 0) return x + 1.0;  /* |x| < 2^-54 */
        if (abstop > 0x408u) {                                /* |x| >= 1024 */
            if (ix == 0xfff0000000000000ull) return 0.0;
            if (abstop == 0x7ffu) return x + 1.0;             /* inf or nan */
            if (ix >> 63) return 0x1p-767 * 0x1p-767;        /* underflow: +0 */
            return 0x1p769 * 0x1p769;                         /* overflow: inf */
        }
        special = 1;                                          /* large |x|: scale may overflow */
    }
    double kd = fma(x, InvLn2N, Shift);
    const uint64_t ki = d2u(kd);
    kd = kd - Shift;
    double r = fma(kd, NegLn2hiN, x);
    r = fma(kd, NegLn2loN, r);
    const uint64_t idx = 2 * (ki & 127), top = ki << 45;
    const double tail = u2d(sw_exp_tab[idx]);
    uint64_t sbits = sw_exp_tab[idx + 1] + top;
    const double r2 = r * r;
    const double p1 = fma(r, C3, C2), p2 = fma(r, C5, C4);
    double tmp = fma(p1, r2, r + tail);
    tmp = fma(r2 * r2, p2, tmp);
    if (special) {  /* specialcase() */
        if ((ki & 0x80000000u) == 0) {
            sbits -= 1009ull << 52;
            const double scale = u2d(sbits);
            return fma(scale, tmp, scale) * 0x1p1009;
        }
        sbits += 1022ull << 52;
        const double scale = u2d(sbits);
        const double st = tmp * scale;
        double y = scale + st;
        if (1.0 > y) {
            const double hi = y + 1.0;
            const double lo = (scale - y) + st;
            y = (((1.0 - hi) + y) + lo + hi) - 1.0;
            if (y == 0.0) y = 0.0;
        }
        return y * 0x1p-1022;
    }
    const double scale = u2d(sbits);
    return fma(scale, tmp, scale);
}

/* glibc 2.39 log1p, FMA build (x86-64 ifunc; fdlibm's s_log1p.c as compiled with FMA): the op
 * sequence of its object code, like so_ref_exp. Used by explore-mode softplus (gater.cpp:32-36);
 * the device copy is select_dev.cuh ref_log1p. */
static double set_high(double u, uint32_t hi) {
    return u2d(((uint64_t)hi << 32) | (d2u(u) & 0xffffffffull));
}

double so_ref_log1p(double x) {
    const double Lp1 = 0x1.5555555555593p-1, Lp2 = 0x1.999999997fa04p-2;
    const double Lp3 = 0x1.2492494229359p-2, Lp4 = 0x1.c71c51d8e78afp-3;
    const double Lp5 = 0x1.7466496cb03dep-3, Lp6 = 0x1.39a09d078c69fp-3;
    const double Lp7 = 0x1.2f112df3e5244p-3;
    const double ln2_hi = 0x1.62e42fee00000p-1, ln2_lo = 0x1.a39ef35793c76p-33;
    const int32_t hx = (int32_t)(d2u(x) >> 32);
    int32_t k = 0;
    uint32_t hu = 0;
    double f, c = 0.0, u, hfsq;
    if (hx <= 0x3fda8279) {                        /* x < 0.41422 */
        const uint32_t ax = (uint32_t)hx & 0x7fffffffu;
        if (ax > 0x3fefffffu) {                    /* x <= -1 */
            if (x == -1.0) return -0x1p54 / 0.0;
            return (x - x) / (x - x);
        }
        if (ax <= 0x3e1fffffu) {                   /* |x| < 2^-29 */
            if (ax <= 0x3c8fffffu) return x;
            return fma(x * x, -0.5, x);
        }
        if ((uint32_t)hx + 0x402d413cu > 0x402d413cu) {  /* k = 0: f = x */
            f = x;
            hfsq = (x * 0.5) * x;
            goto poly;
        }
        goto upath;                                /* -1 < x <= -0.2929 */
    }
    if (hx > 0x7fefffff) return x + x;             /* inf, nan */
    if (hx > 0x433fffff) {                         /* x >= 2^53: u = x, c = 0 */
        k = (hx >> 20) - 0x3ff;
        u = x;
        hu = (uint32_t)hx;
        goto norm;
    }
upath:
    u = x + 1.0;
    hu = (uint32_t)(d2u(u) >> 32);
    k = (int32_t)(hu >> 20) - 0x3ff;
    c = k > 0 ? (1.0 - (u - x)) / u : (x - (u - 1.0)) / u;  /* correction term */
norm:
    hu &= 0xfffffu;
    if (hu > 0x6a09du) {
        k += 1;
        u = set_high(u, hu | 0x3fe00000u);
        hu = (0x100000u - hu) >> 2;
    } else {
        u = set_high(u, hu | 0x3ff00000u);
    }
    f = u - 1.0;
    hfsq = (f * 0.5) * f;
    if (hu == 0) {                                 /* |f| < 2^-20 */
        if (f == 0.0) {
            if (k == 0) return 0.0;
            const double dk = (double)k;
            return fma(dk, ln2_hi, fma(dk, ln2_lo, c));
        }
        const double R = fma(-f, 0x1.5555555555555p-1, 1.0) * hfsq;
        if (k == 0) return f - R;
        const double dk = (double)k;
        return fma(dk, ln2_hi, -((R - fma(dk, ln2_lo, c)) - f));
    }
poly:
    {
        const double s = f / (f + 2.0), z = s * s;
        const double R2 = fma(z, Lp3, Lp2), R3 = fma(z, Lp5, Lp4), R4 = fma(z, Lp7, Lp6);
        const double z2 = z * z, z4 = z2 * z2, z6 = z2 * z4;
        double R = fma(z, Lp1, z2 * R2);
        R = fma(z4, R3, R);
        R = fma(z6, R4, R);
        const double w = (R + hfsq) * s;
        if (k == 0) return f - (hfsq - w);
        const double dk = (double)k;
        return fma(dk, ln2_hi, -((hfsq - (fma(dk, ln2_lo, c) + w)) - f));
    }
}

/* ours and the library's log1p over the same arguments (pinning test only) */
void so_log1p_pair(const double* x, int64_t n, double* ours, double* lib) {
    for (int64_t i = 0; i < n; ++i) {
        ours[i] = so_ref_log1p(x[i]);
        lib[i] = log1p(x[i]);
    }
}

/* ours and the library's exp over the same arguments (pinning test only) */
void so_exp_pair(const double* x, int64_t n, double* ours, double* lib) {
    for (int64_t i = 0; i < n; ++i) {
        ours[i] = so_ref_exp(x[i]);
        lib[i] = exp(x[i]);
    }
}

/* ------------------------------------------------------------------ align + noise (ours) */
/* Philox4x32-R (Salmon et al., SC'11): R rounds of the 4x32 bijection with the Weyl key
 * schedule. so_philox4x32_10 is Random123's default (pinned by its known-answer vector);
 * K4's noise uses R = SW_PHILOX_ROUNDS (noise_def.h). */
void so_philox4x32_r(const uint32_t ctr[4], const uint32_t key[2], int rounds, uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < rounds; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c0 = n0;
        c1 = (uint32_t)p1;
        c2 = n2;
        c3 = (uint32_t)p0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

void so_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    so_philox4x32_r(ctr, key, 10, out);
}

static float as_f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t as_u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

/* The normal transform, our definition, every fp32 rounding spelled
 * out exactly as the device evaluates it (paper_2603_07865_b200/csrc/align.cu icdf4): one normal
 * per 32-bit Philox word w,
 *   v = 2 - asfloat(0x3f800000 | (w & 0x7fffff))   in (0, 1], exact
 *   s = (bits(v) >> 17) - 6656; |z| = fmaf(B[s], v, A[s]); z = |z| with w's sign bit,
 * (A, B) the committed segment table (noise_table.h, generated by tools/gen_noise_table.py: the
 * least-squares lines through sqrt(2) erfcinv(v - 2^-24), 64 per binade). */
static float icdf_normal(uint32_t w) {
    float v = 2.0f - as_f(0x3f800000u | (w & 0x7fffffu));
    uint32_t s = (as_u(v) >> SW_NOISE_SHIFT) - SW_NOISE_BASE;
    float za = fmaf(sw_noise_tab[s][1], v, sw_noise_tab[s][0]);
    return as_f(as_u(za) ^ (w & 0x80000000u));
}

void so_icdf_normals(const uint32_t* words, int64_t n, float* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = icdf_normal(words[i]);
}

void so_philox_normals(uint64_t seed, uint64_t rid, int64_t n, float* out) {
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (int64_t i = 0; i < n; i += 4) {
        uint64_t quad = (uint64_t)i >> 2;
        uint32_t ctr[4] = {(uint32_t)quad, (uint32_t)(quad >> 32), (uint32_t)rid,
                           (uint32_t)(rid >> 32)};
        uint32_t r[4];
        float z[4];
        so_philox4x32_r(ctr, key, SW_PHILOX_ROUNDS, r);
        for (int t = 0; t < 4; ++t) z[t] = icdf_normal(r[t]);
        for (int t = 0; t < 4 && i + t < n; ++t) out[i + t] = z[t];
    }
}

int so_align_noise(const float* latent, int C, int t_src, int F, double start_s,
                   double length_s, double L, double fps, double abar, const float* eps,
                   uint64_t philox_seed, uint64_t rid, float* out) {
    /* frame window: slice_clip index math (simgen.cpp:116-119) at the latent frame rate */
    long long lo = llround(start_s * fps), hi = llround((start_s + length_s) * fps);
    if (lo > t_src) lo = t_src;
    if (hi > t_src) hi = t_src;
    if (hi < lo) hi = lo;
    int t_seg = (int)(hi - lo);
    int t_out = (int)llround(L * fps); /* output length rule of vocoder.cpp:144-145 */
    float s0 = (float)sqrt(abar), s1 = (float)sqrt(1.0 - abar);
    int64_t n = (int64_t)C * t_out * F;
    float* noise = NULL;
    if (!eps) {
        noise = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
        so_philox_normals(philox_seed, rid, n, noise);
        eps = noise;
    }
    for (int c = 0; c < C; ++c)
        for (int t = 0; t < t_out; ++t) {
            int src = t_seg > 0 ? (int)lo + t % t_seg : -1; /* crop, or tile cyclically */
            for (int f = 0; f < F; ++f) {
                int64_t o = ((int64_t)c * t_out + t) * F + f;
                float x0 = src >= 0 ? latent[((int64_t)c * t_src + src) * F + f] : 0.0f;
                out[o] = fmaf(s1, eps[o], s0 * x0);
            }
        }
    free(noise);
    return t_out;
}

void so_abar_table(double* abar) {
    const double b0 = sqrt(0.00085), b1 = sqrt(0.012);
    abar[0] = 1.0;
    for (int t = 1; t <= 1000; ++t) {
        double s = b0 + (b1 - b0) * (double)(t - 1) / 999.0;
        abar[t] = abar[t - 1] * (1.0 - s * s);
    }
}

int so_abar_index(int T, int S) {
    if (T < 1) return 1000;
    long long i = llround((double)(T - S) * 1000.0 / (double)T);
    return (int)(i < 0 ? 0 : (i > 1000 ? 1000 : i));
}
