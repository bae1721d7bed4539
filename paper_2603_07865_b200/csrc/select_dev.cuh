// Device-side restatement of score_candidates + select + context_features + choose_arm + t*,
// shared by the per-request select kernel and the fused per-query finish kernel.
// See select.cu for the parity notes (fp64 operation order, unfused products, glibc's exp).
#pragma once
#include "sw_internal.cuh"

#define SW_EXP_QUAL static __device__ const
#include "exp_table.h"

namespace sw {
namespace dev {

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {  // core.cpp:58-63
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t derive_seed(uint64_t base, uint64_t a, uint64_t b,
                                                         uint64_t c) {  // core.cpp:65-71
    uint64_t s = splitmix64(base ^ 0x53454d5741524dULL);
    s = splitmix64(s ^ a);
    s = splitmix64(s ^ b);
    return splitmix64(s ^ c);
}
// First output of std::mt19937_64(seed): only state words 0, 1 and 156 feed the first refill.
__device__ __forceinline__ uint64_t mt64_first(uint64_t seed) {
    const uint64_t f = 6364136223846793005ULL;
    uint64_t x = seed, x1 = 0;
#pragma unroll 4
    for (uint64_t i = 1; i <= 156; ++i) {
        x = f * (x ^ (x >> 62)) + i;
        if (i == 1) x1 = x;
    }
    const uint64_t y = (seed & 0xFFFFFFFF80000000ULL) | (x1 & 0x7FFFFFFFULL);
    uint64_t z = x ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}
__device__ __forceinline__ double clamp01(double v) { return fmin(1.0, fmax(0.0, v)); }

// The reference's std::exp = glibc 2.39's exp, whose ifunc picks the FMA build of
// sysdeps/ieee754/dbl-64/e_exp.c on an FMA + AVX2 host: this is that object code's operation
// sequence (every fma where the binary has one; table: exp_table.h, tools/gen_exp_table.py),
// so the softmax weights — and with them the cumulative draw — are bit-identical to the
// reference's. Restated in C as so_ref_exp (oracle), pinned there to the library bit for bit.
__device__ __forceinline__ double ref_exp(double x) {
    constexpr double InvLn2N = 0x1.71547652b82fep7, Shift = 0x1.8p52;
    constexpr double NegLn2hiN = -0x1.62e42fefa0000p-8, NegLn2loN = -0x1.cf79abc9e3b3ap-47;
    constexpr double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3;
    constexpr double C4 = 0x1.55555cf172b91p-5, C5 = 0x1.1111167a4d017p-7;
    const uint64_t ix = (uint64_t)__double_as_longlong(x);
    const uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ffu;
    bool special = false;
    if (abstop - 0x3c9u > 0x3eu) {
        if ((int32_t)(abstop - 0x3c9u) < 0) return __dadd_rn(x, 1.0);  // |x| < 2^-54
        if (abstop > 0x408u) {                                          // |x| >= 1024
            if (ix == 0xfff0000000000000ull) return 0.0;
            if (abstop == 0x7ffu) return __dadd_rn(x, 1.0);             // inf or nan
            return (ix >> 63) ? 0.0 : __longlong_as_double(0x7ff0000000000000ll);
        }
        special = true;  // large |x|: the scale may over/underflow
    }
    double kd = __fma_rn(x, InvLn2N, Shift);
    const uint64_t ki = (uint64_t)__double_as_longlong(kd);
    kd = __dsub_rn(kd, Shift);
    double r = __fma_rn(kd, NegLn2hiN, x);
    r = __fma_rn(kd, NegLn2loN, r);
    const uint64_t idx = 2 * (ki & 127), top = ki << 45;
    const double tail = __longlong_as_double((long long)sw_exp_tab[idx]);
    uint64_t sbits = sw_exp_tab[idx + 1] + top;
    const double r2 = __dmul_rn(r, r);
    const double p1 = __fma_rn(r, C3, C2), p2 = __fma_rn(r, C5, C4);
    double tmp = __fma_rn(p1, r2, __dadd_rn(r, tail));
    tmp = __fma_rn(__dmul_rn(r2, r2), p2, tmp);
    if (special) {  // glibc's specialcase()
        if ((ki & 0x80000000u) == 0) {
            sbits -= 1009ull << 52;
            const double scale = __longlong_as_double((long long)sbits);
            return __dmul_rn(__fma_rn(scale, tmp, scale), 0x1p1009);
        }
        sbits += 1022ull << 52;
        const double scale = __longlong_as_double((long long)sbits);
        const double st = __dmul_rn(tmp, scale);
        double y = __dadd_rn(scale, st);
        if (1.0 > y) {
            const double hi = __dadd_rn(y, 1.0);
            const double lo = __dadd_rn(__dsub_rn(scale, y), st);
            y = __dsub_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dsub_rn(1.0, hi), y), lo), hi), 1.0);
            if (y == 0.0) y = 0.0;
        }
        return __dmul_rn(y, 0x1p-1022);
    }
    const double scale = __longlong_as_double((long long)sbits);
    return __fma_rn(scale, tmp, scale);
}

__device__ __forceinline__ double set_high(double u, uint32_t hi) {
    return __longlong_as_double(
        (long long)(((uint64_t)hi << 32) | ((uint64_t)__double_as_longlong(u) & 0xffffffffull)));
}

// glibc 2.39's log1p, FMA build (fdlibm's s_log1p.c as compiled with FMA; x86-64 ifunc): its
// object code's operation sequence, like ref_exp (restated in C as so_ref_log1p, pinned to the
// library bit for bit). Explore-mode softplus (gater.cpp:32-36) is therefore exact too.
__device__ __forceinline__ double ref_log1p(double x) {
    constexpr double Lp1 = 0x1.5555555555593p-1, Lp2 = 0x1.999999997fa04p-2;
    constexpr double Lp3 = 0x1.2492494229359p-2, Lp4 = 0x1.c71c51d8e78afp-3;
    constexpr double Lp5 = 0x1.7466496cb03dep-3, Lp6 = 0x1.39a09d078c69fp-3;
    constexpr double Lp7 = 0x1.2f112df3e5244p-3;
    constexpr double ln2_hi = 0x1.62e42fee00000p-1, ln2_lo = 0x1.a39ef35793c76p-33;
    const int32_t hx = (int32_t)((uint64_t)__double_as_longlong(x) >> 32);
    int32_t k = 0;
    uint32_t hu = 0;
    double f, c = 0.0, u = 0.0, hfsq;
    bool upath = false;
    if (hx <= 0x3fda8279) {  // x < 0.41422
        const uint32_t ax = (uint32_t)hx & 0x7fffffffu;
        if (ax > 0x3fefffffu) {  // x <= -1
            if (x == -1.0) return -__longlong_as_double(0x7ff0000000000000ll);
            return __longlong_as_double(0x7ff8000000000000ll);
        }
        if (ax <= 0x3e1fffffu) {  // |x| < 2^-29
            if (ax <= 0x3c8fffffu) return x;
            return __fma_rn(__dmul_rn(x, x), -0.5, x);
        }
        if ((uint32_t)hx + 0x402d413cu > 0x402d413cu) {  // k = 0: f = x
            f = x;
            hfsq = __dmul_rn(__dmul_rn(x, 0.5), x);
        } else {
            upath = true;  // -1 < x <= -0.2929
        }
    } else {
        if (hx > 0x7fefffff) return __dadd_rn(x, x);  // inf, nan
        if (hx > 0x433fffff) {                          // x >= 2^53: u = x, c = 0
            k = (hx >> 20) - 0x3ff;
            u = x;
            hu = (uint32_t)hx;
        } else {
            upath = true;
        }
    }
    if (k != 0 || upath) {
        if (upath) {
            u = __dadd_rn(x, 1.0);
            hu = (uint32_t)((uint64_t)__double_as_longlong(u) >> 32);
            k = (int32_t)(hu >> 20) - 0x3ff;
            c = k > 0 ? __ddiv_rn(__dsub_rn(1.0, __dsub_rn(u, x)), u)
                      : __ddiv_rn(__dsub_rn(x, __dsub_rn(u, 1.0)), u);  // correction term
        }
        hu &= 0xfffffu;
        if (hu > 0x6a09du) {
            k += 1;
            u = set_high(u, hu | 0x3fe00000u);
            hu = (0x100000u - hu) >> 2;
        } else {
            u = set_high(u, hu | 0x3ff00000u);
        }
        f = __dsub_rn(u, 1.0);
        hfsq = __dmul_rn(__dmul_rn(f, 0.5), f);
        if (hu == 0) {  // |f| < 2^-20
            const double dk = (double)k;
            if (f == 0.0) {
                if (k == 0) return 0.0;
                return __fma_rn(dk, ln2_hi, __fma_rn(dk, ln2_lo, c));
            }
            const double R = __dmul_rn(__fma_rn(-f, 0x1.5555555555555p-1, 1.0), hfsq);
            if (k == 0) return __dsub_rn(f, R);
            return __fma_rn(dk, ln2_hi, -__dsub_rn(__dsub_rn(R, __fma_rn(dk, ln2_lo, c)), f));
        }
    }
    const double s = __ddiv_rn(f, __dadd_rn(f, 2.0)), z = __dmul_rn(s, s);
    const double R2 = __fma_rn(z, Lp3, Lp2), R3 = __fma_rn(z, Lp5, Lp4), R4 = __fma_rn(z, Lp7, Lp6);
    const double z2 = __dmul_rn(z, z), z4 = __dmul_rn(z2, z2), z6 = __dmul_rn(z2, z4);
    double R = __fma_rn(z, Lp1, __dmul_rn(z2, R2));
    R = __fma_rn(z4, R3, R);
    R = __fma_rn(z6, R4, R);
    const double w = __dmul_rn(__dadd_rn(R, hfsq), s);
    if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, w));
    const double dk = (double)k;
    return __fma_rn(dk, ln2_hi,
                    -__dsub_rn(__dsub_rn(hfsq, __dadd_rn(__fma_rn(dk, ln2_lo, c), w)), f));
}

__device__ __forceinline__ double softplus(double x) {  // gater.cpp:32-36
    if (x > 30.0) return x;
    if (x < -30.0) return ref_exp(x);
    return ref_log1p(ref_exp(x));
}

struct GateOut {
    int pick;
    uint32_t flags;
};

__device__ __forceinline__ GateOut select_draw(int n, const double* s_pos, const double* q,
                                               double temp, double thr, double u);

// score_candidates + select over n records; scores optionally written (n x 5).
// Rng(seed).uniform() (core.hpp:83): (first mt19937_64 output >> 11) * 2^-53
__device__ __forceinline__ double uniform_draw(uint64_t rng_seed) {
    return (double)(mt64_first(rng_seed) >> 11) * 0x1.0p-53;
}

// u: the request's selector draw (uniform_draw(derive_seed(seed, id, 2)), pipeline.cpp:211)
__device__ __forceinline__ GateOut gate_select(int n, const double* sims, const double* snegs,
                               const double* durs, double L, double temp, double thr,
                               double u, double* scores) {
    double s_pos[kMaxTopK], a[kMaxTopK], b[kMaxTopK], q[kMaxTopK];
    double max_pos = 0.0, max_neg_dis = 0.0;
    for (int i = 0; i < n; ++i) {
        s_pos[i] = clamp01(sims[i]);
        max_pos = fmax(max_pos, s_pos[i]);
        max_neg_dis = fmax(max_neg_dis, 1.0 - snegs[i]);
    }
    const double lo = 0.5 * L, hi = 1.5 * L;
    for (int i = 0; i < n; ++i) {
        a[i] = max_pos > 0.0 ? __ddiv_rn(s_pos[i], max_pos) : 0.0;
        b[i] = max_neg_dis > 0.0 ? __ddiv_rn(1.0 - snegs[i], max_neg_dis) : 0.0;
        const bool ok = durs[i] >= lo && durs[i] <= hi;
        q[i] = ok ? fmin(a[i], b[i]) : 0.0;
        if (scores) {
            scores[i * 5 + 0] = s_pos[i];
            scores[i * 5 + 1] = snegs[i];
            scores[i * 5 + 2] = a[i];
            scores[i * 5 + 3] = b[i];
            scores[i * 5 + 4] = q[i];
        }
    }
    return select_draw(n, s_pos, q, temp, thr, u);
}

// select (selector.cpp:60-85) given the gate scores and the draw u = rng.uniform()
__device__ __forceinline__ GateOut select_draw(int n, const double* s_pos, const double* q,
                                               double temp, double thr, double u) {
    GateOut g{-1, 0u};
    int surv[kMaxTopK], ns = 0;
    for (int i = 0; i < n; ++i)
        if (q[i] >= thr) surv[ns++] = i;
    if (ns == 0) return g;  // no survivor: miss, and no RNG draw (selector.cpp:67)
    double max_s = s_pos[surv[0]];
    for (int j = 0; j < ns; ++j) max_s = fmax(max_s, s_pos[surv[j]]);
    double w[kMaxTopK], total = 0.0;
    for (int j = 0; j < ns; ++j) {
        w[j] = ref_exp(__ddiv_rn(s_pos[surv[j]] - max_s, temp));
        total = __dadd_rn(total, w[j]);
    }
    const double target = __dmul_rn(u, total);
    double acc = 0.0;
    g.pick = surv[ns - 1];
    for (int j = 0; j < ns; ++j) {
        acc = __dadd_rn(acc, w[j]);
        if (acc >= target) {
            g.pick = surv[j];
            break;
        }
    }
    return g;
}

// value (+ beta * uncertainty) of one arm: head_dot (gater.cpp:52-58), products and sums unfused
__device__ __forceinline__ double arm_score(const float* __restrict__ theta,
                                            const float* __restrict__ psi, int fd, double beta,
                                            const double* phi, int a, int explore) {
    (void)fd;  // always kFeatureDim (sw_set_gater enforces it); constant bounds keep phi in registers
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < kFeatureDim; ++i)
        s = __dadd_rn(s, __dmul_rn((double)theta[a * kFeatureDim + i], phi[i]));
    if (explore) {
        double u = 0.0;
#pragma unroll
        for (int i = 0; i < kFeatureDim; ++i)
            u = __dadd_rn(u, __dmul_rn((double)psi[a * kFeatureDim + i], phi[i]));
        s = __dadd_rn(s, __dmul_rn(beta, softplus(u)));
    }
    return s;
}

// choose_arm (gater.cpp:70-92): products and sums strictly unfused.
__device__ __forceinline__ int choose_arm(const float* __restrict__ theta, const float* __restrict__ psi, int fd,
                          double beta, const double* phi, int explore, uint32_t* flags) {
    for (int i = 0; i < fd; ++i)
        if (!isfinite(phi[i])) {
            *flags |= SW_CHOICE_NONFINITE_PHI;
            return 0;
        }
    // every score is the reference's bit for bit (exploit: IEEE products / sums; explore: plus
    // glibc's exp / log1p restated), so the ">=" scan picks exactly the reference's arm
    int best = 0;
    double best_score = -INFINITY;
    for (int a = 0; a < kNumArms; ++a) {
        const double s = arm_score(theta, psi, fd, beta, phi, a, explore);
        if (s >= best_score) {  // ties to the larger skip fraction
            best_score = s;
            best = a;
        }
    }
    return best;
}

struct SelParams {
    uint64_t seed;
    int top_k;
    double temp, thr;
    int policy, fixed_arm, rule_arm;
    double rule_thr;
    double fps;
    const float* theta;
    const float* psi;
    int fd;
    double beta;
};


// One request: the top-k hit records (sorted, (sim desc, id asc)) -> the ServeOutcome fields.
__device__ __forceinline__ sw_choice select_one(const HitRec* __restrict__ h, int nh,
                                                const sw_request& rq, const SelParams& p) {
    uint32_t flags = 0;
    if (nh < 0) {
        nh = -nh - 1;
        flags |= SW_CHOICE_INCOMPLETE;
    }
    nh = min(nh, p.top_k);
    sw_choice c;
    memset(&c, 0, sizeof(c));
    c.pick = -1;
    c.n_hits = nh;
    int hit = 0;
    double phi[kFeatureDim];
    if (nh > 0) {
        double sims[kMaxTopK], sn[kMaxTopK], du[kMaxTopK];
        for (int i = 0; i < nh; ++i) {
            sims[i] = h[i].sim;
            sn[i] = h[i].s_neg;
            du[i] = h[i].length_s;  // matched segment duration (pipeline.cpp:122)
        }
        GateOut g = gate_select(nh, sims, sn, du, rq.duration_s, p.temp, p.thr,
                                uniform_draw(derive_seed(p.seed, rq.id, 2, 0)), nullptr);
        flags |= g.flags;
        if (g.pick >= 0) {
            const HitRec& ch = h[g.pick];
            hit = 1;
            c.pick = g.pick;
            c.entry_id = ch.entry_id;
            c.segment.level = ch.level;
            c.segment.start_s = ch.start_s;
            c.segment.length_s = ch.length_s;
            c.segment.reserved = ch.row;  // pyramid row of the matched segment
            c.similarity = ch.sim;  // cos(prompt, seg_emb) (pipeline.cpp:173)
            c.owner = ch.owner;
            c.slot = ch.slot;
            phi[0] = ch.sim;
            for (int j = 0; j < 8; ++j) phi[1 + j] = ch.phi[j];
            phi[9] = (double)rq.total_steps / 200.0;
            phi[10] = 1.0;
        }
    }
    int arm = 0;
    if (hit) {
        if (p.policy == SW_POLICY_EXPLOIT || p.policy == SW_POLICY_EXPLORE)
            arm = choose_arm(p.theta, p.psi, p.fd, p.beta, phi, p.policy == SW_POLICY_EXPLORE,
                             &flags);
        else if (p.policy == SW_POLICY_RULE)
            arm = c.similarity >= p.rule_thr ? p.rule_arm : 0;
        else
            arm = p.fixed_arm;
    } else if (p.policy == SW_POLICY_FIXED) {
        arm = p.fixed_arm;  // latency held constant even on a miss (pipeline.cpp:229-231)
    }
    const double skip = 0.05 * (double)arm;
    c.hit = hit;
    c.arm = arm;
    c.skip_fraction = skip;
    c.steps_skipped = (int32_t)llround(skip * (double)rq.total_steps);
    c.t_out = hit ? (int32_t)llround(rq.duration_s * p.fps) : 0;
    c.flags = flags;
    return c;
}

__device__ __forceinline__ double warp_max_d(double v) {
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// gate_select with candidate i held by lane i (n <= 32): the same fp64 operations; the two
// order-dependent sums (softmax total and the cumulative scan) run in candidate order through
// shuffles, identically in every lane. No per-thread arrays, so nothing lands in local memory.
__device__ __forceinline__ GateOut gate_select_warp(int n, double sim, double sneg, double dur,
                                                    double L, double temp, double thr, double u,
                                                    int lane) {
    const unsigned full = 0xffffffffu;
    const bool act = lane < n;
    const double s_pos = act ? clamp01(sim) : 0.0;
    const double max_pos = warp_max_d(act ? s_pos : 0.0);          // starts at 0.0
    const double max_neg_dis = warp_max_d(act ? 1.0 - sneg : 0.0);  // starts at 0.0
    const double a = max_pos > 0.0 ? __ddiv_rn(s_pos, max_pos) : 0.0;
    const double b = max_neg_dis > 0.0 ? __ddiv_rn(1.0 - sneg, max_neg_dis) : 0.0;
    const bool ok = dur >= 0.5 * L && dur <= 1.5 * L;
    const double q = ok ? fmin(a, b) : 0.0;
    const unsigned surv = __ballot_sync(full, act && q >= thr);
    GateOut g{-1, 0u};
    if (!surv) return g;  // no survivor: miss, and no RNG draw (selector.cpp:67)
    const bool me = (surv >> lane) & 1u;
    const double max_s = warp_max_d(me ? s_pos : -INFINITY);
    const double w = me ? ref_exp(__ddiv_rn(s_pos - max_s, temp)) : 0.0;
    double total = 0.0;
    for (int j = 0; j < 32; ++j) {
        const double wj = __shfl_sync(full, w, j);
        if ((surv >> j) & 1u) total = __dadd_rn(total, wj);
    }
    const double target = __dmul_rn(u, total);
    double acc = 0.0;
    g.pick = 31 - __clz(surv);  // last survivor (selector.cpp:84)
    for (int j = 0; j < 32; ++j) {
        const double wj = __shfl_sync(full, w, j);
        if (!((surv >> j) & 1u)) continue;
        acc = __dadd_rn(acc, wj);
        if (acc >= target) {
            g.pick = j;
            break;
        }
    }
    return g;
}

// Warp-cooperative select_one for one request: lane 0 runs the gate and the draw (u precomputed),
// lanes 0..13 score one arm each, and the argmax keeps choose_arm's ">=" rule (ties -> larger
// arm). The result is valid in lane 0.
__device__ __forceinline__ sw_choice select_warp(const HitRec* __restrict__ h, int nh, double u,
                                                 const sw_request& rq, const SelParams& p,
                                                 int lane) {
    uint32_t flags = 0;
    if (nh < 0) {
        nh = -nh - 1;
        flags |= SW_CHOICE_INCOMPLETE;
    }
    nh = min(nh, p.top_k);
    int pick = -1;
    if (nh > 0) {
        const bool act = lane < nh;
        // matched segment duration (pipeline.cpp:122)
        const GateOut g = gate_select_warp(nh, act ? h[lane].sim : 0.0, act ? h[lane].s_neg : 0.0,
                                           act ? h[lane].length_s : 0.0, rq.duration_s, p.temp,
                                           p.thr, u, lane);
        flags |= g.flags;
        pick = g.pick;
    }
    sw_choice c;
    memset(&c, 0, sizeof(c));
    c.pick = pick;
    c.n_hits = nh;
    const int hit = pick >= 0;
    int arm = 0;
    if (hit) {
        const HitRec& ch = h[pick];
        c.entry_id = ch.entry_id;
        c.segment.level = ch.level;
        c.segment.start_s = ch.start_s;
        c.segment.length_s = ch.length_s;
        c.segment.reserved = ch.row;  // pyramid row of the matched segment
        c.similarity = ch.sim;  // cos(prompt, seg_emb) (pipeline.cpp:173)
        c.owner = ch.owner;
        c.slot = ch.slot;
        if (p.policy == SW_POLICY_EXPLOIT || p.policy == SW_POLICY_EXPLORE) {
            double phi[kFeatureDim];
            phi[0] = ch.sim;
#pragma unroll
            for (int j = 0; j < 8; ++j) phi[1 + j] = ch.phi[j];
            phi[9] = (double)rq.total_steps / 200.0;
            phi[10] = 1.0;
            bool finite = true;
#pragma unroll
            for (int i = 0; i < kFeatureDim; ++i) finite = finite && isfinite(phi[i]);
            if (!finite) {
                flags |= SW_CHOICE_NONFINITE_PHI;  // gater.cpp:71-76
            } else {
                const int explore = p.policy == SW_POLICY_EXPLORE;
                double s = lane < kNumArms
                               ? arm_score(p.theta, p.psi, p.fd, p.beta, phi, lane, explore)
                               : -INFINITY;
                // argmax; equal scores -> larger arm (the ">=" scan of gater.cpp:85)
                double bs = s;
                int ba = lane < kNumArms ? lane : -1;
                for (int o = 16; o; o >>= 1) {
                    const double os = __shfl_xor_sync(0xffffffffu, bs, o);
                    const int oa = __shfl_xor_sync(0xffffffffu, ba, o);
                    if (os > bs || (os == bs && oa > ba)) {
                        bs = os;
                        ba = oa;
                    }
                }
                arm = ba;
            }
        } else if (p.policy == SW_POLICY_RULE) {
            arm = c.similarity >= p.rule_thr ? p.rule_arm : 0;
        } else {
            arm = p.fixed_arm;
        }
    } else if (p.policy == SW_POLICY_FIXED) {
        arm = p.fixed_arm;  // latency held constant even on a miss (pipeline.cpp:229-231)
    }
    const double skip = 0.05 * (double)arm;
    c.hit = hit;
    c.arm = arm;
    c.skip_fraction = skip;
    c.steps_skipped = (int32_t)llround(skip * (double)rq.total_steps);
    c.t_out = hit ? (int32_t)llround(rq.duration_s * p.fps) : 0;
    c.flags = flags;
    return c;
}

SelParams make_sel_params(const Ctx& c, uint64_t seed, const sw_selector_config& sel,
                          const sw_policy& pol);

}  // namespace dev
}  // namespace sw
