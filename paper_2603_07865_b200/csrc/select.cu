// K3 — duration/quality gate, stochastic select and Skip Gater, one thread per request.
//
// Restates, in the same fp64 operation order, score_candidates + select (selector.cpp:24-85),
// the selector RNG draw Rng(derive_seed(seed, id, 2)).uniform() (pipeline.cpp:211,
// core.hpp:83), context_features (gater.cpp:13-30), choose_arm (gater.cpp:52-92, double x double
// products WITHOUT fma), the rule / fixed policies (pipeline.cpp:180-202) and
// t* = llround(0.05 * arm * T) (gater.hpp:16-19, simgen.cpp:70).
// The libm calls on the path — exp in the softmax, exp / log1p in explore-mode softplus — are
// glibc's, restated operation for operation (select_dev.cuh ref_exp / ref_log1p), so weights,
// draws and arm scores are bit-identical to the reference's: SW_CHOICE_AMBIGUOUS_DRAW and
// SW_CHOICE_AMBIGUOUS_ARM are no longer set.
#include "select_dev.cuh"

namespace sw {

using namespace dev;

namespace {

__global__ void k_select(int B, const HitRec* __restrict__ hits, const int32_t* __restrict__ nh_in,
                         int ld, const sw_request* __restrict__ reqs, SelParams p,
                         sw_choice* __restrict__ out) {
    const int bq = blockIdx.x * blockDim.x + threadIdx.x;
    if (bq >= B) return;
    out[bq] = select_one(hits + (int64_t)bq * ld, nh_in[bq], reqs[bq], p);
}

// Deterministic merge of world sorted top-k lists (sim desc, id asc) into c.hits.
__global__ void k_merge(int B, int k, int world, const HitRec* __restrict__ g,
                        const int32_t* __restrict__ gn, HitRec* __restrict__ out,
                        int32_t* __restrict__ out_n) {
    const int bq = blockIdx.x * blockDim.x + threadIdx.x;
    if (bq >= B) return;
    int head[16];
    int lim[16];
    bool incomplete = false;
    for (int r = 0; r < world; ++r) {
        head[r] = 0;
        int n = gn[(int64_t)r * B + bq];
        if (n < 0) {
            n = -n - 1;
            incomplete = true;
        }
        lim[r] = n;
    }
    int m = 0;
    for (; m < k; ++m) {
        int br = -1;
        for (int r = 0; r < world; ++r) {
            if (head[r] >= lim[r]) continue;
            const HitRec& x = g[((int64_t)r * B + bq) * k + head[r]];
            if (br < 0) {
                br = r;
                continue;
            }
            const HitRec& y = g[((int64_t)br * B + bq) * k + head[br]];
            if (x.sim > y.sim || (x.sim == y.sim && x.entry_id < y.entry_id)) br = r;
        }
        if (br < 0) break;
        out[(int64_t)bq * kMaxTopK + m] = g[((int64_t)br * B + bq) * k + head[br]];
        head[br]++;
    }
    out_n[bq] = incomplete ? -m - 1 : m;
}

__global__ void k_score_select_one(int n, const double* sims, const double* sneg,
                                   const double* durs, double L, double temp, double thr,
                                   uint64_t rng_seed, double* scores, int32_t* pick) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        GateOut g = gate_select(n, sims, sneg, durs, L, temp, thr, uniform_draw(rng_seed), scores);
        pick[0] = g.pick;
        pick[1] = (int32_t)g.flags;
    }
}

// score_candidates (selector.cpp:24-58) with s_neg = clamp01(cosine(audio_i, negative)) computed
// here (sequential fp64 dot, core.cpp:26-37); lane i = candidate i
__global__ void k_score_candidates(int n, int D, const double* __restrict__ sims,
                                   const float* __restrict__ audio,
                                   const double* __restrict__ durs, const float* __restrict__ neg,
                                   double L, double* __restrict__ scores) {
    __shared__ double sn[kMaxTopK];
    const int i = threadIdx.x;
    if (i < n) {
        const float* a = audio + (int64_t)i * D;
        double s = 0.0;
        for (int d = 0; d < D; ++d) s = fma((double)a[d], (double)neg[d], s);
        sn[i] = clamp01(fmin(1.0, fmax(-1.0, s)));
    }
    __syncthreads();
    if (i == 0) {
        // gate values only: thr = 2 admits no candidate, so no draw is consumed
        gate_select(n, sims, sn, durs, L, 1.0, 2.0, 0.0, scores);
    }
}

__global__ void k_select_draw(int n, const double* __restrict__ s_pos, const double* __restrict__ q,
                              double temp, double thr, double u, int32_t* __restrict__ pick) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const GateOut g = select_draw(n, s_pos, q, temp, thr, u);
        pick[0] = g.pick;
        pick[1] = (int32_t)g.flags;
    }
}

__global__ void k_gater(const float* __restrict__ P, const float* __restrict__ Sg,
                        const int32_t* __restrict__ T, int B, int D, const float* theta,
                        const float* psi, int fd, double beta, int explore, double* phi_out,
                        int32_t* arm_out) {
    const int bq = blockIdx.x * blockDim.x + threadIdx.x;
    if (bq >= B) return;
    const float* p = P + (int64_t)bq * D;
    const float* c = Sg + (int64_t)bq * D;
    double phi[kFeatureDim];
    double s = 0.0;
    for (int i = 0; i < D; ++i) s = fma((double)p[i], (double)c[i], s);
    phi[0] = fmin(1.0, fmax(-1.0, s));
    for (int j = 0; j < 8; ++j) {
        const size_t lo = (size_t)j * D / 8, hi = (size_t)(j + 1) * D / 8;
        double t = 0.0;
        for (size_t i = lo; i < hi; ++i) t = fma((double)p[i], (double)c[i], t);
        phi[1 + j] = t;
    }
    phi[9] = (double)T[bq] / 200.0;
    phi[10] = 1.0;
    uint32_t flags = 0;
    arm_out[bq] = choose_arm(theta, psi, fd, beta, phi, explore, &flags);
    for (int i = 0; i < kFeatureDim; ++i) phi_out[(int64_t)bq * kFeatureDim + i] = phi[i];
}

}  // namespace

SelParams dev::make_sel_params(const Ctx& c, uint64_t seed, const sw_selector_config& sel,
                               const sw_policy& pol) {
    SelParams p;
    p.seed = seed;
    p.top_k = sel.top_k;
    p.temp = sel.temperature;
    p.thr = sel.quality_threshold;
    p.policy = pol.kind;
    p.fixed_arm = pol.fixed_arm;
    p.rule_arm = (int)llround(pol.rule_skip_fraction / 0.05);  // pipeline.cpp:193
    p.rule_thr = pol.rule_similarity_threshold;
    p.fps = c.cfg.latent_fps;
    p.theta = c.theta;
    p.psi = c.psi;
    p.fd = c.fd;
    p.beta = c.beta;
    return p;
}

void launch_select(Ctx& c, const HitRec* d_hits, const int32_t* d_nh, int ld, const float* d_q,
                   const sw_request* d_req, int B, uint64_t seed, const sw_selector_config& sel,
                   const sw_policy& pol, sw_choice* d_out, uint32_t extra_flags_mask,
                   cudaStream_t st) {
    (void)d_q;
    (void)extra_flags_mask;
    if (B == 0) return;
    SelParams p = make_sel_params(c, seed, sel, pol);
    StageScope sc(c, SW_STAGE_SELECT, st);
    k_select<<<(B + 63) / 64, 64, 0, st>>>(B, d_hits, d_nh, ld, d_req, p, d_out);
    SW_CUDA(cudaGetLastError());
}

void launch_merge(Ctx& c, const HitRec* d_gathered, const int32_t* d_gn, int world, int B, int k,
                  cudaStream_t st) {
    SW_REQUIRE(world >= 1 && world <= 16, "world size must be in [1, 16]");
    if (B == 0) return;
    StageScope sc(c, SW_STAGE_MERGE, st);
    k_merge<<<(B + 127) / 128, 128, 0, st>>>(B, k, world, d_gathered, d_gn, c.hits, c.nhits);
    SW_CUDA(cudaGetLastError());
}

void launch_score_select_one(Ctx& c, int n, const double* d_sims, const double* d_sneg,
                             const double* d_dur, double L, const sw_selector_config& sel,
                             uint64_t rng_seed, double* d_scores, int32_t* d_pick,
                             cudaStream_t st) {
    (void)c;
    k_score_select_one<<<1, 32, 0, st>>>(n, d_sims, d_sneg, d_dur, L, sel.temperature,
                                         sel.quality_threshold, rng_seed, d_scores, d_pick);
    SW_CUDA(cudaGetLastError());
}

void launch_score_candidates(int n, int D, const double* d_sims, const float* d_audio,
                             const double* d_dur, const float* d_neg, double L, double* d_scores,
                             cudaStream_t st) {
    k_score_candidates<<<1, 32, 0, st>>>(n, D, d_sims, d_audio, d_dur, d_neg, L, d_scores);
    SW_CUDA(cudaGetLastError());
}

void launch_select_draw(int n, const double* d_spos, const double* d_q, double temp, double thr,
                        double u, int32_t* d_pick, cudaStream_t st) {
    k_select_draw<<<1, 32, 0, st>>>(n, d_spos, d_q, temp, thr, u, d_pick);
    SW_CUDA(cudaGetLastError());
}

void launch_gater(Ctx& c, const float* d_p, const float* d_s, const int32_t* d_T, int B,
                  int explore, double* d_phi, int32_t* d_arm, cudaStream_t st) {
    if (B == 0) return;
    k_gater<<<(B + 63) / 64, 64, 0, st>>>(d_p, d_s, d_T, B, c.D, c.theta, c.psi, c.fd, c.beta,
                                         explore, d_phi, d_arm);
    SW_CUDA(cudaGetLastError());
}

}  // namespace sw
