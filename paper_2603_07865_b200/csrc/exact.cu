// Query preparation and result conversion around IvfIndex::search (index.cpp:289-326).
//
//  k_prep            queries fp32 -> bf16 (K zero-padded) for the tcgen05 pre-filter, |q|,
//                    per-query resets
//  k_hits_to_public  HitRec -> SearchHit (index.hpp:25-29)
// The certified-candidate filter, exact fp64 rescoring and top-k live in finish.cu.
#include <cfloat>

#include "select_dev.cuh"

namespace sw {


namespace {


__global__ void k_prep(const float* __restrict__ q, int B, int D, int Dp,
                       __nv_bfloat16* __restrict__ q_bf, float* __restrict__ q_norm,
                       float* __restrict__ q_eps, const uint32_t* __restrict__ norms,
                       uint32_t* __restrict__ thr, uint32_t* __restrict__ top1) {
    const int b = blockIdx.x;
    if (b >= B) return;
    // the arena's error-bound maxima, loaded first so their latency overlaps the query pass
    uint32_t nrm1 = 0, nrm2 = 0;
    if (threadIdx.x == 0) {
        nrm1 = norms[1];
        nrm2 = norms[2];
    }
    for (int i = threadIdx.x; i < kMaxSlices; i += blockDim.x)
        top1[(int64_t)b * kMaxSlices + i] = f2ord(-INFINITY);
    // (the request's selector draw is computed in k_finish, overlapping its phase A)
    __shared__ double red[3][32];
    const float* qb = q + (int64_t)b * D;
    double nn = 0.0, dd = 0.0, bb = 0.0;
    for (int d = threadIdx.x; d < Dp; d += blockDim.x) {
        const float v = d < D ? qb[d] : 0.0f;
        const __nv_bfloat16 h = __float2bfloat16_rn(v);
        q_bf[(int64_t)b * Dp + d] = h;
        const double x = v, xb = (double)__bfloat162float(h);
        nn += x * x;
        dd += (x - xb) * (x - xb);
        bb += xb * xb;
    }
    for (int o = 16; o; o >>= 1) {
        nn += __shfl_xor_sync(0xffffffffu, nn, o);
        dd += __shfl_xor_sync(0xffffffffu, dd, o);
        bb += __shfl_xor_sync(0xffffffffu, bb, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = nn;
        red[1][threadIdx.x >> 5] = dd;
        red[2][threadIdx.x >> 5] = bb;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t[3] = {0.0, 0.0, 0.0};
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
            for (int j = 0; j < 3; ++j) t[j] += red[j][w];
        const double qn = sqrt(t[0]), qd = sqrt(t[1]), qbn = sqrt(t[2]);
        const double ed = ord2f(nrm1), ebn = ord2f(nrm2);
        const double eps = (qn * ed + qd * ebn + (double)kAccSlack * qbn * ebn) * (1.0 + 1e-5) + 1e-12;
        q_norm[b] = (float)qn * (1.0f + 1e-6f);
        q_eps[b] = (float)eps * (1.0f + 1e-6f);
        thr[b] = f2ord(-INFINITY);
    }
}

__global__ void k_hits_to_public(int B, int k, const HitRec* __restrict__ hits,
                                 const int32_t* __restrict__ nhits, sw_hit* __restrict__ out,
                                 int32_t* __restrict__ out_n) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    // a negative count (-n - 1) would mark an uncertified result; the certified-overflow
    // fallback (k_overflow) rewrites every such query first, so it is passed through as-is
    const int code = nhits[b];
    const int nh = code < 0 ? -code - 1 : code;
    out_n[b] = code;
    for (int i = 0; i < nh; ++i) {
        const HitRec& h = hits[(int64_t)b * kMaxTopK + i];
        sw_hit o;
        o.entry_id = h.entry_id;
        o.segment.level = h.level;
        o.segment.reserved = 0;
        o.segment.start_s = h.start_s;
        o.segment.length_s = h.length_s;
        o.similarity = h.sim;
        out[(int64_t)b * k + i] = o;
    }
}

}  // namespace

int launch_prep(Ctx& c, const float* d_q, int B, const sw_request* d_req, uint64_t seed,
                cudaStream_t st) {
    StageScope sc(c, SW_STAGE_PREP, st);
    k_prep<<<B, 128, 0, st>>>(d_q, B, c.D, c.Dp, c.q_bf, c.q_norm, c.q_eps, c.norms, c.thr, c.top1);
    SW_CUDA(cudaGetLastError());
    return 1;
}

// IvfIndex::search for B queries into c.hits / c.nhits (no select). Returns kernels launched.
int launch_search(Ctx& c, const float* d_q, int B, int k, int rank, cudaStream_t st) {
    return launch_search_fused(c, d_q, B, k, rank, nullptr, nullptr, nullptr, st);
}

void launch_hits_to_public(Ctx& c, int B, int k, sw_hit* d_out, int32_t* d_n, cudaStream_t st) {
    if (B == 0) return;
    k_hits_to_public<<<(B + 127) / 128, 128, 0, st>>>(B, k, c.hits, c.nhits, d_out, d_n);
    SW_CUDA(cudaGetLastError());
}

}  // namespace sw
