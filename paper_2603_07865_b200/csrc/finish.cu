// K2 + K3 fused — everything after the tcgen05 scoring pass, one CTA per query:
//
//  A  certified candidates: T_a = k-th best approximate entry score, taken from the union of the
//     scoring CTAs' final running lists (the global top-k is inside that union), then every
//     emitted entry with approx >= T_a - 2 eps_q (in brute-force mode: every valid slot)
//  B  exact fp64 rescoring of all pyramid rows of each candidate: sequential dot in order
//     i = 0..D-1 (core.cpp:26-30; fp32 x fp32 products are exact in fp64 so fma() rounds like
//     mul-then-add), clamp (core.cpp:35-36), best row per entry by strict '>' in pyramid order
//     (index.cpp:311)
//  C  top-k by (sim desc, id asc) and truncation (index.cpp:320-324)
//  D  enrichment: s_neg of the hit row (selector.cpp:41-42, precomputed at insert) and the 8 gater
//     block sums (gater.cpp:18-26) -> 128-byte HitRec (the multi-GPU all-gather record)
//  E  (optional) score_candidates + select + context_features + choose_arm + t* (select_dev.cuh)
#include <cfloat>

#include "select_dev.cuh"

namespace sw {

namespace {

constexpr int FT = 256;  // threads per query CTA

struct FinishParams {
    int k, rank, implicit_all, n_chunks, cap_local, do_select;
    int64_t n_slots;
    const int32_t* slice_cnt;
    const int32_t* cand_slot;
    const float* cand_score;
    const float* cta_topk;
    const float* q_norm;
    const uint32_t* maxnorm;
    float eps_rel;
    const float* q;
    int D, Df, Rp, logRp;
    const float* rows;
    const int32_t* nrows;
    const uint8_t* valid;
    const uint64_t* ids;
    const sw_segment* segs;
    const double* sneg;
    int32_t* list;
    double* exact;
    int32_t* best_row;
    HitRec* hits;
    int32_t* nhits;
    dev::SelParams sp;
    const sw_request* reqs;
    sw_choice* out;
};

__device__ __forceinline__ bool before(double as, uint64_t aid, double bs, uint64_t bid) {
    return as > bs || (as == bs && aid < bid);
}

// block-wide max of a 64-bit key (all threads get the result)
__device__ __forceinline__ unsigned long long block_max_u64(unsigned long long v,
                                                            unsigned long long* sh) {
    for (int o = 16; o; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, v, o);
        v = x > v ? x : v;
    }
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < (FT >> 5) ? sh[threadIdx.x] : 0ull;
        for (int o = 16; o; o >>= 1) {
            const unsigned long long x = __shfl_xor_sync(0xffffffffu, v, o);
            v = x > v ? x : v;
        }
        if (threadIdx.x == 0) sh[32] = v;
    }
    __syncthreads();
    v = sh[32];
    __syncthreads();
    return v;
}

__global__ void __launch_bounds__(FT) k_finish(const FinishParams p) {
    extern __shared__ float4 qs4[];
    float* qs = reinterpret_cast<float*>(qs4);
    __shared__ unsigned long long red[33];
    __shared__ int s_n, s_ovf;
    __shared__ double s_sim[FT / 32];
    __shared__ uint64_t s_id[FT / 32];
    __shared__ int64_t s_slot[FT / 32], s_item[FT / 32];
    __shared__ int64_t sel_slot[kMaxTopK];
    __shared__ int32_t sel_row[kMaxTopK];
    __shared__ double sel_sim[kMaxTopK];
    __shared__ int sel_n;
    const int b = blockIdx.x;
    const float* qb = p.q + (int64_t)b * p.D;
    for (int d = threadIdx.x; d < p.Df; d += FT) qs[d] = d < p.D ? qb[d] : 0.0f;
    if (threadIdx.x == 0) {
        s_n = 0;
        s_ovf = 0;
        sel_n = 0;
    }
    __syncthreads();
    const int64_t base = (int64_t)b * kCandCap;

    // ---------------- A: certified candidate set
    int64_t n;
    if (!p.implicit_all) {
        const int m = p.n_chunks * p.k;
        const float* tk = p.cta_topk + (int64_t)b * p.n_chunks * kMaxTopK;
        unsigned long long prev = ~0ull;
        float kth = -INFINITY;
        for (int r = 0; r < p.k; ++r) {
            unsigned long long best = 0;
            for (int i = threadIdx.x; i < m; i += FT) {
                const float v = tk[(i / p.k) * kMaxTopK + (i % p.k)];
                if (v == -INFINITY) continue;
                const unsigned long long key =
                    ((unsigned long long)f2ord(v) << 32) | (0xFFFFFFFFu - (uint32_t)i);
                if (key < prev && key > best) best = key;
            }
            best = block_max_u64(best, red);
            if (best == 0) {  // fewer than k valid entries in the whole shard: keep all
                kth = -INFINITY;
                break;
            }
            prev = best;
            kth = ord2f((uint32_t)(best >> 32));
        }
        const float cut = kth - 2.0f * p.eps_rel * p.q_norm[b] * ord2f(*p.maxnorm);
        for (int c = 0; c < p.n_chunks; ++c) {
            const int cnt = p.slice_cnt[(int64_t)b * p.n_chunks + c];
            const int mc = min(cnt, p.cap_local);
            if (cnt > p.cap_local && threadIdx.x == 0) s_ovf = 1;
            const int64_t src = base + (int64_t)c * p.cap_local;
            for (int i = threadIdx.x; i < mc; i += FT) {
                if (p.cand_score[src + i] >= cut) {
                    const int j = atomicAdd(&s_n, 1);
                    p.list[base + j] = p.cand_slot[src + i];
                }
            }
        }
        __syncthreads();
        n = s_n;
    } else {
        n = p.n_slots;
    }

    // ---------------- B: exact rescoring, one thread per (candidate, pyramid row)
    const int64_t items = n << p.logRp;
    const int64_t items_w = (items + 31) & ~int64_t(31);  // whole warps: shuffles converge
    for (int64_t w = threadIdx.x; w < items_w; w += FT) {
        const int64_t i = w >> p.logRp;
        const int r = (int)(w & (p.Rp - 1));
        double sim = -DBL_MAX;
        int row = 0x7fffffff;
        if (w < items) {
            const int64_t slot = p.implicit_all ? i : (int64_t)p.list[base + i];
            if (p.valid[slot] && r < p.nrows[slot]) {
                const float4* rp =
                    reinterpret_cast<const float4*>(p.rows + (slot * p.Rp + r) * p.Df);
                double s = 0.0;
#pragma unroll 4
                for (int d4 = 0; d4 < (p.Df >> 2); ++d4) {
                    const float4 x = __ldg(rp + d4);
                    const float4 y = qs4[d4];
                    s = fma((double)y.x, (double)x.x, s);
                    s = fma((double)y.y, (double)x.y, s);
                    s = fma((double)y.z, (double)x.z, s);
                    s = fma((double)y.w, (double)x.w, s);
                }
                sim = fmin(1.0, fmax(-1.0, s));
                row = r;
            }
        }
        for (int o = 1; o < p.Rp; o <<= 1) {
            const double os = __shfl_xor_sync(0xffffffffu, sim, o);
            const int orow = __shfl_xor_sync(0xffffffffu, row, o);
            if (os > sim || (os == sim && orow < row)) {
                sim = os;
                row = orow;
            }
        }
        if (w < items && r == 0) {
            p.exact[base + i] = sim;
            p.best_row[base + i] = row;
        }
    }
    __syncthreads();

    // ---------------- C: top-k, (sim desc, id asc)
    double prev_sim = DBL_MAX;
    uint64_t prev_id = 0;
    bool have_prev = false;
    for (int r = 0; r < p.k; ++r) {
        double bs = -DBL_MAX;
        uint64_t bid = ~0ull;
        int64_t bslot = -1, bitem = -1;
        for (int64_t i = threadIdx.x; i < n; i += FT) {
            const int64_t slot = p.implicit_all ? i : (int64_t)p.list[base + i];
            if (p.implicit_all && !p.valid[slot]) continue;
            const double s = p.exact[base + i];
            if (s == -DBL_MAX) continue;  // entry had no rows
            const uint64_t id = p.ids[slot];
            if (have_prev && !before(prev_sim, prev_id, s, id)) continue;
            if (bslot < 0 || before(s, id, bs, bid)) {
                bs = s;
                bid = id;
                bslot = slot;
                bitem = i;
            }
        }
        for (int o = 16; o; o >>= 1) {
            const double os = __shfl_xor_sync(0xffffffffu, bs, o);
            const uint64_t oid = __shfl_xor_sync(0xffffffffu, bid, o);
            const int64_t oslot = __shfl_xor_sync(0xffffffffu, bslot, o);
            const int64_t oitem = __shfl_xor_sync(0xffffffffu, bitem, o);
            if (oslot >= 0 && (bslot < 0 || before(os, oid, bs, bid))) {
                bs = os;
                bid = oid;
                bslot = oslot;
                bitem = oitem;
            }
        }
        if ((threadIdx.x & 31) == 0) {
            s_sim[threadIdx.x >> 5] = bs;
            s_id[threadIdx.x >> 5] = bid;
            s_slot[threadIdx.x >> 5] = bslot;
            s_item[threadIdx.x >> 5] = bitem;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int w0 = -1;
            for (int w = 0; w < FT / 32; ++w) {
                if (s_slot[w] < 0) continue;
                if (w0 < 0 || before(s_sim[w], s_id[w], s_sim[w0], s_id[w0])) w0 = w;
            }
            if (w0 >= 0) {
                sel_slot[sel_n] = s_slot[w0];
                sel_row[sel_n] = p.best_row[base + s_item[w0]];
                sel_sim[sel_n] = s_sim[w0];
                red[0] = s_id[w0];
                sel_n++;
            }
            red[1] = w0 >= 0 ? 1 : 0;
        }
        __syncthreads();
        if (red[1] == 0) break;
        prev_sim = sel_sim[sel_n - 1];
        prev_id = red[0];
        have_prev = true;
        __syncthreads();
    }
    __syncthreads();
    const int nh = sel_n;

    // ---------------- D: enrichment (8 threads per hit)
    HitRec* hb = p.hits + (int64_t)b * kMaxTopK;
    for (int t = threadIdx.x; t < nh * 8; t += FT) {
        const int h = t >> 3, j = t & 7;
        const int64_t row = sel_slot[h] * p.Rp + sel_row[h];
        const float* rp = p.rows + row * p.Df;
        const size_t lo = (size_t)j * p.D / 8, hi = (size_t)(j + 1) * p.D / 8;
        double s = 0.0;
        for (size_t i = lo; i < hi; ++i) s = fma((double)qs[i], (double)rp[i], s);
        hb[h].phi[j] = s;
        if (j == 0) {
            const sw_segment sg = p.segs[row];
            hb[h].sim = sel_sim[h];
            hb[h].entry_id = p.ids[sel_slot[h]];
            hb[h].level = sg.level;
            hb[h].slot = (int32_t)sel_slot[h];
            hb[h].start_s = sg.start_s;
            hb[h].length_s = sg.length_s;
            hb[h].s_neg = p.sneg[row];
            hb[h].row = sel_row[h];
            hb[h].owner = p.rank;
        }
    }
    const int nh_code = s_ovf ? -nh - 1 : nh;
    if (threadIdx.x == 0) p.nhits[b] = nh_code;
    __syncthreads();

    // ---------------- E: gate + select + Skip Gater + t*
    if (p.do_select && threadIdx.x == 0) p.out[b] = dev::select_one(hb, nh_code, p.reqs[b], p.sp);
}

}  // namespace

int launch_score_tc(Ctx& c, int B, int k, cudaStream_t st);

// Search (+ optionally select) for B queries. Results land in c.hits / c.nhits (and d_out).
int launch_search_fused(Ctx& c, const float* d_q, int B, int k, int rank, const sw_request* d_req,
                        const dev::SelParams* sp, sw_choice* d_out, cudaStream_t st) {
    SW_REQUIRE(k >= 1, "search k must be >= 1");  // index.cpp:291
    SW_REQUIRE(k <= kMaxTopK, "top-k above 32 is not supported");
    SW_REQUIRE(B >= 0 && B <= c.Bmax, "batch exceeds the context's max_batch");
    if (B == 0) return 0;
    int kernels = 0;
    const int64_t rows_hw = c.high_water * c.Rp;
    const bool exact_only = (c.cfg.flags & SW_FLAG_EXACT_ONLY) != 0;
    const bool tc = c.tc_ok && !exact_only && c.high_water > 0 &&
                    (rows_hw >= 4096 || (c.cfg.flags & SW_FLAG_TC_ALWAYS));
    if (!tc)
        SW_REQUIRE(c.high_water <= kCandCap,
                   "exact-only search is limited to 16384 slots; enable the tcgen05 path");
    kernels += launch_prep(c, d_q, B, st);
    if (tc) {
        StageScope sc(c, SW_STAGE_SCORE_TC, st);
        kernels += launch_score_tc(c, B, k, st);
    }
    FinishParams p{};
    p.k = k;
    p.rank = rank;
    p.implicit_all = tc ? 0 : 1;
    p.n_chunks = c.last_chunks;
    p.cap_local = kCandCap / c.last_chunks;
    p.do_select = sp != nullptr;
    p.n_slots = c.high_water;
    p.slice_cnt = c.slice_cnt;
    p.cand_slot = c.cand_slot;
    p.cand_score = c.cand_score;
    p.cta_topk = c.cta_topk;
    p.q_norm = c.q_norm;
    p.maxnorm = c.maxnorm;
    p.eps_rel = kEpsRel;
    p.q = d_q;
    p.D = c.D;
    p.Df = c.Df;
    p.Rp = c.Rp;
    p.logRp = c.logRp;
    p.rows = c.rows;
    p.nrows = c.nrows;
    p.valid = c.valid;
    p.ids = c.ids;
    p.segs = c.segs;
    p.sneg = c.sneg;
    p.list = c.cand_list;
    p.exact = c.cand_exact;
    p.best_row = c.cand_row;
    p.hits = c.hits;
    p.nhits = c.nhits;
    if (sp) p.sp = *sp;
    p.reqs = d_req;
    p.out = d_out;
    {
        StageScope sc(c, SW_STAGE_FINISH, st);
        k_finish<<<B, FT, sizeof(float) * c.Df, st>>>(p);
    }
    SW_CUDA(cudaGetLastError());
    c.last_tc = tc ? 1 : 0;
    return kernels + 1;
}

}  // namespace sw
