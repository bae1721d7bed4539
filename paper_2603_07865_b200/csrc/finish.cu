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

constexpr int WPB = 4;  // queries (warps) per CTA

struct FinishParams {
    int B, k, rank, implicit_all, n_chunks, cap_local, do_select;
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
    const double* u_draw;
    dev::SelParams sp;
    const sw_request* reqs;
    sw_choice* out;
};

__device__ __forceinline__ bool before(double as, uint64_t aid, double bs, uint64_t bid) {
    return as > bs || (as == bs && aid < bid);
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
    for (int o = 16; o; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, v, o);
        v = x > v ? x : v;
    }
    return v;
}

// fp64 sequential dot of a stored row with the query in shared memory (core.cpp:26-30)
__device__ __forceinline__ double seq_dot4(const float4* __restrict__ rp,
                                           const float4* __restrict__ qs4, int n4) {
    double s = 0.0;
#pragma unroll 4
    for (int d4 = 0; d4 < n4; ++d4) {
        const float4 x = __ldg(rp + d4);
        const float4 y = qs4[d4];
        s = fma((double)y.x, (double)x.x, s);
        s = fma((double)y.y, (double)x.y, s);
        s = fma((double)y.z, (double)x.z, s);
        s = fma((double)y.w, (double)x.w, s);
    }
    return s;
}

// One warp per query: no block barriers, only warp shuffles / ballots.
__global__ void __launch_bounds__(32 * WPB) k_finish(const FinishParams p) {
    extern __shared__ float4 qs_all[];
    __shared__ int64_t sel_slot[WPB][kMaxTopK];
    __shared__ int32_t sel_row[WPB][kMaxTopK];
    __shared__ double sel_sim[WPB][kMaxTopK];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * WPB + warp;
    if (b >= p.B) return;
    const unsigned full = 0xffffffffu;
    float4* qs4 = qs_all + warp * (p.Df >> 2);
    float* qs = reinterpret_cast<float*>(qs4);
    const float* qb = p.q + (int64_t)b * p.D;
    for (int d = lane; d < p.Df; d += 32) qs[d] = d < p.D ? qb[d] : 0.0f;
    __syncwarp();
    const int64_t base = (int64_t)b * kCandCap;

    // ---------------- A: certified candidate set
    int64_t n = 0;
    bool ovf = false;
    if (!p.implicit_all) {
        const int m = p.n_chunks * p.k;
        const float* tk = p.cta_topk + (int64_t)b * p.n_chunks * kMaxTopK;
        unsigned long long prev = ~0ull;
        float kth = -INFINITY;
        for (int r = 0; r < p.k; ++r) {
            unsigned long long best = 0;
            for (int i = lane; i < m; i += 32) {
                const float v = tk[(i / p.k) * kMaxTopK + (i % p.k)];
                if (v == -INFINITY) continue;
                const unsigned long long key =
                    ((unsigned long long)f2ord(v) << 32) | (0xFFFFFFFFu - (uint32_t)i);
                if (key < prev && key > best) best = key;
            }
            best = warp_max_u64(best);
            if (best == 0) {  // fewer than k valid entries in the shard: keep everything
                kth = -INFINITY;
                break;
            }
            prev = best;
            kth = ord2f((uint32_t)(best >> 32));
        }
        const float cut = kth - 2.0f * p.eps_rel * p.q_norm[b] * ord2f(*p.maxnorm);
        for (int c0 = 0; c0 < p.n_chunks; c0 += 32) {
            const int my_cnt = c0 + lane < p.n_chunks
                                   ? p.slice_cnt[(int64_t)b * p.n_chunks + c0 + lane] : 0;
            ovf = ovf || __any_sync(full, my_cnt > p.cap_local);
            const int cmax = min(32, p.n_chunks - c0);
            for (int j = 0; j < cmax; ++j) {
                const int cnt = min(__shfl_sync(full, my_cnt, j), p.cap_local);
                const int64_t src = base + (int64_t)(c0 + j) * p.cap_local;
                for (int i0 = 0; i0 < cnt; i0 += 32) {
                    const int i = i0 + lane;
                    const bool pass = i < cnt && p.cand_score[src + i] >= cut;
                    const unsigned bal = __ballot_sync(full, pass);
                    if (pass) p.list[base + n + __popc(bal & ((1u << lane) - 1u))] = p.cand_slot[src + i];
                    n += __popc(bal);
                }
            }
        }
        __syncwarp();
    } else {
        n = p.n_slots;
    }

    // ---------------- B: exact rescoring, lane = (candidate, pyramid row); 2 chains per lane
    const int64_t items = n << p.logRp;
    const int64_t items_w = (items + 31) & ~int64_t(31);
    const int n4 = p.Df >> 2;
    for (int64_t w0 = lane; w0 < items_w; w0 += 64) {
        double sim[2] = {-DBL_MAX, -DBL_MAX};
        int row[2] = {0x7fffffff, 0x7fffffff};
        const float4* rp[2] = {nullptr, nullptr};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t w = w0 + 32 * h;
            if (w < items) {
                const int64_t i = w >> p.logRp;
                const int r = (int)(w & (p.Rp - 1));
                const int64_t slot = p.implicit_all ? i : (int64_t)p.list[base + i];
                if (p.valid[slot] && r < p.nrows[slot]) {
                    rp[h] = reinterpret_cast<const float4*>(p.rows + (slot * p.Rp + r) * p.Df);
                    row[h] = r;
                }
            }
        }
        // two independent sequential chains interleaved for ILP (each keeps its own order)
        double s0 = 0.0, s1 = 0.0;
        if (rp[0] && rp[1]) {
#pragma unroll 2
            for (int d4 = 0; d4 < n4; ++d4) {
                const float4 x0 = __ldg(rp[0] + d4), x1 = __ldg(rp[1] + d4);
                const float4 y = qs4[d4];
                s0 = fma((double)y.x, (double)x0.x, s0);
                s1 = fma((double)y.x, (double)x1.x, s1);
                s0 = fma((double)y.y, (double)x0.y, s0);
                s1 = fma((double)y.y, (double)x1.y, s1);
                s0 = fma((double)y.z, (double)x0.z, s0);
                s1 = fma((double)y.z, (double)x1.z, s1);
                s0 = fma((double)y.w, (double)x0.w, s0);
                s1 = fma((double)y.w, (double)x1.w, s1);
            }
        } else if (rp[0]) {
            s0 = seq_dot4(rp[0], qs4, n4);
        } else if (rp[1]) {
            s1 = seq_dot4(rp[1], qs4, n4);
        }
        if (rp[0]) sim[0] = fmin(1.0, fmax(-1.0, s0));
        if (rp[1]) sim[1] = fmin(1.0, fmax(-1.0, s1));
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            double sm = sim[h];
            int rw = row[h];
            for (int o = 1; o < p.Rp; o <<= 1) {  // best row: max, ties -> lowest row
                const double os = __shfl_xor_sync(full, sm, o);
                const int orow = __shfl_xor_sync(full, rw, o);
                if (os > sm || (os == sm && orow < rw)) {
                    sm = os;
                    rw = orow;
                }
            }
            const int64_t w = w0 + 32 * h;
            if (w < items && (w & (p.Rp - 1)) == 0) {
                p.exact[base + (w >> p.logRp)] = sm;
                p.best_row[base + (w >> p.logRp)] = rw;
            }
        }
    }
    __syncwarp();

    // ---------------- C: top-k by (sim desc, id asc)
    double prev_sim = DBL_MAX;
    uint64_t prev_id = 0;
    bool have_prev = false;
    int nh = 0;
    for (int r = 0; r < p.k; ++r) {
        double bs = -DBL_MAX;
        uint64_t bid = ~0ull;
        int64_t bslot = -1, bitem = -1;
        for (int64_t i = lane; i < n; i += 32) {
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
            const double os = __shfl_xor_sync(full, bs, o);
            const uint64_t oid = __shfl_xor_sync(full, bid, o);
            const int64_t oslot = __shfl_xor_sync(full, bslot, o);
            const int64_t oitem = __shfl_xor_sync(full, bitem, o);
            if (oslot >= 0 && (bslot < 0 || before(os, oid, bs, bid))) {
                bs = os;
                bid = oid;
                bslot = oslot;
                bitem = oitem;
            }
        }
        if (bslot < 0) break;
        if (lane == 0) {
            sel_slot[warp][nh] = bslot;
            sel_row[warp][nh] = p.best_row[base + bitem];
            sel_sim[warp][nh] = bs;
        }
        ++nh;
        prev_sim = bs;
        prev_id = bid;
        have_prev = true;
    }
    __syncwarp();

    // ---------------- D: enrichment (8 lanes per hit)
    HitRec* hb = p.hits + (int64_t)b * kMaxTopK;
    for (int t = lane; t < nh * 8; t += 32) {
        const int h = t >> 3, j = t & 7;
        const int64_t row = sel_slot[warp][h] * p.Rp + sel_row[warp][h];
        const float* rp = p.rows + row * p.Df;
        const size_t lo = (size_t)j * p.D / 8, hi = (size_t)(j + 1) * p.D / 8;
        double s = 0.0;
        for (size_t i = lo; i < hi; ++i) s = fma((double)qs[i], (double)rp[i], s);
        hb[h].phi[j] = s;
        if (j == 0) {
            const sw_segment sg = p.segs[row];
            hb[h].sim = sel_sim[warp][h];
            hb[h].entry_id = p.ids[sel_slot[warp][h]];
            hb[h].level = sg.level;
            hb[h].slot = (int32_t)sel_slot[warp][h];
            hb[h].start_s = sg.start_s;
            hb[h].length_s = sg.length_s;
            hb[h].s_neg = p.sneg[row];
            hb[h].row = sel_row[warp][h];
            hb[h].owner = p.rank;
        }
    }
    const int nh_code = ovf ? -nh - 1 : nh;
    if (lane == 0) p.nhits[b] = nh_code;
    __syncwarp();

    // ---------------- E: gate + select + Skip Gater + t*
    if (p.do_select) {
        const sw_choice c = dev::select_warp(hb, nh_code, p.u_draw[b], p.reqs[b], p.sp, lane);
        if (lane == 0) p.out[b] = c;
    }
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
    kernels += launch_prep(c, d_q, B, d_req, sp ? sp->seed : 0, st);
    if (tc) {
        StageScope sc(c, SW_STAGE_SCORE_TC, st);
        kernels += launch_score_tc(c, B, k, st);
    }
    FinishParams p{};
    p.B = B;
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
    p.u_draw = c.u_draw;
    if (sp) p.sp = *sp;
    p.reqs = d_req;
    p.out = d_out;
    {
        StageScope sc(c, SW_STAGE_FINISH, st);
        k_finish<<<(B + WPB - 1) / WPB, 32 * WPB, sizeof(float) * c.Df * WPB, st>>>(p);
    }
    SW_CUDA(cudaGetLastError());
    c.last_tc = tc ? 1 : 0;
    return kernels + 1;
}

}  // namespace sw
