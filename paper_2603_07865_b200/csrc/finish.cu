// K2 + K3 fused — everything after the tcgen05 scoring pass, one warp per query:
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
    int32_t* dbg;  // [B][8]: emitted, kept, then clock64 deltas per phase (debug stats)
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

constexpr int SCH = 64;         // dims per staged chunk
constexpr int SPAD = SCH + 4;   // row stride 272 B: 16 B aligned for cp.async, and the 8 lanes of
                                // each LDS.128 phase hit disjoint banks (row l -> banks 4l..4l+3)
constexpr int SMAXC = 256;      // candidates whose exact results stay in shared memory

struct WarpSmem {
    float stage[2][32][SPAD];  // double-buffered: 32 candidate rows x one 64-dim chunk
    int32_t pref[160];         // prefix of emission-slice sizes
    double ex[SMAXC];          // exact similarity per candidate
    int32_t slot[SMAXC];
    int32_t brow[SMAXC];
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// One warp per query: no block barriers, only warp shuffles / ballots.
__global__ void __launch_bounds__(32 * WPB) k_finish(const FinishParams p) {
    extern __shared__ float4 dyn[];
    __shared__ int64_t sel_slot[WPB][kMaxTopK];
    __shared__ int32_t sel_row[WPB][kMaxTopK];
    __shared__ double sel_sim[WPB][kMaxTopK];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * WPB + warp;
    if (b >= p.B) return;
    const unsigned full = 0xffffffffu;
    WarpSmem& W = reinterpret_cast<WarpSmem*>(dyn)[warp];
    double* qd = reinterpret_cast<double*>(reinterpret_cast<WarpSmem*>(dyn) + WPB) + warp * p.Df;
    const float* qb = p.q + (int64_t)b * p.D;
    for (int d = lane; d < p.Df; d += 32) qd[d] = d < p.D ? (double)qb[d] : 0.0;
    __syncwarp();
    const int64_t base = (int64_t)b * kCandCap;
    const long long t_start = clock64();
    int emitted = 0;

    // ---------------- A: certified candidate set
    int64_t n = 0;
    bool ovf = false;
    if (!p.implicit_all) {
        // T_a = k-th best approx entry score over the union of the scoring CTAs' final lists
        const int m = p.n_chunks * p.k;
        const float* tk = p.cta_topk + (int64_t)b * p.n_chunks * kMaxTopK;
        float vals[8];
        int nv = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {  // m <= 256 stays in registers (148 CTAs x 8 = 1184 max)
            const int i = lane + 32 * u;
            vals[u] = i < m ? tk[(i / p.k) * kMaxTopK + (i % p.k)] : -INFINITY;
        }
        nv = min(8, (m + 31) / 32);
        unsigned long long prev = ~0ull;
        float kth = -INFINITY;
        for (int r = 0; r < p.k; ++r) {
            unsigned long long best = 0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (u >= nv || vals[u] == -INFINITY) continue;
                const unsigned long long key = ((unsigned long long)f2ord(vals[u]) << 32) |
                                               (0xFFFFFFFFu - (uint32_t)(lane + 32 * u));
                if (key < prev && key > best) best = key;
            }
            for (int i = lane + 256; i < m; i += 32) {  // rare: more than 256 list values
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
        // prefix sums of the slice sizes, then one flattened pass with many loads in flight
        int run = 0;
        for (int c0 = 0; c0 < p.n_chunks; c0 += 32) {
            const int raw = c0 + lane < p.n_chunks
                                ? p.slice_cnt[(int64_t)b * p.n_chunks + c0 + lane] : 0;
            ovf = ovf || __any_sync(full, raw > p.cap_local);
            int v = min(raw, p.cap_local);
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(full, v, o);
                if (lane >= o) v += t;
            }
            if (c0 + lane < p.n_chunks) W.pref[c0 + lane + 1] = run + v;
            run += __shfl_sync(full, v, 31);
        }
        if (lane == 0) W.pref[0] = 0;
        __syncwarp();
        const int T = run;
        emitted = T;
        for (int t0 = 0; t0 < T; t0 += 32 * 8) {
            float sc[8];
            int64_t at[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int t = t0 + 32 * u + lane;
                sc[u] = -INFINITY;
                at[u] = -1;
                if (t < T) {
                    int lo = 0, hi = p.n_chunks;  // chunk c with pref[c] <= t < pref[c+1]
                    while (hi - lo > 1) {
                        const int mid = (lo + hi) >> 1;
                        if (W.pref[mid] <= t) lo = mid; else hi = mid;
                    }
                    at[u] = base + (int64_t)lo * p.cap_local + (t - W.pref[lo]);
                    sc[u] = p.cand_score[at[u]];
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const bool pass = at[u] >= 0 && sc[u] >= cut;
                const unsigned bal = __ballot_sync(full, pass);
                if (pass) {
                    const int64_t j = n + __popc(bal & ((1u << lane) - 1u));
                    const int32_t sl = p.cand_slot[at[u]];
                    p.list[base + j] = sl;
                    if (j < SMAXC) W.slot[j] = sl;
                }
                n += __popc(bal);
            }
        }
        __syncwarp();
    } else {
        n = p.n_slots;
    }

    const long long t_a = clock64();
    // ---------------- B: exact rescoring. Items = (candidate, pyramid row); 32 items per round,
    // their rows staged cooperatively (coalesced, all loads in flight) 128 dims at a time into
    // padded shared memory; lane l then runs ITS row's sequential fp64 chain.
    const int64_t items = n << p.logRp;
    for (int64_t g0 = 0; g0 < items; g0 += 32) {
        const int64_t w = g0 + lane;
        const int64_t i = w >> p.logRp;
        const int r = (int)(w & (p.Rp - 1));
        int64_t row = -1;
        if (w < items) {
            const int64_t slot = p.implicit_all ? i
                                 : (i < SMAXC ? (int64_t)W.slot[i] : (int64_t)p.list[base + i]);
            if (p.valid[slot] && r < p.nrows[slot]) row = slot * p.Rp + r;
        }
        double s = 0.0;
        const int nch = (p.Df + SCH - 1) / SCH;
        auto issue = [&](int ch) {  // 32 rows x 64 dims, 16 B per lane per row, all in flight
            const int d0 = ch * SCH;
            const int dn = min(SCH, p.Df - d0);
            for (int j = 0; j < 32; ++j) {
                const int64_t rj = __shfl_sync(full, row, j);
                if (rj >= 0 && 4 * lane < dn)
                    cp_async16(&W.stage[ch & 1][j][4 * lane], p.rows + rj * p.Df + d0 + 4 * lane);
            }
            cp_async_commit();
        };
        __syncwarp();
        issue(0);
        for (int ch = 0; ch < nch; ++ch) {
            if (ch + 1 < nch) {
                issue(ch + 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncwarp();
            if (row >= 0) {
                const int d0 = ch * SCH;
                const int dn4 = min(SCH, p.Df - d0) >> 2;
                const float4* sr4 = reinterpret_cast<const float4*>(&W.stage[ch & 1][lane][0]);
                const double* qq = qd + d0;
                for (int d4 = 0; d4 < dn4; ++d4) {  // sequential order i = 0..D-1
                    const float4 x = sr4[d4];
                    s = fma(qq[4 * d4 + 0], (double)x.x, s);
                    s = fma(qq[4 * d4 + 1], (double)x.y, s);
                    s = fma(qq[4 * d4 + 2], (double)x.z, s);
                    s = fma(qq[4 * d4 + 3], (double)x.w, s);
                }
            }
            __syncwarp();  // the buffer is refilled two chunks later
        }
        double sim = row >= 0 ? fmin(1.0, fmax(-1.0, s)) : -DBL_MAX;
        int rw = row >= 0 ? r : 0x7fffffff;
        for (int o = 1; o < p.Rp; o <<= 1) {  // best row: max, ties -> lowest row
            const double os = __shfl_xor_sync(full, sim, o);
            const int orow = __shfl_xor_sync(full, rw, o);
            if (os > sim || (os == sim && orow < rw)) {
                sim = os;
                rw = orow;
            }
        }
        if (w < items && r == 0) {
            if (i < SMAXC) {
                W.ex[i] = sim;
                W.brow[i] = rw;
                if (p.implicit_all) W.slot[i] = (int32_t)i;
            } else {
                p.exact[base + i] = sim;
                p.best_row[base + i] = rw;
            }
        }
    }
    __syncwarp();

    const long long t_b = clock64();
    // ---------------- C: top-k by (sim desc, id asc)
    double prev_sim = DBL_MAX;
    uint64_t prev_id = 0;
    bool have_prev = false;
    int nh = 0;
    for (int r = 0; r < p.k; ++r) {
        double bs = -DBL_MAX;
        uint64_t bid = ~0ull;
        int64_t bslot = -1;
        int brw = 0;
        for (int64_t i = lane; i < n; i += 32) {
            const bool sm = i < SMAXC;
            const int64_t slot = sm ? (int64_t)W.slot[i]
                                    : (p.implicit_all ? i : (int64_t)p.list[base + i]);
            const double s = sm ? W.ex[i] : p.exact[base + i];
            if (s == -DBL_MAX) continue;  // invalid slot or entry without rows
            const uint64_t id = p.ids[slot];
            if (have_prev && !before(prev_sim, prev_id, s, id)) continue;
            if (bslot < 0 || before(s, id, bs, bid)) {
                bs = s;
                bid = id;
                bslot = slot;
                brw = sm ? W.brow[i] : p.best_row[base + i];
            }
        }
        for (int o = 16; o; o >>= 1) {
            const double os = __shfl_xor_sync(full, bs, o);
            const uint64_t oid = __shfl_xor_sync(full, bid, o);
            const int64_t oslot = __shfl_xor_sync(full, bslot, o);
            const int orw = __shfl_xor_sync(full, brw, o);
            if (oslot >= 0 && (bslot < 0 || before(os, oid, bs, bid))) {
                bs = os;
                bid = oid;
                bslot = oslot;
                brw = orw;
            }
        }
        if (bslot < 0) break;
        if (lane == 0) {
            sel_slot[warp][nh] = bslot;
            sel_row[warp][nh] = brw;
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
        for (size_t i = lo; i < hi; ++i) s = fma(qd[i], (double)rp[i], s);
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
    const long long t_d = clock64();

    // ---------------- E: gate + select + Skip Gater + t*
    if (p.do_select) {
        const sw_choice c = dev::select_warp(hb, nh_code, p.u_draw[b], p.reqs[b], p.sp, lane);
        if (lane == 0) p.out[b] = c;
    }
    if (lane == 0) {
        int32_t* d = p.dbg + (int64_t)b * 8;
        d[0] = emitted;
        d[1] = (int32_t)n;
        d[2] = (int32_t)(t_a - t_start);
        d[3] = (int32_t)(t_b - t_a);
        d[4] = (int32_t)(t_d - t_b);
        d[5] = (int32_t)(clock64() - t_d);
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
    p.dbg = c.dbg;
    if (sp) p.sp = *sp;
    p.reqs = d_req;
    p.out = d_out;
    {
        StageScope sc(c, SW_STAGE_FINISH, st);
        const size_t smem = sizeof(WarpSmem) * WPB + sizeof(double) * c.Df * WPB;
        static size_t attr = 0;
        if (smem > attr) {
            SW_CUDA(cudaFuncSetAttribute(k_finish, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
            attr = smem;
        }
        k_finish<<<(B + WPB - 1) / WPB, 32 * WPB, smem, st>>>(p);
    }
    SW_CUDA(cudaGetLastError());
    c.last_tc = tc ? 1 : 0;
    return kernels + 1;
}

}  // namespace sw
