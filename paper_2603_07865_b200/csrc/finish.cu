// K2 + K3 fused — everything after the tcgen05 scoring pass, one 2-warp CTA per query:
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
#include <cstdlib>

#include "select_dev.cuh"

namespace sw {

namespace {

constexpr int FT = 64;      // threads per query CTA (2 warps)
constexpr int NWARP = FT / 32;
constexpr int SMAXC = 256;  // candidates whose exact results stay in shared memory
constexpr int SC = 32;      // dims per staged chunk of the rescoring ring
constexpr int SP = SC + 4;  // 144-byte smem rows: 16 B aligned for cp.async; the 8 lanes of each
                            // LDS.128 phase read rows l..l+7 -> banks 4l..4l+3, conflict-free
constexpr int NST = 4;      // ring stages per warp
constexpr int SPHI = 64;    // candidates whose block sums phase B keeps in shared memory

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

struct FinishParams {
    int B, k, rank, implicit_all, n_chunks, cap_local, do_select;
    int64_t n_slots;
    const int32_t* slice_cnt;
    const int32_t* cand_slot;
    const int32_t* sorted_slot;  // grouped IVF: emitted slots are list-sorted rows -> arena slot
    const float* cand_score;
    const float* cta_topk;
    const float* q_eps;
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
    int32_t* dbg;  // [B][8]: emitted, kept, then clock64 deltas per phase (debug stats)
    dev::SelParams sp;
    const sw_request* reqs;
    sw_choice* out;
    int ivf;                  // IVF mode: rows outside the query's probed lists do not count
    const int16_t* row_list;  // [rows] list of each stored row
    const uint8_t* prank;     // [B][kMaxCentroids] probe rank of each list (255: not probed)
    // certified-overflow fallback (k_overflow)
    int32_t* ovf;             // state: header, flagged queries [bmax], chunk done / merged flags
    struct OvfRec* ovf_ring;  // [kOvfRing][kOvfQG][n_warps][kMaxTopK]
    int bmax;
};

// One entry of a fallback top-k list: exact clamped similarity, arena slot, best pyramid row.
struct OvfRec {
    double sim;
    int32_t slot;
    int32_t row;
};

struct FinSmem {
    double ex[SMAXC];  // exact similarity per candidate
    uint64_t id[SMAXC];
    int32_t slot[SMAXC];
    int32_t brow[SMAXC];
    int64_t sel_slot[kMaxTopK];
    int32_t sel_row[kMaxTopK];
    double sel_sim[kMaxTopK];
    HitRec rec[kMaxTopK];  // mirror of the hit records for the select stage
    double phi[SPHI][8];   // gater block sums of the best row of candidates i < SPHI (phase B)
    int32_t sel_idx[kMaxTopK];
    int32_t pre[kMaxSlices + 1];  // exclusive prefix of the slices' emission counts (phase A)
    float cut;
    int n, ovf, nh, emitted;
    long long t_ta, t_sync;
    double u;  // the request's selector draw (computed by warp 1 during phase A)
    uint32_t tsv[256];  // wide-grid T_a: each warp's survivors (>= its local k-th best)
    int tsn;
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

// Sequential fp64 dot (core.cpp:26-30) of a global row with the query (doubles in smem), N4
// float4 steps, with a PF-deep ring of row loads in flight so the chain never waits on memory.
template <int N4, int PF>
__device__ __forceinline__ double chain_dot(const float4* __restrict__ rp,
                                            const double* __restrict__ qd) {
    float4 ring[PF];
#pragma unroll
    for (int i = 0; i < PF; ++i) ring[i] = __ldg(rp + i);
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N4; ++i) {
        const float4 x = ring[i % PF];
        if (i + PF < N4) ring[i % PF] = __ldg(rp + i + PF);
        s = fma(qd[4 * i + 0], (double)x.x, s);
        s = fma(qd[4 * i + 1], (double)x.y, s);
        s = fma(qd[4 * i + 2], (double)x.z, s);
        s = fma(qd[4 * i + 3], (double)x.w, s);
    }
    return s;
}

// chain_dot that also produces the gater's 8 block sums (gater.cpp:18-26: block j is the
// sequential fp64 sum over [j D/8, (j+1) D/8) starting from 0) as a second, independent chain;
// valid when D == Df and D % 32 == 0 (blocks are whole float4 runs).
// The loops are ROLLED (one PF-float4 body, ~130 instructions): a fully unrolled 512-step
// chain is ~32 KB of straight-line code per instantiation that each warp executes once, so
// every instruction fetch missed the instruction cache (measured: phase B 41K cycles cold vs
// 15K with the code cached).
template <int N4, int PF>
__device__ __forceinline__ double chain_dot_phi(const float4* __restrict__ rp,
                                                const double* __restrict__ qd, double (&phi)[8]) {
    constexpr int BS4 = N4 / 8;
    static_assert(BS4 % PF == 0, "ring period divides a block");
    float4 ring[PF];
#pragma unroll
    for (int u = 0; u < PF; ++u) ring[u] = __ldg(rp + u);
#pragma unroll
    for (int j = 0; j < 8; ++j) phi[j] = 0.0;
    double s = 0.0;
#pragma unroll 1
    for (int blk = 0; blk < 8; ++blk) {
        double bsum = 0.0;
#pragma unroll 1
        for (int i0 = blk * BS4; i0 < (blk + 1) * BS4; i0 += PF) {
#pragma unroll
            for (int u = 0; u < PF; ++u) {
                const int i = i0 + u;
                const float4 x = ring[u];
                if (i + PF < N4) ring[u] = __ldg(rp + i + PF);
                const double2 a = reinterpret_cast<const double2*>(qd)[2 * i];
                const double2 b = reinterpret_cast<const double2*>(qd)[2 * i + 1];
                const double x0 = x.x, x1 = x.y, x2 = x.z, x3 = x.w;
                s = fma(a.x, x0, s);
                bsum = fma(a.x, x0, bsum);
                s = fma(a.y, x1, s);
                bsum = fma(a.y, x1, bsum);
                s = fma(b.x, x2, s);
                bsum = fma(b.x, x2, bsum);
                s = fma(b.y, x3, s);
                bsum = fma(b.y, x3, bsum);
            }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) phi[j] = j == blk ? bsum : phi[j];  // static register index
    }
    return s;
}

__device__ __forceinline__ double chain_dot_any(const float4* __restrict__ rp,
                                                const double* __restrict__ qd, int n4) {
    // rolled like chain_dot_phi (instruction-cache footprint), 8 float4 loads in flight
    constexpr int PF = 8;
    float4 ring[PF];
#pragma unroll
    for (int u = 0; u < PF; ++u) ring[u] = u < n4 ? __ldg(rp + u) : make_float4(0.f, 0.f, 0.f, 0.f);
    double s = 0.0;
#pragma unroll 1
    for (int i0 = 0; i0 < n4; i0 += PF) {
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            const int i = i0 + u;
            if (i < n4) {
                const float4 x = ring[u];
                if (i + PF < n4) ring[u] = __ldg(rp + i + PF);
                s = fma(qd[4 * i + 0], (double)x.x, s);
                s = fma(qd[4 * i + 1], (double)x.y, s);
                s = fma(qd[4 * i + 2], (double)x.z, s);
                s = fma(qd[4 * i + 3], (double)x.w, s);
            }
        }
    }
    return s;
}

// k-th largest key (duplicates counted) of a warp's register-held ordered keys (0 = no value):
// descending distinct keys by a warp max (REDUX) below the previous one, then a warp count of
// its copies. 0 when fewer than k keys are real. Warp-uniform result.
template <int NV>
__device__ __forceinline__ uint32_t kth_key(const uint32_t (&key)[NV], int k) {
    const unsigned full = 0xffffffffu;
    uint32_t prev = 0xFFFFFFFFu;
    int total = 0;
    for (;;) {
        uint32_t lm = 0u;
#pragma unroll
        for (int u = 0; u < NV; ++u) lm = max(lm, key[u] < prev ? key[u] : 0u);
        const uint32_t cur = __reduce_max_sync(full, lm);
        if (cur == 0u) return 0u;
        int c = 0;
#pragma unroll
        for (int u = 0; u < NV; ++u) c += key[u] == cur ? 1 : 0;
        total += (int)__reduce_add_sync(full, (unsigned)c);
        prev = cur;
        if (total >= k) return cur;
    }
}

// k-th largest (duplicates counted) of the m <= 32 NV values tk[(i / k) * kMaxTopK + i % k],
// by descending distinct values: a warp max (REDUX) of the keys below the previous one, then a
// warp count of its copies. -inf when fewer than k values are real. Warp-uniform result.
template <int NV>
__device__ __forceinline__ float kth_largest(const float* __restrict__ tk, int m, int k, int lane) {
    const unsigned full = 0xffffffffu;
    const bool pow2 = (k & (k - 1)) == 0;
    const int lk = __ffs(k) - 1;
    uint32_t key[NV];
#pragma unroll
    for (int u = 0; u < NV; ++u) {
        const int i = lane + 32 * u;
        key[u] = 0u;  // below every real score's key
        if (i < m) {
            const int sl = pow2 ? i >> lk : i / k;
            const float v = tk[sl * kMaxTopK + (i - sl * k)];
            if (v != -INFINITY) key[u] = f2ord(v);
        }
    }
    uint32_t prev = 0xFFFFFFFFu;
    int total = 0;
    for (;;) {
        uint32_t lm = 0u;
#pragma unroll
        for (int u = 0; u < NV; ++u) lm = max(lm, key[u] < prev ? key[u] : 0u);
        const uint32_t cur = __reduce_max_sync(full, lm);
        if (cur == 0u) return -INFINITY;  // fewer than k valid entries: keep everything
        int c = 0;
#pragma unroll
        for (int u = 0; u < NV; ++u) c += key[u] == cur ? 1 : 0;
        total += (int)__reduce_add_sync(full, (unsigned)c);
        prev = cur;
        if (total >= k) return ord2f(cur);
    }
}

// FTT threads per query CTA: 64 (2 warps, 7 CTAs/SM: a 1024-query batch is one wave) or, for
// small batches whose per-query latency is the metric, 256 (the flat candidate walk and the
// enrichment spread over 8 warps).
template <bool RING, int FTT = FT>
__global__ void __launch_bounds__(FTT, FTT == 64 ? 7 : 1) k_finish(const FinishParams p) {
    extern __shared__ double qd[];  // query as doubles, Df
    __shared__ FinSmem S;
    const int b = blockIdx.x;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const unsigned full = 0xffffffffu;
    const float* qb = p.q + (int64_t)b * p.D;
    for (int d = t; d < p.Df; d += FTT) qd[d] = d < p.D ? (double)qb[d] : 0.0;
    if (t == 0) {
        S.n = 0;
        S.ovf = 0;
        S.emitted = 0;
    }
    const int64_t base = (int64_t)b * kCandCap;
    const long long t_start = clock64();
    // the request's selector draw Rng(derive_seed(seed, id, 2)).uniform() (pipeline.cpp:211):
    // a 156-step serial MT64 seeding, run by one lane of warp 1 while warp 0 selects T_a
    if (p.do_select && t == 32)
        S.u = dev::uniform_draw(dev::derive_seed(p.sp.seed, p.reqs[b].id, 2, 0));

    // ---------------- A: certified candidate set
    if (!p.implicit_all) {
        if (warp == 1) {
            // meanwhile: exclusive prefix of the slices' emission counts (capped at the slice
            // capacity; an overflowing slice flags the query) into shared memory
            int carry = 0;
            constexpr int kPre = (kMaxSlices + 31) / 32;
            int raws[kPre];  // every count's load in flight at once (one L2 round trip)
#pragma unroll
            for (int u = 0; u < kPre; ++u) {
                const int j = 32 * u + lane;
                const int v = p.slice_cnt[(int64_t)b * p.n_chunks + min(j, p.n_chunks - 1)];
                raws[u] = j < p.n_chunks ? v : 0;
            }
#pragma unroll
            for (int u = 0; u < kPre; ++u) {
                const int j0 = 32 * u;
                if (j0 >= p.n_chunks) break;
                const int j = j0 + lane;
                const int raw = raws[u];
                if (__any_sync(full, raw > p.cap_local) && lane == 0) S.ovf = 1;
                const int c = min(raw, p.cap_local);
                int incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(full, incl, o);
                    if (lane >= o) incl += v;
                }
                if (j < p.n_chunks) S.pre[j] = carry + incl - c;
                carry += __shfl_sync(full, incl, 31);
            }
            if (lane == 0) S.pre[p.n_chunks] = carry;
        }
        bool ta_done = false;
        if constexpr (FTT >= 256) {
            // wide grids (small batches: 148 slices x k): the 8 warps each take 256 of the
            // m <= 2048 slice scores, keep those >= their local k-th best (a superset of the
            // global top-k), and warp 0 selects the exact k-th largest among the survivors
            const int m = p.n_chunks * p.k;
            if (m > 32 * 16 && m <= 8 * 256) {
                const float* tk = p.cta_topk + (int64_t)b * p.n_chunks * kMaxTopK;
                if (t == 0) S.tsn = 0;
                const bool pow2 = (p.k & (p.k - 1)) == 0;
                const int lk = __ffs(p.k) - 1;
                uint32_t key[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int i = warp * 256 + lane + 32 * u;
                    key[u] = 0u;
                    if (i < m) {
                        const int sl = pow2 ? i >> lk : i / p.k;
                        const float v = tk[sl * kMaxTopK + (i - sl * p.k)];
                        if (v != -INFINITY) key[u] = f2ord(v);
                    }
                }
                __syncthreads();  // S.tsn reset
                const uint32_t lw = kth_key<8>(key, p.k);
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (key[u] != 0u && key[u] >= lw) {
                        const int pos = atomicAdd(&S.tsn, 1);
                        if (pos < 256) S.tsv[pos] = key[u];
                    }
                __syncthreads();
                if (S.tsn <= 256) {  // else (many ties) the single-warp path below
                    if (warp == 0) {
                        const int ns = S.tsn;
                        uint32_t sv[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int i = lane + 32 * u;
                            sv[u] = i < ns ? S.tsv[i] : 0u;
                        }
                        const uint32_t c = kth_key<8>(sv, p.k);
                        const float kth = c ? ord2f(c) : -INFINITY;
                        if (lane == 0) {
                            S.cut = kth - 2.0f * p.q_eps[b];
                            S.t_ta = clock64();
                        }
                    }
                    ta_done = true;
                }
            }
        }
        if (warp == 0 && !ta_done) {  // T_a over the union of the scoring CTAs' final lists
            const int m = p.n_chunks * p.k;
            const float* tk = p.cta_topk + (int64_t)b * p.n_chunks * kMaxTopK;
            float kth = -INFINITY;
            if (m <= 32 * 16) {
                kth = kth_largest<16>(tk, m, p.k, lane);
            } else if (m <= 32 * 40) {  // 148 slices x k = 8 (single-query batches)
                kth = kth_largest<40>(tk, m, p.k, lane);
            } else {  // very wide grids (small batches): 64-bit (value, index) keys from L2
                unsigned long long prev = ~0ull;
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
                    if (best == 0) {
                        kth = -INFINITY;
                        break;
                    }
                    prev = best;
                    kth = ord2f((uint32_t)(best >> 32));
                }
            }
            if (lane == 0) S.cut = kth - 2.0f * p.q_eps[b];
            if (lane == 0) S.t_ta = clock64();
        }
        __syncthreads();
        const long long t_sync = clock64();
        const float cut = S.cut;
        const int64_t row_bytes = (int64_t)p.Rp * p.Df * 4;
        // keeps one candidate: shared list (+ global spill list) and an L2 prefetch of its rows
        auto keep = [&](int slot) {
            const int pos = atomicAdd(&S.n, 1);  // list order is irrelevant (phase C sorts)
            if (pos < SMAXC) S.slot[pos] = slot;
            p.list[base + pos] = slot;
            const char* rp = reinterpret_cast<const char*>(p.rows + (int64_t)slot * p.Rp * p.Df);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(rp),
                         "r"((uint32_t)row_bytes)
                         : "memory");
        };
        // The emitted entries of all slices as one flat sequence (slice-major): thread t walks
        // its contiguous share [t L, (t + 1) L), slice by slice, 8 score loads in flight, and
        // loads the slot index only for entries that pass the cut.
        const int total = S.pre[p.n_chunks];
        const int L = (total + FTT - 1) / FTT;
        int f = min(total, t * L);
        const int fend = min(total, f + L);
        int sl = 0;  // slice containing f: the last slice with pre[sl] <= f
        {
            int lo = 0, hi = p.n_chunks - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (S.pre[mid] <= f) lo = mid; else hi = mid - 1;
            }
            sl = lo;
        }
        while (f < fend) {
            while (S.pre[sl + 1] <= f) ++sl;  // skip empty slices
            const int seg_end = min(fend, S.pre[sl + 1]);
            const int64_t src = base + (int64_t)sl * p.cap_local - S.pre[sl];  // + flat index
            for (; f < seg_end; f += 8) {
                float v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = f + u < seg_end ? p.cand_score[src + f + u] : -INFINITY;
#pragma unroll
                for (int u = 0; u < 8; ++u)  // (cut may be -inf: keep every real entry)
                    if (f + u < seg_end && v[u] >= cut) {
                        const int32_t cs = p.cand_slot[src + f + u];
                        keep(p.sorted_slot ? __ldg(p.sorted_slot + cs) : cs);
                    }
            }
            f = seg_end;
        }
        const int emitted = total;
        if (t == 0) {
            S.t_sync = t_sync;
            S.emitted = emitted;
        }
    } else if (t == 0) {
        S.n = (int)p.n_slots;
    }
    __syncthreads();
    const int64_t n = S.n;
    const long long t_a = clock64();

    // ---------------- B: exact rescoring. Warp w takes groups of 32 items (candidate, pyramid
    // row), g = w, w + NWARP, ...; the 32 rows are staged 32 dims at a time through an NST-deep
    // cp.async ring (coalesced 128-byte row segments), and lane l runs ITS row's sequential fp64
    // chain from shared memory.
    const int64_t items = n << p.logRp;
    // block sums ride along phase B for D in {64, 128, 256, 512} (unpadded, whole-float4 blocks)
    const bool fast_phi = !RING && p.D == p.Df && (p.D == 64 || p.D == 128 || p.D == 256 ||
                                                   p.D == 512);
    float* ring = RING ? reinterpret_cast<float*>(qd + p.Df) + (size_t)warp * NST * 32 * SP
                       : nullptr;
    const int nch = (p.Df + SC - 1) / SC;
    for (int64_t g0 = (int64_t)warp * 32; g0 < items; g0 += FTT) {
        const int64_t w = g0 + lane;
        const int64_t i = w >> p.logRp;
        const int r = (int)(w & (p.Rp - 1));
        int64_t row = -1, slot = -1;
        int key = r;  // tie order among an entry's rows (index.cpp:306-311)
        if (w < items) {
            slot = p.implicit_all ? i : (i < SMAXC ? (int64_t)S.slot[i] : (int64_t)p.list[base + i]);
            if (p.valid[slot] && r < p.nrows[slot]) row = slot * p.Rp + r;
            if (row >= 0 && p.ivf) {
                // only rows of probed lists are scanned; lists are visited in probe order and
                // an entry's rows sit in pyramid order inside a list, so the first maximum in
                // scan order is the lowest (probe rank, row)
                const int l = p.row_list[row];
                const int pr = l >= 0 ? p.prank[(int64_t)b * kMaxCentroids + l] : kNotProbed;
                if (pr == kNotProbed)
                    row = -1;
                else
                    key = (pr << 6) | r;
            }
        }
        double s = 0.0;
        double phi[8];
        if constexpr (!RING) {
            // lane l streams ITS row straight from L2 (phase A bulk-prefetched it) with a
            // 16-deep float4 register ring; no shared-memory staging, so 1024 query CTAs fit
            // in one wave. With whole-float4 gater blocks the same pass also yields the block
            // sums (phase D then does not re-read the row)
            if (row >= 0) {
                const float4* rp4 = reinterpret_cast<const float4*>(p.rows + row * p.Df);
                if (fast_phi) {
                    switch (p.D) {
                        // 16 float4 in flight per lane where registers allow (the 8-warp
                        // small-batch CTAs: B=1 phase B 28K -> 22K cycles); 8 in the 2-warp
                        // CTAs held to 128 registers (16 measured 30K -> 40K there)
                        case 512: s = chain_dot_phi<128, (FTT >= 256 ? 16 : 8)>(rp4, qd, phi); break;
                        case 256: s = chain_dot_phi<64, 8>(rp4, qd, phi); break;
                        case 128: s = chain_dot_phi<32, 4>(rp4, qd, phi); break;
                        default: s = chain_dot_phi<16, 2>(rp4, qd, phi); break;
                    }
                } else {
                    s = chain_dot_any(rp4, qd, p.Df >> 2);
                }
            }
        } else {
            // lane l stages float4 (l & 7) of rows (l >> 3) + 4u, u = 0..7
            const float* src[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t rj = __shfl_sync(full, row, (lane >> 3) + 4 * u);
                src[u] = rj >= 0 ? p.rows + rj * p.Df + 4 * (lane & 7) : nullptr;
            }
            auto issue = [&](int ch) {
                if (ch < nch) {
                    const int d0 = ch * SC;
                    float* dst = ring + (size_t)(ch % NST) * 32 * SP + 4 * (lane & 7);
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (src[u] && d0 + 4 * (lane & 7) < p.Df)
                            cp_async16(dst + ((lane >> 3) + 4 * u) * SP, src[u] + d0);
                }
                cp_async_commit();  // empty groups keep the wait count uniform
            };
            __syncwarp();
#pragma unroll
            for (int c = 0; c < NST - 1; ++c) issue(c);
            s = 0.0;
            for (int ch = 0; ch < nch; ++ch) {
                issue(ch + NST - 1);
                cp_async_wait<NST - 1>();
                __syncwarp();
                if (row >= 0) {
                    const float4* sr4 =
                        reinterpret_cast<const float4*>(ring + ((size_t)(ch % NST) * 32 + lane) * SP);
                    const double* qq = qd + ch * SC;
                    const int dn4 = min(SC, p.Df - ch * SC) >> 2;
#pragma unroll
                    for (int d4 = 0; d4 < SC / 4; ++d4) {  // sequential order i = 0..D-1
                        if (d4 < dn4) {
                            const float4 x = sr4[d4];
                            s = fma(qq[4 * d4 + 0], (double)x.x, s);
                            s = fma(qq[4 * d4 + 1], (double)x.y, s);
                            s = fma(qq[4 * d4 + 2], (double)x.z, s);
                            s = fma(qq[4 * d4 + 3], (double)x.w, s);
                        }
                    }
                }
                __syncwarp();  // this ring slot is refilled NST - 1 chunks later
            }
        }
        double sim = row >= 0 ? fmin(1.0, fmax(-1.0, s)) : -DBL_MAX;  // core.cpp:35-36
        int rw = row >= 0 ? key : 0x7fffffff;
        for (int o = 1; o < p.Rp; o <<= 1) {  // best row: max, ties -> lowest key (index.cpp:311)
            const double os = __shfl_xor_sync(full, sim, o);
            const int orow = __shfl_xor_sync(full, rw, o);
            if (os > sim || (os == sim && orow < rw)) {
                sim = os;
                rw = orow;
            }
        }
        if (rw != 0x7fffffff) rw &= 63;  // key -> row index
        if constexpr (!RING) {
            if (fast_phi && w < items && i < SPHI && row >= 0 && r == rw) {
#pragma unroll
                for (int j = 0; j < 8; ++j) S.phi[i][j] = phi[j];
            }
        }
        if (w < items && r == 0) {
            if (i < SMAXC) {
                S.ex[i] = sim;
                S.brow[i] = rw;
                S.slot[i] = (int32_t)slot;
                S.id[i] = p.ids[slot];
            } else {
                p.exact[base + i] = sim;
                p.best_row[base + i] = rw;
            }
        }
    }
    __syncthreads();
    const long long t_b = clock64();

    // ---------------- C: top-k by (sim desc, id asc) (index.cpp:320-324), warp 0
    if (warp == 0 && n <= 32) {
        // one candidate per lane: its rank is the number of lanes ordered before it (31
        // independent shuffle rounds, no dependent reduction chain); ranks < k are the hits.
        // ids are unique, so ranks are distinct.
        const bool v = lane < n && S.ex[lane] != -DBL_MAX;  // invalid slot / entry without rows
        const double sv = v ? S.ex[lane] : -DBL_MAX;
        const uint64_t id = v ? S.id[lane] : ~0ull;
        int rank = 0;
#pragma unroll 4
        for (int r = 1; r < 32; ++r) {
            const int j = (lane + r) & 31;
            const double os = __shfl_sync(full, sv, j);
            const uint64_t oid = __shfl_sync(full, id, j);
            const bool ov = __shfl_sync(full, v, j);
            rank += (ov && before(os, oid, sv, id)) ? 1 : 0;
        }
        if (v && rank < p.k) {
            S.sel_slot[rank] = S.slot[lane];
            S.sel_row[rank] = S.brow[lane];
            S.sel_sim[rank] = sv;
            S.sel_idx[rank] = lane;
        }
        const int nv = __popc(__ballot_sync(full, v));
        if (lane == 0) S.nh = min(nv, p.k);
    } else if (warp == 0) {
        double prev_sim = DBL_MAX;
        uint64_t prev_id = 0;
        bool have_prev = false;
        int nh = 0;
        for (int r = 0; r < p.k; ++r) {
            double bs = -DBL_MAX;
            uint64_t bid = ~0ull;
            int64_t bslot = -1;
            int brw = 0, bidx = 0;
            for (int64_t i = lane; i < n; i += 32) {
                const bool sm = i < SMAXC;
                const double sv = sm ? S.ex[i] : p.exact[base + i];
                if (sv == -DBL_MAX) continue;  // invalid slot or entry without rows
                const int64_t slot = sm ? (int64_t)S.slot[i]
                                        : (p.implicit_all ? i : (int64_t)p.list[base + i]);
                const uint64_t id = sm ? S.id[i] : p.ids[slot];
                if (have_prev && !before(prev_sim, prev_id, sv, id)) continue;
                if (bslot < 0 || before(sv, id, bs, bid)) {
                    bs = sv;
                    bid = id;
                    bslot = slot;
                    brw = sm ? S.brow[i] : p.best_row[base + i];
                    bidx = (int)i;
                }
            }
            for (int o = 16; o; o >>= 1) {
                const double os = __shfl_xor_sync(full, bs, o);
                const uint64_t oid = __shfl_xor_sync(full, bid, o);
                const int64_t oslot = __shfl_xor_sync(full, bslot, o);
                const int orw = __shfl_xor_sync(full, brw, o);
                const int oidx = __shfl_xor_sync(full, bidx, o);
                if (oslot >= 0 && (bslot < 0 || before(os, oid, bs, bid))) {
                    bs = os;
                    bid = oid;
                    bslot = oslot;
                    brw = orw;
                    bidx = oidx;
                }
            }
            if (bslot < 0) break;
            if (lane == 0) {
                S.sel_slot[nh] = bslot;
                S.sel_row[nh] = brw;
                S.sel_sim[nh] = bs;
                S.sel_idx[nh] = bidx;
            }
            ++nh;
            prev_sim = bs;
            prev_id = bid;
            have_prev = true;
        }
        if (lane == 0) S.nh = nh;
    }
    __syncthreads();
    const int nh = S.nh;

    // ---------------- D: enrichment (8 threads per hit): s_neg + gater block sums
    HitRec* hb = p.hits + (int64_t)b * kMaxTopK;
    for (int tt = t; tt < nh * 8; tt += FTT) {
        const int h = tt >> 3, j = tt & 7;
        const int64_t row = S.sel_slot[h] * p.Rp + S.sel_row[h];
        const float* rp = p.rows + row * p.Df;
        const size_t lo = (size_t)j * p.D / 8, hi = (size_t)(j + 1) * p.D / 8;
        sw_segment sg;
        double sn = 0.0;
        uint64_t eid = 0;
        if (j == 0) {  // issued before the chain so their latency overlaps it
            sg = p.segs[row];
            sn = p.sneg[row];
            eid = p.ids[S.sel_slot[h]];
        }
        double s = 0.0;
        if (fast_phi && S.sel_idx[h] < SPHI) {
            s = S.phi[S.sel_idx[h]][j];  // computed by phase B from the same row
        } else if ((p.D & 31) == 0 && hi - lo == 64 && (lo & 3) == 0) {
            s = chain_dot<16, 16>(reinterpret_cast<const float4*>(rp + lo), qd + lo);
        } else {
            for (size_t i = lo; i < hi; ++i) s = fma(qd[i], (double)rp[i], s);
        }
        S.rec[h].phi[j] = s;
        if (j == 0) {
            HitRec& o = S.rec[h];
            o.sim = S.sel_sim[h];
            o.entry_id = eid;
            o.level = sg.level;
            o.slot = (int32_t)S.sel_slot[h];
            o.start_s = sg.start_s;
            o.length_s = sg.length_s;
            o.s_neg = sn;
            o.row = S.sel_row[h];
            o.owner = p.rank;
        }
    }
    const int nh_code = S.ovf ? -nh - 1 : nh;
    if (t == 0) p.nhits[b] = nh_code;
    // an overflowing slice dropped candidates: hand the query to the exact fallback (k_overflow,
    // next on this stream), which replaces its records and choice with a certified result
    if (t == 0 && S.ovf) p.ovf[kOvfHdr + atomicAdd(&p.ovf[0], 1)] = b;
    __syncthreads();
    {  // copy the smem records out (16-byte words)
        const int nw = nh * (int)(sizeof(HitRec) / 16);
        const int4* srcw = reinterpret_cast<const int4*>(S.rec);
        int4* dstw = reinterpret_cast<int4*>(hb);
        for (int i = t; i < nw; i += FTT) dstw[i] = srcw[i];
    }
    const long long t_d = clock64();

    // ---------------- E: gate + select + Skip Gater + t* (warp 0)
    if (p.do_select && warp == 0) {  // (phase D covered 8 hits x 8 block sums in one pass)
        const sw_choice c = dev::select_warp(S.rec, nh_code, S.u, p.reqs[b], p.sp, lane);
        if (lane == 0) p.out[b] = c;
    }
    if (t == 0) {
        int32_t* d = p.dbg + (int64_t)b * 8;
        d[0] = S.emitted;
        d[1] = (int32_t)n;
        d[2] = (int32_t)(t_a - t_start);
        d[3] = (int32_t)(t_b - t_a);
        d[4] = (int32_t)(t_d - t_b);
        d[5] = (int32_t)(clock64() - t_d);
        if (!p.implicit_all) {  // phase A split: T_a selection, barrier wait
            d[6] = (int32_t)(S.t_ta - t_start);
            d[7] = (int32_t)(S.t_sync - t_start);
        }
    }
}

// ------------------------------------------------------------------------------------------
// Certified-overflow fallback. A query whose candidate slices overflowed (more emissions than a
// slice holds, e.g. thousands of identical rows in its range) lost candidates, so k_finish's
// result for it is not certified. This kernel recomputes such queries exactly: every stored row's
// fp64 sequential dot (core.cpp:26-37), best row per entry by strict '>' in list order
// (index.cpp:306-311), top-k by (sim desc, id asc) (index.cpp:320-324) — IvfIndex::search by
// brute force, so it is correct for any data. kOvfQG flagged queries per pass share each row
// read (kOvfQG independent chains per lane). Each warp keeps its own top-k lists (lane i holds
// the i-th best); they go to a ring in global memory and the LAST CTA to finish a pass merges
// them, enriches the hits (segment, s_neg, gater block sums) and re-runs the gate / select /
// gater for those queries — replacing k_finish's records, count and choice. With no flagged
// query (the normal case) every CTA returns at once.
// ------------------------------------------------------------------------------------------
struct WL {  // lane-distributed sorted list entry
    double s;
    uint64_t id;
    int32_t slot, row;
};

__device__ __forceinline__ void wl_empty(WL& l) {
    l.s = -INFINITY;
    l.id = ~0ull;
    l.slot = -1;
    l.row = 0;
}

// inserts the warp-uniform candidate (s, id, slot, row) into the k-entry list (no-op if it is not
// before the k-th entry); the list stays sorted by (sim desc, id asc)
__device__ __forceinline__ void wl_insert(WL& l, double s, uint64_t id, int slot, int row, int k,
                                          int lane) {
    const unsigned full = 0xffffffffu;
    const bool cb = lane < k && before(s, id, l.s, l.id);
    const unsigned m = __ballot_sync(full, cb);
    if (!m) return;
    const int pos = __ffs(m) - 1;  // sorted: every lane from pos on is after the candidate
    const double us = __shfl_up_sync(full, l.s, 1);
    const uint64_t uid = __shfl_up_sync(full, l.id, 1);
    const int uslot = __shfl_up_sync(full, l.slot, 1);
    const int urow = __shfl_up_sync(full, l.row, 1);
    if (lane == pos) {
        l.s = s;
        l.id = id;
        l.slot = slot;
        l.row = row;
    } else if (lane > pos && lane < k) {
        l.s = us;
        l.id = uid;
        l.slot = uslot;
        l.row = urow;
    }
}

// offers each lane's candidate (valid where `has`) to the list, lowest lane first
__device__ __forceinline__ void wl_offer(WL& l, bool has, double s, uint64_t id, int slot, int row,
                                         int k, int lane) {
    const unsigned full = 0xffffffffu;
    const double ks = __shfl_sync(full, l.s, k - 1);
    const uint64_t kid = __shfl_sync(full, l.id, k - 1);
    unsigned m = __ballot_sync(full, has && before(s, id, ks, kid));
    while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        wl_insert(l, __shfl_sync(full, s, src), __shfl_sync(full, id, src),
                  __shfl_sync(full, slot, src), __shfl_sync(full, row, src), k, lane);
    }
}

__global__ void __launch_bounds__(32 * kOvfWarps, 1) k_overflow(const FinishParams p) {
    extern __shared__ double qd[];  // [Df][kOvfQG] flagged queries as doubles, dimension-major
    __shared__ uint8_t prs[kOvfQG][kMaxCentroids];
    __shared__ int last;
    const unsigned full = 0xffffffffu;
    const int nflag = __ldcg(&p.ovf[0]);
    if (nflag == 0) return;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int nwarps = gridDim.x * kOvfWarps, gw = blockIdx.x * kOvfWarps + warp;
    const int nchunks = (nflag + kOvfQG - 1) / kOvfQG;
    const int chunk_cap = (p.bmax + kOvfQG - 1) / kOvfQG;
    int32_t* done = p.ovf + kOvfHdr + p.bmax;  // [chunk_cap] CTAs finished with the pass
    int32_t* merged = done + chunk_cap;         // [chunk_cap] pass merged (its ring slot free)
    const int64_t rows_total = p.n_slots << p.logRp;
    const int k = p.k;
    for (int c = 0; c < nchunks; ++c) {
        const int nq = min(kOvfQG, nflag - c * kOvfQG);
        int qb[kOvfQG];
#pragma unroll
        for (int j = 0; j < kOvfQG; ++j) qb[j] = j < nq ? __ldcg(&p.ovf[kOvfHdr + c * kOvfQG + j]) : -1;
        __syncthreads();  // the previous pass is done with qd / prs
        for (int i = t; i < p.Df * kOvfQG; i += blockDim.x) {
            const int d = i / kOvfQG, j = i - d * kOvfQG;
            qd[i] = (qb[j] >= 0 && d < p.D) ? (double)p.q[(int64_t)qb[j] * p.D + d] : 0.0;
        }
        if (p.ivf)
            for (int i = t; i < kOvfQG * kMaxCentroids; i += blockDim.x) {
                const int j = i / kMaxCentroids, l = i - j * kMaxCentroids;
                prs[j][l] = qb[j] >= 0 ? p.prank[(int64_t)qb[j] * kMaxCentroids + l] : kNotProbed;
            }
        __syncthreads();
        WL L[kOvfQG];
#pragma unroll
        for (int j = 0; j < kOvfQG; ++j) wl_empty(L[j]);
        // ---- scan: warp gw takes 32-row groups gw, gw + nwarps, ...; lane = row
        for (int64_t g = gw; g * 32 < rows_total; g += nwarps) {
            const int64_t row = g * 32 + lane;
            const int64_t slot = row >> p.logRp;
            const int r = (int)(row & (p.Rp - 1));
            const bool ok = row < rows_total && p.valid[slot] && r < p.nrows[slot];
            double s[kOvfQG];
#pragma unroll
            for (int j = 0; j < kOvfQG; ++j) s[j] = 0.0;
            if (ok) {
                const float4* rp4 = reinterpret_cast<const float4*>(p.rows + row * p.Df);
                const double2* q2 = reinterpret_cast<const double2*>(qd);
#pragma unroll 2
                for (int i4 = 0; i4 < (p.Df >> 2); ++i4) {
                    const float4 x = __ldg(rp4 + i4);
                    const double xs[4] = {(double)x.x, (double)x.y, (double)x.z, (double)x.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {  // dimension 4 i4 + u, in order
#pragma unroll
                        for (int j2 = 0; j2 < kOvfQG / 2; ++j2) {
                            const double2 qq = q2[(4 * i4 + u) * (kOvfQG / 2) + j2];
                            s[2 * j2] = fma(qq.x, xs[u], s[2 * j2]);
                            s[2 * j2 + 1] = fma(qq.y, xs[u], s[2 * j2 + 1]);
                        }
                    }
                }
            }
            int l = -1;
            if (ok && p.ivf) l = p.row_list[row];
            uint64_t id = 0;
            if (ok && r == 0) id = p.ids[slot];
#pragma unroll
            for (int j = 0; j < kOvfQG; ++j) {
                bool el = ok && j < nq;
                int key = r;
                if (el && p.ivf) {  // rows of lists the query does not probe are not scanned
                    const int pr = l >= 0 ? prs[j][l] : kNotProbed;
                    el = pr != kNotProbed;
                    key = (pr << 6) | r;  // scan order: probe rank, then pyramid row
                }
                double sim = el ? fmin(1.0, fmax(-1.0, s[j])) : -DBL_MAX;  // core.cpp:35-36
                int kw = el ? key : 0x7fffffff;
                for (int o = 1; o < p.Rp; o <<= 1) {  // best row: max, ties -> lowest key
                    const double os = __shfl_xor_sync(full, sim, o);
                    const int ok2 = __shfl_xor_sync(full, kw, o);
                    if (os > sim || (os == sim && ok2 < kw)) {
                        sim = os;
                        kw = ok2;
                    }
                }
                const bool has = r == 0 && kw != 0x7fffffff;
                wl_offer(L[j], has, sim, id, (int)slot, kw & 63, k, lane);
            }
        }
        // ---- this warp's lists -> ring slot c % kOvfRing (free once pass c - kOvfRing merged)
        if (c >= kOvfRing) {
            if (lane == 0)
                while (atomicAdd(&merged[c - kOvfRing], 0) == 0) __nanosleep(256);
            __syncwarp();
        }
        OvfRec* ring = p.ovf_ring + (int64_t)(c % kOvfRing) * kOvfQG * nwarps * kMaxTopK;
#pragma unroll
        for (int j = 0; j < kOvfQG; ++j)
            if (lane < k) {
                OvfRec o;
                o.sim = L[j].s;
                o.slot = L[j].slot;
                o.row = L[j].row;
                ring[((int64_t)j * nwarps + gw) * kMaxTopK + lane] = o;
            }
        __threadfence();
        __syncthreads();
        if (t == 0) last = atomicAdd(&done[c], 1) == (int)gridDim.x - 1;
        __syncthreads();
        if (!last) continue;
        __threadfence();  // every CTA's lists are visible
        // ---- merge (warp j: query j of the pass), enrich, select
        if (warp < nq) {
            const int j = warp, b = qb[j];
            WL F;
            wl_empty(F);
            for (int i0 = 0; i0 < nwarps * k; i0 += 32) {
                const int i = i0 + lane;
                double os = -INFINITY;
                int oslot = -1, orow = 0;
                if (i < nwarps * k) {  // L2 reads: the lists were written by other CTAs
                    const OvfRec* o = ring + ((int64_t)j * nwarps + i / k) * kMaxTopK + i % k;
                    os = __ldcg(&o->sim);
                    oslot = __ldcg(&o->slot);
                    orow = __ldcg(&o->row);
                }
                const bool has = oslot >= 0;
                const uint64_t id = has ? p.ids[oslot] : ~0ull;
                wl_offer(F, has, os, id, oslot, orow, k, lane);
            }
            const int nh = __popc(__ballot_sync(full, lane < k && F.slot >= 0));
            // enrichment (phase D): segment, s_neg, owner; then the 8 gater block sums
            HitRec* hb = p.hits + (int64_t)b * kMaxTopK;
            if (lane < nh) {
                const int64_t row = (int64_t)F.slot * p.Rp + F.row;
                const sw_segment sg = p.segs[row];
                HitRec& o = hb[lane];
                o.sim = F.s;
                o.entry_id = F.id;
                o.level = sg.level;
                o.slot = F.slot;
                o.start_s = sg.start_s;
                o.length_s = sg.length_s;
                o.s_neg = p.sneg[row];
                o.row = F.row;
                o.owner = p.rank;
            }
            __syncwarp();
            // block sums: each lane computes (hit h, block blk) pairs; slots and rows from the list
            for (int base = 0; base < nh * 8; base += 32) {
                const int hj = base + lane;
                const int h = min(hj >> 3, 31);
                const int slot_h = __shfl_sync(full, F.slot, h);
                const int row_h = __shfl_sync(full, F.row, h);
                if (hj < nh * 8) {
                    const int blk = hj & 7;
                    const float* rp = p.rows + ((int64_t)slot_h * p.Rp + row_h) * p.Df;
                    const size_t lo = (size_t)blk * p.D / 8, hi = (size_t)(blk + 1) * p.D / 8;
                    double bs = 0.0;
                    for (size_t i = lo; i < hi; ++i) bs = fma(qd[i * kOvfQG + j], (double)rp[i], bs);
                    hb[h].phi[blk] = bs;
                }
            }
            __syncwarp();
            __threadfence_block();
            if (lane == 0) p.nhits[b] = nh;
            if (p.do_select) {
                const double u = dev::uniform_draw(dev::derive_seed(p.sp.seed, p.reqs[b].id, 2, 0));
                const sw_choice ch = dev::select_warp(hb, nh, u, p.reqs[b], p.sp, lane);
                if (lane == 0) p.out[b] = ch;
            }
        }
        __syncthreads();
        if (t == 0) {
            __threadfence();
            atomicExch(&merged[c], 1);
            if (atomicAdd(&p.ovf[1], 1) == nchunks - 1) {  // the last pass: reset for the next batch
                for (int i = 0; i < nchunks; ++i) {
                    done[i] = 0;
                    merged[i] = 0;
                }
                atomicAdd(reinterpret_cast<unsigned long long*>(p.ovf + 2), (unsigned long long)nflag);
                p.ovf[1] = 0;
                __threadfence();
                atomicExch(&p.ovf[0], 0);
            }
        }
    }
}

}  // namespace

int launch_score_tc(Ctx& c, int B, int k, bool ivf, cudaStream_t st);
bool launch_probe_rank(Ctx& c, const float* d_q, int B, cudaStream_t st);

// Search (+ optionally select) for B queries. Results land in c.hits / c.nhits (and d_out).
int launch_search_fused(Ctx& c, const float* d_q, int B, int k, int rank, const sw_request* d_req,
                        const dev::SelParams* sp, sw_choice* d_out, cudaStream_t st) {
    return launch_search_fused(c, d_q, B, k, rank, d_req, sp, d_out, st, st);
}

// st_finish != st: prep, probe ranking and scoring on st, the finish kernel on st_finish after
// an event (cross-batch pipelining; the caller manages the scratch parities)
int launch_search_fused(Ctx& c, const float* d_q, int B, int k, int rank, const sw_request* d_req,
                        const dev::SelParams* sp, sw_choice* d_out, cudaStream_t st,
                        cudaStream_t st_finish) {
    SW_REQUIRE(k >= 1, "search k must be >= 1");  // index.cpp:291
    SW_REQUIRE(k <= kMaxTopK, "top-k above 32 is not supported");
    SW_REQUIRE(B >= 0 && B <= c.Bmax, "batch exceeds the context's max_batch");
    if (B == 0) return 0;
    int kernels = 0;
    const int64_t rows_hw = c.high_water * c.Rp;
    const bool exact_only = (c.cfg.flags & SW_FLAG_EXACT_ONLY) != 0;
    // the tcgen05 pre-filter wins at every cache size and batch measured (tools/exact_vs_tc.py:
    // 256 rows B = 1 0.046 vs 0.052 ms; 1000 rows B = 1024 0.074 vs 0.652 ms), so the exact
    // brute force only runs when asked for (SW_FLAG_EXACT_ONLY)
    const bool tc = c.tc_ok && !exact_only && c.high_water > 0;
    (void)rows_hw;
    if (!tc)
        SW_REQUIRE(c.high_water <= kCandCap,
                   "exact-only search is limited to 16384 slots; enable the tcgen05 path");
    kernels += launch_prep(c, d_q, B, d_req, sp ? sp->seed : 0, st);
    bool ivf;
    {
        StageScope sc(c, SW_STAGE_PREP, st);
        ivf = launch_probe_rank(c, d_q, B, st);  // IvfIndex probe lists (nprobe < C)
    }
    kernels += ivf ? 1 : 0;
    int64_t grp_items = 0;
    if (ivf && tc) {  // reference-default IVF, one row per entry: list-grouped tcgen05 GEMM
        StageScope sc(c, SW_STAGE_PREP, st);
        grp_items = ivf_group_prepare(c, B, st);
        kernels += grp_items > 0 ? 4 : 0;
    }
    if (tc) {
        StageScope sc(c, SW_STAGE_SCORE_TC, st);
        kernels += grp_items > 0 ? launch_score_tc_grouped(c, B, k, grp_items, st)
                                 : launch_score_tc(c, B, k, ivf, st);
    }
    FinishParams p{};
    p.B = B;
    p.k = k;
    p.rank = rank;
    p.implicit_all = tc ? 0 : 1;
    p.n_chunks = c.last_chunks;
    p.cap_local = (kCandCap / c.last_chunks) & ~3;
    p.do_select = sp != nullptr;
    p.n_slots = c.high_water;
    p.slice_cnt = c.slice_cnt;
    p.cand_slot = c.cand_slot;
    // the grouped scoring emits list-sorted row indices (no lookup on its emission path); the
    // kept candidates are mapped to arena slots here. The sorted copy is rebuilt only after a
    // mutation, which first drains in-flight batches (wait_readers), so it is stable here.
    p.sorted_slot = grp_items > 0 ? c.d_sorted_slot : nullptr;
    p.cand_score = c.cand_score;
    p.cta_topk = c.cta_topk;
    p.q_eps = c.q_eps;
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
    p.dbg = c.dbg;
    if (sp) p.sp = *sp;
    p.reqs = d_req;
    p.out = d_out;
    p.ivf = ivf ? 1 : 0;
    p.row_list = c.row_list;
    p.prank = c.prank;
    p.ovf = c.ovf_state;
    p.ovf_ring = reinterpret_cast<OvfRec*>(c.ovf_ring);
    p.bmax = c.Bmax;
    c.last_ivf = ivf;
    if (st_finish != st) {
        SW_CUDA(cudaEventRecord(c.async_score_ev, st));
        SW_CUDA(cudaStreamWaitEvent(st_finish, c.async_score_ev, 0));
        st = st_finish;
    }
    {
        StageScope sc(c, SW_STAGE_FINISH, st);
        static const bool ring = [] {
            const char* e = std::getenv("SW_FINISH_RING");
            return e && e[0] == '1';
        }();
        const size_t smem =
            sizeof(double) * c.Df + (ring ? sizeof(float) * NWARP * NST * 32 * SP : 0);
        ensure_smem_attr(c, k_finish<true>, smem);
        ensure_smem_attr(c, k_finish<false>, smem);
        ensure_smem_attr(c, k_finish<false, 256>, smem);
        if (ring)
            k_finish<true><<<B, FT, smem, st>>>(p);
        else if (B <= 64)
            k_finish<false, 256><<<B, 256, smem, st>>>(p);
        else
            k_finish<false><<<B, FT, smem, st>>>(p);
        SW_CUDA(cudaGetLastError());
        if (tc) {
            // certified fallback for queries whose candidate slices overflowed (returns at once
            // when none did); ~18 KB of shared memory, so it co-runs with the next scoring kernel
            const size_t osmem = sizeof(double) * (size_t)c.Df * kOvfQG;
            ensure_smem_attr(c, k_overflow, osmem);
            k_overflow<<<c.num_sms, 32 * kOvfWarps, osmem, st>>>(p);
            ++kernels;
        }
    }
    SW_CUDA(cudaGetLastError());
    c.last_tc = tc ? (c.last_score_ts ? 3 : c.last_score_pair ? 2 : 1) : 0;  // 2: pairs, 3: +TS
    return kernels + 1;
}

}  // namespace sw
