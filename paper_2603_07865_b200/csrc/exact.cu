// K2 — exact rescoring and top-k for IvfIndex::search (index.cpp:289-326).
//
//  k_prep      queries fp32 -> bf16 (K zero-padded) for the tcgen05 pre-filter, |q|, resets
//  k_compact   keeps the certified candidates: approx >= T_a - 2 eps_q (T_a = k-th best approx)
//  k_rescore   fp64 sequential dot of every row of every candidate entry (i = 0..D-1, exactly
//              the order of dot(), core.cpp:26-30), clamp (core.cpp:35-36), best row per entry
//              by strict '>' in pyramid order (index.cpp:311)
//  k_topk      (sim desc, id asc) selection of the top k (index.cpp:320-324) + hit enrichment
//              (s_neg, gater block sums) so the select stage needs no embeddings.
// In brute-force mode (tiny caches or SW_FLAG_EXACT_ONLY) every valid slot is a candidate.
#include <cfloat>

#include "sw_internal.cuh"

namespace sw {

int launch_score_tc(Ctx& c, int B, int k, cudaStream_t st);

namespace {

constexpr int kRescoreBlocksPerQuery = 8;

__device__ __forceinline__ double clamp_cos(double v) {
    if (v > 1.0) v = 1.0;
    if (v < -1.0) v = -1.0;
    return v;
}

__global__ void k_prep(const float* __restrict__ q, int B, int D, int Dp,
                       __nv_bfloat16* __restrict__ q_bf, float* __restrict__ q_norm,
                       uint32_t* __restrict__ thr, int32_t* __restrict__ cand_n) {
    const int b = blockIdx.x;
    if (b >= B) return;
    __shared__ double red[32];
    const float* qb = q + (int64_t)b * D;
    double s = 0.0;
    for (int d = threadIdx.x; d < Dp; d += blockDim.x) {
        float v = d < D ? qb[d] : 0.0f;
        q_bf[(int64_t)b * Dp + d] = __float2bfloat16_rn(v);
        s += (double)v * v;
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        q_norm[b] = (float)sqrt(t) * (1.0f + 1e-6f);
        thr[b] = f2ord(-INFINITY);
        cand_n[b] = 0;
    }
}

// Gathers the per-(query, CTA) emission slices of the tcgen05 pass into shared memory, finds
// T_a = the k-th best approximate entry score among them (k rounds of block argmax with
// exclusion) and keeps the certified candidates approx >= T_a - 2 eps_q.
__global__ void k_compact(int k, int n_chunks, int cap_local, const int32_t* __restrict__ slice_cnt,
                          const int32_t* __restrict__ cand_slot, const float* __restrict__ cand_score,
                          const float* __restrict__ q_norm, const uint32_t* __restrict__ maxnorm,
                          float eps_rel, int32_t* __restrict__ out_slot, int32_t* __restrict__ out_n,
                          int32_t* __restrict__ overflow) {
    extern __shared__ uint8_t sm_raw[];
    float* sc = reinterpret_cast<float*>(sm_raw);                 // [kCandCap]
    int32_t* sl = reinterpret_cast<int32_t*>(sc + kCandCap);      // [kCandCap]
    __shared__ int off[149];
    __shared__ unsigned long long sh[33];
    __shared__ int cnt;
    __shared__ int ovf;
    const int b = blockIdx.x;
    if (threadIdx.x == 0) {
        int o = 0, f = 0;
        for (int c = 0; c < n_chunks; ++c) {
            const int n = slice_cnt[(int64_t)b * n_chunks + c];
            off[c] = o;
            o += min(n, cap_local);
            f |= n > cap_local;
        }
        off[n_chunks] = o;
        ovf = f;
        cnt = 0;
    }
    __syncthreads();
    const int n = off[n_chunks];
    for (int c = 0; c < n_chunks; ++c) {
        const int m = off[c + 1] - off[c];
        const int64_t src = (int64_t)b * kCandCap + (int64_t)c * cap_local;
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            sc[off[c] + i] = cand_score[src + i];
            sl[off[c] + i] = cand_slot[src + i];
        }
    }
    __syncthreads();
    // k-th largest (ties broken by position so every round removes exactly one element)
    unsigned long long prev = ~0ull;
    float kth = -INFINITY;
    for (int r = 0; r < k; ++r) {
        unsigned long long best = 0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const unsigned long long key =
                ((unsigned long long)f2ord(sc[i]) << 32) | (0xFFFFFFFFu - (uint32_t)i);
            if (key < prev && key > best) best = key;
        }
        for (int o = 16; o; o >>= 1) {
            const unsigned long long x = __shfl_xor_sync(0xffffffffu, best, o);
            best = x > best ? x : best;
        }
        if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = best;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long b2 = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b2 = sh[w] > b2 ? sh[w] : b2;
            sh[32] = b2;
        }
        __syncthreads();
        best = sh[32];
        __syncthreads();
        if (best == 0) {  // fewer than k candidates: keep everything
            kth = -INFINITY;
            break;
        }
        prev = best;
        kth = ord2f((uint32_t)(best >> 32));
    }
    const float eps2 = 2.0f * eps_rel * q_norm[b] * ord2f(*maxnorm);
    const float cut = kth - eps2;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        if (sc[i] >= cut) {
            const int j = atomicAdd(&cnt, 1);
            out_slot[(int64_t)b * kCandCap + j] = sl[i];
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        out_n[b] = cnt;
        overflow[b] = ovf;
    }
}

// Work item = (candidate i, row r) with r in [0, Rp); lanes of one candidate are adjacent.
__global__ void k_rescore(int B, int implicit_all, int64_t n_slots, const int32_t* __restrict__ list,
                          const int32_t* __restrict__ list_n, const float* __restrict__ q,
                          const float* __restrict__ rows, const int32_t* __restrict__ nrows,
                          const uint8_t* __restrict__ valid, int D, int Df, int Rp, int logRp,
                          double* __restrict__ exact, int32_t* __restrict__ best_row) {
    extern __shared__ float4 qs4[];
    const int b = blockIdx.y;
    const float* qb = q + (int64_t)b * D;
    float* qs = reinterpret_cast<float*>(qs4);
    for (int d = threadIdx.x; d < Df; d += blockDim.x) qs[d] = d < D ? qb[d] : 0.0f;
    __syncthreads();
    const int64_t n = implicit_all ? n_slots : (int64_t)list_n[b];
    const int64_t items = n << logRp;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // grid-stride; the loop bound is rounded to whole warps so shuffles stay converged
    const int64_t items_w = (items + 31) & ~int64_t(31);
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < items_w; w += stride) {
        const int64_t i = w >> logRp;
        const int r = (int)(w & (Rp - 1));
        double sim = -DBL_MAX;
        int row = 0x7fffffff;
        int64_t slot = -1;
        if (w < items) {
            slot = implicit_all ? i : (int64_t)list[(int64_t)b * kCandCap + i];
            if (valid[slot] && r < nrows[slot]) {
                const float4* rp = reinterpret_cast<const float4*>(rows + (slot * Rp + r) * Df);
                double s = 0.0;
#pragma unroll 4
                for (int d4 = 0; d4 < (Df >> 2); ++d4) {
                    const float4 x = __ldg(rp + d4);
                    const float4 y = qs4[d4];
                    s = fma((double)y.x, (double)x.x, s);
                    s = fma((double)y.y, (double)x.y, s);
                    s = fma((double)y.z, (double)x.z, s);
                    s = fma((double)y.w, (double)x.w, s);
                }
                sim = clamp_cos(s);
                row = r;
            }
        }
        // best row of the entry: max sim, ties -> lowest row (strict '>' in list order)
        for (int o = 1; o < Rp; o <<= 1) {
            double os = __shfl_xor_sync(0xffffffffu, sim, o);
            int orow = __shfl_xor_sync(0xffffffffu, row, o);
            if (os > sim || (os == sim && orow < row)) {
                sim = os;
                row = orow;
            }
        }
        if (w < items && r == 0) {
            const int64_t o = (int64_t)b * kCandCap + i;
            exact[o] = sim;
            best_row[o] = row;
        }
    }
}

struct Key {
    double sim;
    uint64_t id;
};
// true if a precedes b in (sim desc, id asc) order
__device__ __forceinline__ bool before(double as, uint64_t aid, double bs, uint64_t bid) {
    return as > bs || (as == bs && aid < bid);
}

__global__ void k_topk(int k, int implicit_all, int64_t n_slots, const int32_t* __restrict__ list,
                       const int32_t* __restrict__ list_n, const double* __restrict__ exact,
                       const int32_t* __restrict__ best_row, const uint64_t* __restrict__ ids,
                       const uint8_t* __restrict__ valid, const int32_t* __restrict__ nrows,
                       const sw_segment* __restrict__ segs, const double* __restrict__ sneg,
                       const float* __restrict__ rows, const float* __restrict__ q, int D, int Df,
                       int Rp, int rank, const int32_t* __restrict__ overflow,
                       HitRec* __restrict__ hits, int32_t* __restrict__ nhits) {
    const int b = blockIdx.x;
    __shared__ double s_sim[32];
    __shared__ uint64_t s_id[32];
    __shared__ int64_t s_slot[32];
    __shared__ int64_t s_item[32];
    __shared__ int64_t sel_slot[kMaxTopK];
    __shared__ int32_t sel_row[kMaxTopK];
    __shared__ double sel_sim[kMaxTopK];
    __shared__ int sel_n;
    const int64_t n = implicit_all ? n_slots : (int64_t)list_n[b];
    const int64_t base = (int64_t)b * kCandCap;
    double prev_sim = DBL_MAX;
    uint64_t prev_id = 0;
    bool have_prev = false;
    if (threadIdx.x == 0) sel_n = 0;
    for (int r = 0; r < k; ++r) {
        double bs = -DBL_MAX;
        uint64_t bid = ~0ull;
        int64_t bslot = -1, bitem = -1;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const int64_t slot = implicit_all ? i : (int64_t)list[base + i];
            if (implicit_all && !valid[slot]) continue;
            const double s = exact[base + i];
            const uint64_t id = ids[slot];
            if (have_prev && !before(prev_sim, prev_id, s, id)) continue;  // already taken
            if (bslot < 0 || before(s, id, bs, bid)) {
                bs = s;
                bid = id;
                bslot = slot;
                bitem = i;
            }
        }
        for (int o = 16; o; o >>= 1) {
            double os = __shfl_xor_sync(0xffffffffu, bs, o);
            uint64_t oid = __shfl_xor_sync(0xffffffffu, bid, o);
            int64_t oslot = __shfl_xor_sync(0xffffffffu, bslot, o);
            int64_t oitem = __shfl_xor_sync(0xffffffffu, bitem, o);
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
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
                if (s_slot[w] < 0) continue;
                if (w0 < 0 || before(s_sim[w], s_id[w], s_sim[w0], s_id[w0])) w0 = w;
            }
            if (w0 >= 0) {
                sel_slot[sel_n] = s_slot[w0];
                sel_row[sel_n] = best_row[base + s_item[w0]];
                sel_sim[sel_n] = s_sim[w0];
                s_id[0] = s_id[w0];
                sel_n++;
            } else {
                s_id[0] = 0;
            }
            s_slot[0] = w0 >= 0 ? 1 : -1;
        }
        __syncthreads();
        if (s_slot[0] < 0) break;
        prev_sim = sel_sim[sel_n - 1];
        prev_id = s_id[0];
        have_prev = true;
        __syncthreads();
    }
    __syncthreads();
    const int nh = sel_n;
    // enrichment: hit h, feature block j (gater.cpp:18-26) -- 8 threads per hit
    const float* qb = q + (int64_t)b * D;
    for (int t = threadIdx.x; t < nh * 8; t += blockDim.x) {
        const int h = t >> 3, j = t & 7;
        const int64_t row = sel_slot[h] * Rp + sel_row[h];
        const float* rp = rows + row * Df;
        const size_t lo = (size_t)j * D / 8, hi = (size_t)(j + 1) * D / 8;
        double s = 0.0;
        for (size_t i = lo; i < hi; ++i) s = fma((double)qb[i], (double)rp[i], s);
        HitRec* o = hits + (int64_t)b * kMaxTopK + h;
        o->phi[j] = s;
        if (j == 0) {
            const sw_segment sg = segs[row];
            o->sim = sel_sim[h];
            o->entry_id = ids[sel_slot[h]];
            o->level = sg.level;
            o->slot = (int32_t)sel_slot[h];
            o->start_s = sg.start_s;
            o->length_s = sg.length_s;
            o->s_neg = sneg[row];
            o->row = sel_row[h];
            o->owner = rank;
        }
    }
    if (threadIdx.x == 0) nhits[b] = overflow && overflow[b] ? -nh - 1 : nh;
}

__global__ void k_hits_to_public(int B, int k, const HitRec* __restrict__ hits,
                                 const int32_t* __restrict__ nhits, sw_hit* __restrict__ out,
                                 int32_t* __restrict__ out_n) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    int nh = nhits[b];
    if (nh < 0) nh = -nh - 1;
    out_n[b] = nh;
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

// Search for B queries into c.hits / c.nhits. Returns the number of kernels launched.
int launch_search(Ctx& c, const float* d_q, int B, int k, int rank, cudaStream_t st) {
    SW_REQUIRE(k >= 1, "search k must be >= 1");  // index.cpp:291
    SW_REQUIRE(B >= 0 && B <= c.Bmax, "batch exceeds the context's max_batch");
    if (B == 0) return 0;
    int kernels = 0;
    const int64_t rows_hw = c.high_water * c.Rp;
    const bool exact_only = (c.cfg.flags & SW_FLAG_EXACT_ONLY) != 0;
    const bool tc = c.tc_ok && !exact_only && k <= kMaxTopK && c.high_water > 0 &&
                    (rows_hw >= 4096 || (c.cfg.flags & SW_FLAG_TC_ALWAYS));
    if (!tc) {
        SW_REQUIRE(k <= kMaxTopK, "top-k above 32 is not supported");
        SW_REQUIRE(c.high_water <= kCandCap,
                   "exact-only search is limited to 8192 slots; enable the tcgen05 path");
    }
    {
        StageScope sc(c, SW_STAGE_PREP, st);
        k_prep<<<B, 128, 0, st>>>(d_q, B, c.D, c.Dp, c.q_bf, c.q_norm, c.thr, c.cand_n);
    }
    ++kernels;
    int32_t* list = nullptr;
    int32_t* list_n = nullptr;
    int32_t* overflow = nullptr;
    if (tc) {
        {
            StageScope sc(c, SW_STAGE_SCORE_TC, st);
            kernels += launch_score_tc(c, B, k, st);
        }
        list = c.cand_list;
        list_n = c.cand_n + c.Bmax;
        overflow = c.cand_n + 2 * c.Bmax;
        {
            StageScope sc(c, SW_STAGE_COMPACT, st);
            static bool attr = false;
            const size_t smem = (size_t)kCandCap * 8;
            if (!attr) {
                SW_CUDA(cudaFuncSetAttribute(k_compact, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem));
                attr = true;
            }
            k_compact<<<B, 256, smem, st>>>(k, c.last_chunks, kCandCap / c.last_chunks,
                                            c.slice_cnt, c.cand_slot, c.cand_score, c.q_norm,
                                            c.maxnorm, 0.0081f, list, list_n, overflow);
        }
        ++kernels;
    }
    const int implicit = tc ? 0 : 1;
    int gx = kRescoreBlocksPerQuery;
    if (implicit) gx = (int)std::max<int64_t>(1, (rows_hw + 127) / 128);
    dim3 g2(gx, B);
    {
        StageScope sc(c, SW_STAGE_RESCORE, st);
        k_rescore<<<g2, 128, sizeof(float) * c.Df, st>>>(B, implicit, c.high_water, list, list_n,
                                                         d_q, c.rows, c.nrows, c.valid, c.D, c.Df,
                                                         c.Rp, c.logRp, c.cand_exact, c.cand_row);
    }
    ++kernels;
    {
        StageScope sc(c, SW_STAGE_TOPK, st);
        k_topk<<<B, 256, 0, st>>>(k, implicit, c.high_water, list, list_n, c.cand_exact,
                                  c.cand_row, c.ids, c.valid, c.nrows, c.segs, c.sneg, c.rows, d_q,
                                  c.D, c.Df, c.Rp, rank, overflow, c.hits, c.nhits);
    }
    ++kernels;
    SW_CUDA(cudaGetLastError());
    c.last_tc = tc ? 1 : 0;
    return kernels;
}

void launch_hits_to_public(Ctx& c, int B, int k, sw_hit* d_out, int32_t* d_n, cudaStream_t st) {
    if (B == 0) return;
    k_hits_to_public<<<(B + 127) / 128, 128, 0, st>>>(B, k, c.hits, c.nhits, d_out, d_n);
    SW_CUDA(cudaGetLastError());
}

}  // namespace sw
