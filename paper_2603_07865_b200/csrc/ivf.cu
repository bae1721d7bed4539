// IVF coarse quantiser on the device arena — the reference's DEFAULT search mode
// (IvfIndex, index.hpp:47-101; pipeline.cpp:28-31: index.centroids = 64, index.nprobe = 8,
// index.rebuild_interval = 1024).
//
//   probe ranking   index.cpp:295-304  fp64 sequential dot(query, centroid_j), partial sort by
//                                      (sim desc, j asc), first nprobe lists probed
//   list assignment index.cpp:210-222  nearest centroid, strict '>' (first maximum wins)
//   insert/remove   index.cpp:224-255  mutation counting; first insert into an empty index
//                                      seeds one centroid with the first vector
//   rebuild         index.cpp:257-283  rows sorted by (id, level, start), C = min(n, target),
//                                      kmeans(seed = derive_seed(seed_, rebuild_count_))
//   kmeans          index.cpp:59-184   k-means++ seeding + <= 50 spherical Lloyd iterations
//
// Every floating-point value the reference computes is reproduced bit for bit: each dot product
// is one thread's sequential fp64 chain in dimension order (fp32 x fp32 products are exact in
// fp64, so fma == mul-then-add), per-cluster sums run in ascending row order, and the sequential
// reductions of the k-means++ seeding (running total, cumulative scan) run on the host in the
// reference's order. The parallel work (n x C dot products per Lloyd iteration, the per-(cluster,
// dim) member sums, the farthest-point search) runs on the GPU.
#include <cstdlib>
#include <algorithm>
#include <cmath>
#include <numeric>
#include <random>

#include "select_dev.cuh"

namespace sw {

namespace {

constexpr int AT = 256;        // threads per argmax block (8 warps)
constexpr int RPW = 4;         // rows per warp per pass
constexpr int CH = 32;         // dims per staged centroid chunk

// argmax_j dot(row_i, centroid_j) for rows i of `perm` (arena row indices), strict '>' (lowest
// j among equal maxima). Lane l of a warp owns centroids l, l+32, ... (MC of them); the block
// stages 32-dim chunks of all centroids transposed in smem and every warp runs RPW rows.
template <int MC>
__global__ void __launch_bounds__(AT) k_argmax_centroid(const float* __restrict__ rows, int Df,
                                                         int D, const int64_t* __restrict__ perm,
                                                         int64_t n, const float* __restrict__ cent,
                                                         int C, int16_t* __restrict__ row_list,
                                                         int32_t* __restrict__ assign) {
    __shared__ float cT[CH][32 * MC + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int ROWS = (AT / 32) * RPW;
    for (int64_t i0 = (int64_t)blockIdx.x * ROWS; i0 < n; i0 += (int64_t)gridDim.x * ROWS) {
        int64_t myrow[RPW];
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
            const int64_t i = i0 + warp * RPW + r;
            myrow[r] = i < n ? perm[i] : -1;
        }
        double acc[RPW][MC];
#pragma unroll
        for (int r = 0; r < RPW; ++r)
#pragma unroll
            for (int m = 0; m < MC; ++m) acc[r][m] = 0.0;
        for (int d0 = 0; d0 < D; d0 += CH) {
            __syncthreads();
            for (int t = threadIdx.x; t < CH * 32 * MC; t += AT) {
                const int j = t / CH, d = t % CH;
                cT[d][j] = (j < C && d0 + d < D) ? cent[(int64_t)j * Df + d0 + d] : 0.0f;
            }
            __syncthreads();
            float x[RPW];
#pragma unroll
            for (int r = 0; r < RPW; ++r)
                x[r] = (myrow[r] >= 0 && d0 + lane < D) ? rows[myrow[r] * Df + d0 + lane] : 0.0f;
            const int dn = min(CH, D - d0);
            for (int d = 0; d < dn; ++d) {  // dimension order within the chunk
#pragma unroll
                for (int r = 0; r < RPW; ++r) {
                    const double xd = (double)__shfl_sync(0xffffffffu, x[r], d);
#pragma unroll
                    for (int m = 0; m < MC; ++m)
                        acc[r][m] = fma(xd, (double)cT[d][lane + 32 * m], acc[r][m]);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
            double best = -INFINITY;
            int bj = 0x7fffffff;
#pragma unroll
            for (int m = 0; m < MC; ++m) {
                const int j = lane + 32 * m;
                if (j < C && (acc[r][m] > best || (acc[r][m] == best && j < bj))) {
                    best = acc[r][m];
                    bj = j;
                }
            }
            for (int o = 16; o; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
                if (ob > best || (ob == best && oj < bj)) {
                    best = ob;
                    bj = oj;
                }
            }
            if (lane == 0 && myrow[r] >= 0) {
                if (row_list) row_list[myrow[r]] = (int16_t)bj;
                if (assign) assign[i0 + warp * RPW + r] = bj;
            }
        }
    }
}

// k-means++ distances: d2[i] = 2 - 2 dot(x_i, c) (init) or min(d2[i], 2 - 2 dot(x_i, c))
// (index.cpp:83, :104-106). One thread per row, sequential chain, centroid broadcast from smem.
__global__ void k_seed_d2(const float* __restrict__ rows, int Df, int D,
                          const int64_t* __restrict__ perm, int64_t n,
                          const float* __restrict__ c, double* __restrict__ d2, int init) {
    extern __shared__ float cs[];
    for (int d = threadIdx.x; d < D; d += blockDim.x) cs[d] = c[d];
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4* x4 = reinterpret_cast<const float4*>(rows + perm[i] * Df);
    double s = 0.0;
    int d = 0;
    for (; d + 4 <= D; d += 4) {
        const float4 v = __ldg(x4 + (d >> 2));
        s = fma((double)v.x, (double)cs[d], s);
        s = fma((double)v.y, (double)cs[d + 1], s);
        s = fma((double)v.z, (double)cs[d + 2], s);
        s = fma((double)v.w, (double)cs[d + 3], s);
    }
    for (; d < D; ++d) s = fma((double)rows[perm[i] * Df + d], (double)cs[d], s);
    const double v = __dsub_rn(2.0, __dmul_rn(2.0, s));
    d2[i] = init ? v : (v < d2[i] ? v : d2[i]);  // std::min(d2, v) keeps d2 on ties
}

// Lloyd sums: sums[j][d] = sum over members i of cluster j (ascending i) of x_i[d], in fp64
// (index.cpp:129-135). grid (C, ceil(D / 128)); thread = one dimension's sequential chain.
__global__ void k_cluster_sums(const float* __restrict__ rows, int Df, int D,
                               const int64_t* __restrict__ perm, const int32_t* __restrict__ mem,
                               const int64_t* __restrict__ moff, double* __restrict__ sums) {
    const int j = blockIdx.x;
    const int d = blockIdx.y * blockDim.x + threadIdx.x;
    if (d >= D) return;
    double s = 0.0;
    for (int64_t m = moff[j]; m < moff[j + 1]; ++m) s = __dadd_rn(s, (double)rows[perm[mem[m]] * Df + d]);
    sums[(int64_t)j * D + d] = s;
}

// Empty-cluster reseeding: argmax_i (2 - 2 dot(x_i, c_assign[i])), first maximum (index.cpp:
// 142-151). Per-block (value, index) winners; the host reduces the blocks in order.
__global__ void k_farthest(const float* __restrict__ rows, int Df, int D,
                           const int64_t* __restrict__ perm, int64_t n,
                           const int32_t* __restrict__ assign, const float* __restrict__ cent,
                           double* __restrict__ bv, int64_t* __restrict__ bi) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double v = -INFINITY;
    int64_t idx = INT64_MAX;
    if (i < n) {
        const float* x = rows + perm[i] * Df;
        const float* c = cent + (int64_t)assign[i] * Df;
        double s = 0.0;
        for (int d = 0; d < D; ++d) s = fma((double)x[d], (double)c[d], s);
        v = __dsub_rn(2.0, __dmul_rn(2.0, s));
        idx = i;
    }
    for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (ov > v || (ov == v && oi < idx)) {
            v = ov;
            idx = oi;
        }
    }
    __shared__ double sv[32];
    __shared__ int64_t si[32];
    if ((threadIdx.x & 31) == 0) {
        sv[threadIdx.x >> 5] = v;
        si[threadIdx.x >> 5] = idx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (sv[w] > v || (sv[w] == v && si[w] < idx)) {
                v = sv[w];
                idx = si[w];
            }
        bv[blockIdx.x] = v;
        bi[blockIdx.x] = idx;
    }
}

// Probe ranking (index.cpp:295-304), G = 256 / CP queries per block: thread (g, j) computes
// dot(q_b, c_j) sequentially in dimension order and then its rank = #{i : s_i > s_j or (s_i ==
// s_j and i < j)}, its position in the reference's partial sort (nprobe first -> probed). The
// operands are staged in shared memory AS DOUBLES, DH dimensions at a time (centroids
// transposed [DH][CP + 1], conflict-free for the lane-per-centroid reads; the queries
// [G][DH]), so the chain is LDS + DFMA only: an fp32 -> fp64 conversion on the chain costs
// more than the DFMA's latency on this part, and the float staging converted twice per step.
template <int CP>
__global__ void __launch_bounds__(256) k_probe_rank_smem(const float* __restrict__ q, int B, int D,
                                                          const float* __restrict__ cent, int Df,
                                                          int C, int np,
                                                          uint8_t* __restrict__ prank,
                                                          uint64_t* __restrict__ pmask) {
    constexpr int G = 256 / CP;                  // queries per block
    constexpr int DH = CP <= 64 ? 192 : CP == 128 ? 96 : 48;  // dims per stage (~150 KB)
    constexpr int CS = CP + 1;                   // padded centroid stride (doubles)
    extern __shared__ double smd[];
    double* cT = smd;                            // [DH][CS]
    double* qs = cT + (size_t)DH * CS;           // [G][DH]
    double* sc = qs + (size_t)G * DH;            // [G][CP]
    const int g = threadIdx.x / CP, j = threadIdx.x % CP;
    const int b = blockIdx.x * G + g;
    double a = 0.0;
    for (int d0 = 0; d0 < D; d0 += DH) {
        const int dn = min(DH, D - d0);
        __syncthreads();  // previous stage consumed
        for (int i = threadIdx.x; i < dn * CP; i += 256) {  // coalesced along d
            const int jj = i / dn, d = i - jj * dn;
            cT[d * CS + jj] = jj < C ? (double)cent[(int64_t)jj * Df + d0 + d] : 0.0;
        }
        for (int i = threadIdx.x; i < G * dn; i += 256) {
            const int gg = i / dn, d = i - gg * dn;
            const int bb = blockIdx.x * G + gg;
            qs[gg * DH + d] = bb < B ? (double)q[(int64_t)bb * D + d0 + d] : 0.0;
        }
        __syncthreads();
        if (b < B && j < C) {
            const double* qg = qs + g * DH;
#pragma unroll 8
            for (int d = 0; d < dn; ++d) a = fma(qg[d], cT[d * CS + j], a);
        }
    }
    sc[g * CP + j] = a;
    __syncthreads();
    if (b < B) {
        uint8_t r = kNotProbed;
        if (j < C) {
            int rank = 0;
            const double sj = sc[g * CP + j];
            for (int i = 0; i < C; ++i) {
                const double si = sc[g * CP + i];
                rank += (si > sj || (si == sj && i < j)) ? 1 : 0;
            }
            if (rank < np) r = (uint8_t)rank;
        }
        for (int jj = j; jj < kMaxCentroids; jj += CP)
            prank[(int64_t)b * kMaxCentroids + jj] = jj == j ? r : kNotProbed;
        const unsigned ballot = __ballot_sync(0xffffffffu, r != kNotProbed);
        if ((j & 31) == 0) {
            uint32_t* pm32 = reinterpret_cast<uint32_t*>(pmask + (int64_t)b * 4);
            pm32[j >> 5] = ballot;
            if (j == 0)
                for (int w = CP / 32; w < 8; ++w) pm32[w] = 0u;
        }
    }
}


// rows [nrows[slot], Rp) of each slot belong to no list (pad rows repeat row 0 in the bf16
// shadow; they must never make an entry eligible through a stale list id)
__global__ void k_list_tails(const int64_t* __restrict__ slots, const int32_t* __restrict__ nr,
                             int64_t n, int Rp, int16_t* __restrict__ row_list) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * Rp) return;
    const int64_t e = i / Rp;
    const int r = (int)(i - e * Rp);
    if (r >= nr[e]) row_list[slots[e] * Rp + r] = -1;
}

// ---- grouped IVF search (one row per entry) --------------------------------------------
// queries of each probed list: qlist[l][*] (order irrelevant: a query's results do not depend
// on which block it shares)
__global__ void k_group_count(const uint8_t* __restrict__ prank, int C, int np,
                              int32_t* __restrict__ qcnt, int32_t* __restrict__ qlist, int Bmax) {
    const int q = blockIdx.x, j = threadIdx.x;
    if (j >= C) return;
    if (prank[(int64_t)q * kMaxCentroids + j] < np) {
        const int pos = atomicAdd(&qcnt[j], 1);
        qlist[(int64_t)j * Bmax + pos] = q;
    }
}

// work items: list j, query block b of its queries, tile chunk jj of its tiles. pair: a list's
// blocks come in pairs (the odd one padded with an empty block) and one item covers two blocks —
// a CTA pair (cta_group::2, M = 256) — so the list's tiles stream from HBM once per 256 queries
// instead of once per 128.
// SW_IVF_LPT=0: grouped IVF items in list order instead of longest-first (A/B timing)
static bool ivf_lpt() {
    static const bool on = [] {
        const char* e = getenv("SW_IVF_LPT");
        return !(e && e[0] == '0');
    }();
    return on;
}

constexpr int kMaxTpc = 255;  // tiles per grouped item (SW_IVF_TPC), bucketed by k_group_plan

__global__ void k_group_plan(const int32_t* __restrict__ qcnt, int C,
                             const int32_t* __restrict__ tile0, const int32_t* __restrict__ ntl,
                             int tpc, int pair, int sort_items, int32_t* __restrict__ qbase,
                             int4* __restrict__ items) {
    __shared__ int s_nb[kMaxCentroids], s_ni[kMaxCentroids];
    const int j = threadIdx.x;
    int nb = 0, ch = 0;
    if (j < C && qcnt[j] > 0 && ntl[j] > 0) {
        nb = (qcnt[j] + 127) / 128;
        if (pair) nb += nb & 1;
        ch = (ntl[j] + tpc - 1) / tpc;
    }
    const int bstep = pair ? 2 : 1;
    s_nb[j] = nb;
    s_ni[j] = nb / bstep * ch;
    __syncthreads();
    if (j == 0) {  // exclusive scans over <= 256 lists
        int a = 0, b = 0;
        for (int i = 0; i < kMaxCentroids; ++i) {
            const int x = s_nb[i], y = s_ni[i];
            s_nb[i] = a;
            s_ni[i] = b;
            a += x;
            b += y;
        }
        qbase[kMaxCentroids] = a;
        qbase[kMaxCentroids + 1] = b;  // work items (persistent scoring CTAs walk them)
        qbase[kMaxCentroids + 2] = 0;  // their ticket counter (dynamic item scheduling)
    }
    __syncthreads();
    if (j < kMaxCentroids) qbase[j] = s_nb[j];
    // Item order = the order the persistent CTAs take tickets in. Items are long (a chunk of
    // ~20 tiles streams ~5 MB at an SM's share of HBM) and each CTA runs only ~2-3 of them, so
    // the kernel's tail is set by what is left at the end: a list's tiles are split into ch
    // near-equal chunks (no short remainder chunk), and items are taken largest first
    // (longest-processing-time order) through shared-memory bucket counters by size (the
    // order within a size is arbitrary: results do not depend on which CTA scores an item).
    // The static walk (SW_IVF_DYN=0, pairs) keeps list order and tpc-sized chunks.
    __shared__ int s_bkt[kMaxTpc + 1];
    const bool lpt = !pair && sort_items && tpc <= kMaxTpc;
    if (lpt) {
        const int nbs = nb / bstep;
        const int csz = ch > 0 ? ntl[j] / ch : 0, cex = ch > 0 ? ntl[j] % ch : 0;  // sizes
        if (j <= kMaxTpc) s_bkt[j] = 0;
        __syncthreads();
        if (nbs > 0 && cex > 0) atomicAdd(&s_bkt[csz + 1], nbs * cex);
        if (nbs > 0 && csz > 0) atomicAdd(&s_bkt[csz], nbs * (ch - cex));
        __syncthreads();
        if (j == 0) {  // bucket starts, largest chunks first
            int a = 0;
            for (int r = kMaxTpc; r >= 1; --r) {
                const int x = s_bkt[r];
                s_bkt[r] = a;
                a += x;
            }
        }
        __syncthreads();
        int pbig = 0, psmall = 0;
        if (nbs > 0 && cex > 0) pbig = atomicAdd(&s_bkt[csz + 1], nbs * cex);
        if (nbs > 0 && csz > 0) psmall = atomicAdd(&s_bkt[csz], nbs * (ch - cex));
        for (int b = 0; b < nb; b += bstep)
            for (int jj = 0; jj < ch; ++jj) {
                const int nt = csz + (jj < cex ? 1 : 0);
                const int t0 = jj * csz + min(jj, cex);
                items[jj < cex ? pbig++ : psmall++] =
                    make_int4((s_nb[j] + b) * 128, tile0[j] + t0, nt, j | (jj << 8));
            }
        return;
    }
    for (int b = 0; b < nb; b += bstep)
        for (int jj = 0; jj < ch; ++jj)
            items[s_ni[j] + b / bstep * ch + jj] =
                make_int4((s_nb[j] + b) * 128, tile0[j] + jj * tpc, min(tpc, ntl[j] - jj * tpc),
                          j | (jj << 8));
}

// gathered query rows (one warp per row): qg[g] = q_bf[qmap[g]] (zeros for padding)
__global__ void k_group_gather(const int32_t* __restrict__ qcnt,
                               const int32_t* __restrict__ qlist, const int32_t* __restrict__ qbase,
                               int C, int Bmax, const __nv_bfloat16* __restrict__ q_bf, int Dp,
                               __nv_bfloat16* __restrict__ qg, int32_t* __restrict__ qmap,
                               int64_t rows) {
    const int64_t g = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (g >= rows) return;
    const int blk = (int)(g / 128), r = (int)(g % 128);
    int q = -1;
    if (blk < qbase[kMaxCentroids]) {
        int lo = 0, hi = C - 1;  // last list with qbase <= blk
        while (lo < hi) {
            const int mid = (lo + hi + 1) / 2;
            if (qbase[mid] <= blk) lo = mid; else hi = mid - 1;
        }
        const int idx = (blk - qbase[lo]) * 128 + r;
        if (idx < qcnt[lo]) q = qlist[(int64_t)lo * Bmax + idx];
    }
    if (lane == 0) qmap[g] = q;
    const uint4* src = reinterpret_cast<const uint4*>(q_bf + (int64_t)(q < 0 ? 0 : q) * Dp);
    uint4* dst = reinterpret_cast<uint4*>(qg + g * Dp);
    for (int i = lane; i < Dp / 8; i += 32) dst[i] = q < 0 ? make_uint4(0, 0, 0, 0) : src[i];
}

// list-sorted arena copy: row r <- arena row sorted_slot[r] (zeros for tile padding)
__global__ void k_sort_rows(const int32_t* __restrict__ sorted_slot, int64_t rows,
                            const __nv_bfloat16* __restrict__ src, int Dp,
                            __nv_bfloat16* __restrict__ dst) {
    const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const int32_t s = sorted_slot[r];
    const uint4* a = reinterpret_cast<const uint4*>(src + (int64_t)(s < 0 ? 0 : s) * Dp);
    uint4* b = reinterpret_cast<uint4*>(dst + r * Dp);
    for (int i = lane; i < Dp / 8; i += 32) b[i] = s < 0 ? make_uint4(0, 0, 0, 0) : a[i];
}

// unvisited (query, slice) pairs read as empty by the finish kernel
__global__ void k_fill_slices(int B, int n_chunks, int k, int32_t* __restrict__ slice_cnt,
                              float* __restrict__ cta_topk) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)B * n_chunks) return;
    slice_cnt[i] = 0;
    for (int t = 0; t < k; ++t) cta_topk[i * kMaxTopK + t] = -INFINITY;
}

// --------------------------------------------------------------------------- host helpers
struct MtRng {  // Rng (core.hpp:75-93) over the standard-specified mt19937_64
    std::mt19937_64 g;
    explicit MtRng(uint64_t s) : g(s) {}
    uint64_t uniform_int(uint64_t n) {  // core.cpp:73-82, rejection sampling
        const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
        uint64_t x;
        do {
            x = g();
        } while (x >= limit);
        return x % n;
    }
    double uniform() { return (double)(g() >> 11) * 0x1.0p-53; }
};

template <typename T>
struct DBuf {
    T* p = nullptr;
    explicit DBuf(size_t n) { SW_CUDA(cudaMalloc(&p, sizeof(T) * std::max<size_t>(n, 1))); }
    ~DBuf() { cudaFree(p); }
    DBuf(const DBuf&) = delete;
};

void argmax_rows(Ctx& c, const int64_t* d_perm, int64_t n, int C, int16_t* row_list,
                 int32_t* assign, cudaStream_t st) {
    if (n == 0 || C == 0) return;
    const int ROWS = (AT / 32) * RPW;
    const int grid = (int)std::min<int64_t>((n + ROWS - 1) / ROWS, 148 * 8);
    if (C <= 32)
        k_argmax_centroid<1><<<grid, AT, 0, st>>>(c.rows, c.Df, c.D, d_perm, n, c.cent, C, row_list, assign);
    else if (C <= 64)
        k_argmax_centroid<2><<<grid, AT, 0, st>>>(c.rows, c.Df, c.D, d_perm, n, c.cent, C, row_list, assign);
    else if (C <= 128)
        k_argmax_centroid<4><<<grid, AT, 0, st>>>(c.rows, c.Df, c.D, d_perm, n, c.cent, C, row_list, assign);
    else
        k_argmax_centroid<8><<<grid, AT, 0, st>>>(c.rows, c.Df, c.D, d_perm, n, c.cent, C, row_list, assign);
    SW_CUDA(cudaGetLastError());
}

void upload_centroids(Ctx& c, const std::vector<float>& h, int C) {
    std::vector<float> pad((size_t)C * c.Df, 0.0f);
    for (int j = 0; j < C; ++j)
        std::copy(h.begin() + (size_t)j * c.D, h.begin() + (size_t)(j + 1) * c.D,
                  pad.begin() + (size_t)j * c.Df);
    if (C > 0)
        mcopy(c, c.cent, pad.data(), sizeof(float) * pad.size(), cudaMemcpyHostToDevice);
}

void fetch_row(Ctx& c, int64_t row, float* out) {
    mcopy(c, out, c.rows + row * c.Df, sizeof(float) * c.D, cudaMemcpyDeviceToHost);
}

// kmeans (index.cpp:59-184) over the rows perm[0..n) (arena row indices, reference input order).
void kmeans(Ctx& c, const std::vector<int64_t>& perm, int cnum, uint64_t seed) {
    const int64_t n = (int64_t)perm.size();
    const int D = c.D;
    cudaStream_t st = c.mstream;
    MtRng rng(seed);
    MScratch<int64_t> d_perm(c, (size_t)n);
    mcopy(c, d_perm.p, perm.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice);
    std::vector<float> cent((size_t)cnum * D);
    auto crow = [&](int j) { return cent.data() + (size_t)j * D; };

    // ---- k-means++ seeding with a running minimum distance (index.cpp:79-107)
    const uint64_t first = rng.uniform_int((uint64_t)n);
    fetch_row(c, perm[first], crow(0));
    MScratch<double> d_d2(c, (size_t)n);
    MScratch<float> d_c(c, (size_t)D);
    std::vector<double> d2((size_t)n);
    const int TB = 256;
    const int nb = (int)((n + TB - 1) / TB);
    auto d2_pass = [&](int j, int init) {
        mcopy(c, d_c.p, crow(j), sizeof(float) * D, cudaMemcpyHostToDevice);
        k_seed_d2<<<nb, TB, sizeof(float) * D, st>>>(c.rows, c.Df, D, d_perm.p, n, d_c.p, d_d2.p,
                                                     init);
        SW_CUDA(cudaGetLastError());
    };
    d2_pass(0, 1);
    for (int k = 1; k < cnum; ++k) {
        SW_CUDA(cudaMemcpyAsync(d2.data(), d_d2.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        SW_CUDA(cudaStreamSynchronize(st));
        double total = 0.0;
        for (int64_t i = 0; i < n; ++i) total += std::max(0.0, d2[(size_t)i]);
        int64_t pick;
        if (total > 0.0) {
            const double target = rng.uniform() * total;
            double acc = 0.0;
            pick = n - 1;
            for (int64_t i = 0; i < n; ++i) {
                acc += std::max(0.0, d2[(size_t)i]);
                if (acc >= target) {
                    pick = i;
                    break;
                }
            }
        } else {
            pick = (int64_t)rng.uniform_int((uint64_t)n);
        }
        fetch_row(c, perm[(size_t)pick], crow(k));
        d2_pass(k, 0);
    }

    // ---- Lloyd iterations on the sphere (index.cpp:109-176)
    MScratch<int32_t> d_assign(c, (size_t)n);
    MScratch<int32_t> d_mem(c, (size_t)n);
    MScratch<int64_t> d_moff(c, (size_t)cnum + 1);
    MScratch<double> d_sums(c, (size_t)cnum * D);
    std::vector<int32_t> assign((size_t)n), mem((size_t)n);
    std::vector<int64_t> moff((size_t)cnum + 1);
    std::vector<double> sums((size_t)cnum * D);
    for (int iter = 0; iter < 50; ++iter) {
        upload_centroids(c, cent, cnum);
        argmax_rows(c, d_perm.p, n, cnum, nullptr, d_assign.p, st);
        SW_CUDA(cudaMemcpyAsync(assign.data(), d_assign.p, sizeof(int32_t) * n,
                                cudaMemcpyDeviceToHost, st));
        SW_CUDA(cudaStreamSynchronize(st));
        // members of each cluster in ascending row order (stable counting sort)
        std::fill(moff.begin(), moff.end(), 0);
        for (int64_t i = 0; i < n; ++i) ++moff[(size_t)assign[(size_t)i] + 1];
        for (int j = 0; j < cnum; ++j) moff[(size_t)j + 1] += moff[(size_t)j];
        {
            std::vector<int64_t> pos(moff.begin(), moff.end() - 1);
            for (int64_t i = 0; i < n; ++i) mem[(size_t)pos[(size_t)assign[(size_t)i]]++] = (int32_t)i;
        }
        SW_CUDA(cudaMemcpyAsync(d_mem.p, mem.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
        SW_CUDA(cudaMemcpyAsync(d_moff.p, moff.data(), sizeof(int64_t) * (cnum + 1),
                                cudaMemcpyHostToDevice, st));
        dim3 g((unsigned)cnum, (unsigned)((D + 127) / 128));
        k_cluster_sums<<<g, 128, 0, st>>>(c.rows, c.Df, D, d_perm.p, d_mem.p, d_moff.p, d_sums.p);
        SW_CUDA(cudaGetLastError());
        SW_CUDA(cudaMemcpyAsync(sums.data(), d_sums.p, sizeof(double) * sums.size(),
                                cudaMemcpyDeviceToHost, st));
        SW_CUDA(cudaStreamSynchronize(st));

        double max_shift = 0.0;
        std::vector<float> next((size_t)D);
        for (int j = 0; j < cnum; ++j) {
            const int64_t cnt = moff[(size_t)j + 1] - moff[(size_t)j];
            if (cnt == 0) {
                // re-seed with the point farthest from its (current) centroid (index.cpp:142-151)
                upload_centroids(c, cent, cnum);
                const int fb = (int)((n + 255) / 256);
                MScratch<double> bv(c, (size_t)fb);
                MScratch<int64_t> bi(c, (size_t)fb);
                k_farthest<<<fb, 256, 0, st>>>(c.rows, c.Df, D, d_perm.p, n, d_assign.p, c.cent,
                                               bv.p, bi.p);
                SW_CUDA(cudaGetLastError());
                std::vector<double> hv((size_t)fb);
                std::vector<int64_t> hi((size_t)fb);
                mcopy(c, hv.data(), bv.p, sizeof(double) * fb, cudaMemcpyDeviceToHost);
                mcopy(c, hi.data(), bi.p, sizeof(int64_t) * fb, cudaMemcpyDeviceToHost);
                double worst = -2.0;
                int64_t pick = 0;
                for (int b = 0; b < fb; ++b)
                    if (hv[(size_t)b] > worst) {  // blocks are in ascending row order
                        worst = hv[(size_t)b];
                        pick = hi[(size_t)b];
                    }
                fetch_row(c, perm[(size_t)pick], next.data());
            } else {
                double nrm = 0.0;
                const double* s = sums.data() + (size_t)j * D;
                for (int d = 0; d < D; ++d) nrm += s[d] * s[d];
                nrm = std::sqrt(nrm);
                if (nrm < 1e-12) {
                    fetch_row(c, perm[(size_t)rng.uniform_int((uint64_t)n)], next.data());
                } else {
                    for (int d = 0; d < D; ++d) next[(size_t)d] = (float)(s[d] / nrm);
                }
            }
            double shift2 = 0.0;
            for (int d = 0; d < D; ++d) {
                const double diff = (double)next[(size_t)d] - crow(j)[d];
                shift2 += diff * diff;
            }
            max_shift = std::max(max_shift, std::sqrt(shift2));
            std::copy(next.begin(), next.end(), crow(j));
        }
        if (max_shift < 1e-4) break;
    }
    c.h_cent = cent;
    c.ivf_C = cnum;
    upload_centroids(c, cent, cnum);
}

}  // namespace

void ivf_mark_tails(Ctx& c, const std::vector<int64_t>& slots, const std::vector<int32_t>& nr) {
    if (slots.empty()) return;
    MScratch<int64_t> d_s(c, slots.size());
    MScratch<int32_t> d_n(c, nr.size());
    mcopy(c, d_s.p, slots.data(), sizeof(int64_t) * slots.size(), cudaMemcpyHostToDevice);
    mcopy(c, d_n.p, nr.data(), sizeof(int32_t) * nr.size(), cudaMemcpyHostToDevice);
    const int64_t tot = (int64_t)slots.size() * c.Rp;
    k_list_tails<<<(unsigned)((tot + 255) / 256), 256, 0, c.mstream>>>(d_s.p, d_n.p,
                                                                    (int64_t)slots.size(), c.Rp,
                                                                    c.row_list);
    SW_CUDA(cudaGetLastError());
    SW_CUDA(cudaStreamSynchronize(c.mstream));
}

// Rows the index knows about, in the reference's rebuild order: entries by id, each entry's rows
// by (level, start) (index.cpp:267-272).
static std::vector<int64_t> rebuild_order(Ctx& c) {
    std::vector<std::pair<uint64_t, int64_t>> ents;
    ents.reserve(c.slot_of.size());
    for (auto& kv : c.slot_of)
        if (c.ivf_rows[(size_t)kv.second] > 0) ents.emplace_back(kv.first, kv.second);
    std::sort(ents.begin(), ents.end());
    std::vector<sw_segment> segs((size_t)c.Rp);
    std::vector<int64_t> perm;
    for (auto& [id, slot] : ents) {
        const int nr = c.ivf_rows[(size_t)slot];
        mcopy(c, segs.data(), c.segs + slot * c.Rp, sizeof(sw_segment) * nr,
                           cudaMemcpyDeviceToHost);
        std::vector<int> o((size_t)nr);
        std::iota(o.begin(), o.end(), 0);
        std::stable_sort(o.begin(), o.end(), [&](int a, int b) {
            if (segs[(size_t)a].level != segs[(size_t)b].level)
                return segs[(size_t)a].level < segs[(size_t)b].level;
            return segs[(size_t)a].start_s < segs[(size_t)b].start_s;
        });
        for (int r : o) perm.push_back(slot * c.Rp + r);
    }
    return perm;
}

// IvfIndex::rebuild (index.cpp:257-283)
void ivf_rebuild(Ctx& c) {
    c.grp_dirty = true;
    c.ivf_mutations = 0;
    c.ivf_rebuilds++;
    std::vector<int64_t> perm = rebuild_order(c);
    if (perm.empty()) {
        c.ivf_C = 0;
        c.h_cent.clear();
        return;
    }
    const int cnum = (int)std::min<int64_t>((int64_t)perm.size(), std::max(c.ivf_target, 1));
    kmeans(c, perm, cnum, dev::derive_seed(c.ivf_seed, c.ivf_rebuilds, 0, 0));
    MScratch<int64_t> d_perm(c, perm.size());
    mcopy(c, d_perm.p, perm.data(), sizeof(int64_t) * perm.size(), cudaMemcpyHostToDevice);
    argmax_rows(c, d_perm.p, (int64_t)perm.size(), c.ivf_C, c.row_list, nullptr, c.mstream);
    SW_CUDA(cudaStreamSynchronize(c.mstream));
}

// IvfIndex::build(vecs, C, seed, nprobe) (index.cpp:186-208) over rows already in the arena:
// kmeans over `perm` (the vecs order) with the build seed itself (no rebuild derivation),
// C reduced to the row count, every row assigned to its nearest centroid; no mutation counted.
void ivf_build_from(Ctx& c, const std::vector<int64_t>& perm) {
    c.grp_dirty = true;
    c.ivf_mutations = 0;
    c.ivf_rebuilds = 0;
    if (perm.empty()) {
        c.ivf_C = 0;
        c.h_cent.clear();
        return;
    }
    const int cnum = (int)std::min<int64_t>((int64_t)perm.size(), std::max(c.ivf_target, 1));
    kmeans(c, perm, cnum, c.ivf_seed);
    MScratch<int64_t> d_perm(c, perm.size());
    mcopy(c, d_perm.p, perm.data(), sizeof(int64_t) * perm.size(), cudaMemcpyHostToDevice);
    argmax_rows(c, d_perm.p, (int64_t)perm.size(), c.ivf_C, c.row_list, nullptr, c.mstream);
    SW_CUDA(cudaStreamSynchronize(c.mstream));
}

// IvfIndex::check_consistent (index.cpp:334-343): every stored row sits in the list of its
// nearest centroid (recomputed here with the same fp64 chains), rows beyond an entry's count
// in no list, and (exhaustive mode) no row carries a list.
bool ivf_check_consistent(Ctx& c) {
    std::vector<int64_t> rows;
    std::vector<int16_t> want;
    for (auto& kv : c.slot_of) {
        const int64_t slot = kv.second;
        const int nr = c.h_nrows[(size_t)slot];
        if (c.ivf && c.ivf_rows[(size_t)slot] != nr) return false;
        for (int r = 0; r < nr; ++r) rows.push_back(slot * c.Rp + r);
    }
    if (rows.empty()) return true;
    std::vector<int16_t> have(rows.size());
    {
        std::vector<int16_t> all((size_t)c.high_water * c.Rp);
        mcopy(c, all.data(), c.row_list, sizeof(int16_t) * all.size(),
                           cudaMemcpyDeviceToHost);
        for (size_t i = 0; i < rows.size(); ++i) have[i] = all[(size_t)rows[i]];
    }
    if (!c.ivf) {
        for (int16_t l : have)
            if (l != -1) return false;
        return true;
    }
    if (c.ivf_C == 0) return false;
    MScratch<int64_t> d_rows(c, rows.size());
    MScratch<int32_t> d_as(c, rows.size());
    mcopy(c, d_rows.p, rows.data(), sizeof(int64_t) * rows.size(), cudaMemcpyHostToDevice);
    argmax_rows(c, d_rows.p, (int64_t)rows.size(), c.ivf_C, nullptr, d_as.p, c.mstream);
    SW_CUDA(cudaStreamSynchronize(c.mstream));
    std::vector<int32_t> as(rows.size());
    mcopy(c, as.data(), d_as.p, sizeof(int32_t) * as.size(), cudaMemcpyDeviceToHost);
    for (size_t i = 0; i < rows.size(); ++i)
        if ((int32_t)have[i] != as[i]) return false;
    return true;
}

// IvfIndex::insert (index.cpp:224-234) for entries just written to the arena, in order: entry e
// added rows [base[e], base[e] + nr[e]) of slot[e]. Rebuilds trigger between entries exactly
// where the reference's per-entry insert calls trigger them.
void ivf_on_insert(Ctx& c, const std::vector<int64_t>& slot, const std::vector<int32_t>& base,
                   const std::vector<int32_t>& nr) {
    const size_t n = slot.size();
    c.grp_dirty = true;
    {
        std::vector<int32_t> tot(n);
        for (size_t e = 0; e < n; ++e) tot[e] = base[e] + nr[e];
        ivf_mark_tails(c, slot, tot);
    }
    size_t e0 = 0;
    while (e0 < n) {
        if (nr[e0] > 0 && c.ivf_C == 0) {  // first insertion seeds a single centroid
            std::vector<float> v((size_t)c.D);
            fetch_row(c, slot[e0] * c.Rp + base[e0], v.data());
            c.h_cent = v;
            c.ivf_C = 1;
            upload_centroids(c, c.h_cent, 1);
        }
        // entries [e0, e1] share the current centroids (a rebuild can only follow e1)
        size_t e1 = e0;
        for (;; ++e1) {
            c.ivf_mutations += (uint64_t)nr[e1];
            c.ivf_rows[(size_t)slot[e1]] = base[e1] + nr[e1];
            if (c.ivf_mutations >= c.ivf_interval || e1 + 1 == n) break;
        }
        std::vector<int64_t> rows;
        for (size_t e = e0; e <= e1; ++e)
            for (int r = 0; r < nr[e]; ++r) rows.push_back(slot[e] * c.Rp + base[e] + r);
        if (!rows.empty()) {
            MScratch<int64_t> d_rows(c, rows.size());
            mcopy(c, d_rows.p, rows.data(), sizeof(int64_t) * rows.size(),
                               cudaMemcpyHostToDevice);
            argmax_rows(c, d_rows.p, (int64_t)rows.size(), c.ivf_C, c.row_list, nullptr, c.mstream);
            SW_CUDA(cudaStreamSynchronize(c.mstream));
        }
        if (c.ivf_mutations >= c.ivf_interval) ivf_rebuild(c);
        e0 = e1 + 1;
    }
}

// IvfIndex::remove (index.cpp:236-255), after the slot was cleared.
void ivf_on_remove(Ctx& c, int64_t slot) {
    c.grp_dirty = true;
    c.ivf_mutations += (uint64_t)c.ivf_rows[(size_t)slot];
    c.ivf_rows[(size_t)slot] = 0;
    if (c.ivf_mutations >= c.ivf_interval) ivf_rebuild(c);
}

void ivf_set_centroids(Ctx& c, const float* h, int C) {
    c.grp_dirty = true;
    c.h_cent.assign(h, h + (size_t)C * c.D);
    c.ivf_C = C;
    upload_centroids(c, c.h_cent, C);
    // reassign every stored row (list membership follows the centroids)
    std::vector<int64_t> rows;
    for (auto& kv : c.slot_of)
        for (int r = 0; r < c.ivf_rows[(size_t)kv.second]; ++r) rows.push_back(kv.second * c.Rp + r);
    if (!rows.empty() && C > 0) {
        MScratch<int64_t> d_rows(c, rows.size());
        mcopy(c, d_rows.p, rows.data(), sizeof(int64_t) * rows.size(), cudaMemcpyHostToDevice);
        argmax_rows(c, d_rows.p, (int64_t)rows.size(), C, c.row_list, nullptr, c.mstream);
        SW_CUDA(cudaStreamSynchronize(c.mstream));
    }
}

// ---------------------------------------------------------------- grouped IVF search
// The list-sorted arena copy: rows of list l contiguous from tile grp_tile0[l] (tile-aligned,
// so every 256-row tile belongs to ONE list), ascending slot order inside a list.
static void build_sorted(Ctx& c) {
    const int64_t S = c.high_water;
    const int C = c.ivf_C;
    std::vector<uint8_t> valid((size_t)S);
    std::vector<int16_t> rl((size_t)S);
    if (S > 0) {
        mcopy(c, valid.data(), c.valid, S, cudaMemcpyDeviceToHost);
        mcopy(c, rl.data(), c.row_list, 2 * S, cudaMemcpyDeviceToHost);
    }
    std::vector<int64_t> cnt((size_t)C, 0);
    for (int64_t i = 0; i < S; ++i)
        if (valid[(size_t)i] && rl[(size_t)i] >= 0 && rl[(size_t)i] < C) ++cnt[(size_t)rl[(size_t)i]];
    c.grp_tile0.assign((size_t)C, 0);
    c.grp_ntiles.assign((size_t)C, 0);
    int64_t t = 0;
    int maxt = 0;
    for (int j = 0; j < C; ++j) {
        c.grp_tile0[(size_t)j] = (int32_t)t;
        c.grp_ntiles[(size_t)j] = (int32_t)((cnt[(size_t)j] + 255) / 256);
        t += c.grp_ntiles[(size_t)j];
        maxt = std::max(maxt, (int)c.grp_ntiles[(size_t)j]);
    }
    c.grp_rows = t * 256;
    std::vector<int32_t> sorted((size_t)std::max<int64_t>(c.grp_rows, 1), -1);
    std::vector<int64_t> pos((size_t)C);
    for (int j = 0; j < C; ++j) pos[(size_t)j] = (int64_t)c.grp_tile0[(size_t)j] * 256;
    for (int64_t i = 0; i < S; ++i)
        if (valid[(size_t)i] && rl[(size_t)i] >= 0 && rl[(size_t)i] < C)
            sorted[(size_t)pos[(size_t)rl[(size_t)i]]++] = (int32_t)i;
    // chunking: tpc tiles per work item, <= kMaxSlices / nprobe chunks per list
    const int np = std::max(1, std::min(eff_nprobe(c), C));
    // 16+ tiles per item amortise the per-item pipeline ramp (A load, TMA / MMA fill, drain).
    // At the reference default (64 lists, nprobe 8, B = 1024, 1M rows: ~61 tiles per list),
    // with near-equal chunks taken largest first (k_group_plan): score 0.257 ms at 24 or 28
    // (3 or 2-3 chunks of ~20-30 tiles per list) vs 0.277 (16, 20) and 0.309 (32: 2 chunks
    // per list, too few items to balance over 148 CTAs). SW_IVF_TPC overrides.
    static const int tpc_min = [] {
        const char* e = getenv("SW_IVF_TPC");
        return e ? std::max(1, atoi(e)) : 24;
    }();
    c.grp_tpc = std::max(tpc_min, (maxt * np + kMaxSlices - 1) / kMaxSlices);
    c.grp_ch = std::max(1, (maxt + c.grp_tpc - 1) / c.grp_tpc);
    if (c.grp_rows > c.grp_cap_rows) {
        cudaFree(c.d_sorted_slot);
        cudaFree(c.d_rows_sorted);
        cudaFree(c.d_sorted_vbits);
        c.grp_cap_rows = c.grp_rows + 64 * 256;
        SW_CUDA(cudaMalloc(&c.d_sorted_slot, sizeof(int32_t) * c.grp_cap_rows));
        SW_CUDA(cudaMalloc(&c.d_rows_sorted, sizeof(__nv_bfloat16) * c.grp_cap_rows * c.Dp));
        SW_CUDA(cudaMalloc(&c.d_sorted_vbits, sizeof(uint32_t) * (c.grp_cap_rows / 32 + 16)));
        SW_REQUIRE(encode_2d_map(&c.tm_sorted, c.d_rows_sorted, (uint64_t)c.Dp,
                                 (uint64_t)c.grp_cap_rows, 256) &&
                       encode_2d_map(&c.tm_sorted_half, c.d_rows_sorted, (uint64_t)c.Dp,
                                     (uint64_t)c.grp_cap_rows, 128),
                   "grouped IVF: tensor map encode failed");
    }
    if (!c.d_list_tile0) {
        SW_CUDA(cudaMalloc(&c.d_list_tile0, sizeof(int32_t) * kMaxCentroids));
        SW_CUDA(cudaMalloc(&c.d_list_ntiles, sizeof(int32_t) * kMaxCentroids));
        SW_CUDA(cudaMalloc(&c.d_qcnt, sizeof(int32_t) * kMaxCentroids));
        SW_CUDA(cudaMalloc(&c.d_qbase, sizeof(int32_t) * (kMaxCentroids + 3)));
        SW_CUDA(cudaMalloc(&c.d_qlist, sizeof(int32_t) * (size_t)kMaxCentroids * c.Bmax));
    }
    std::vector<uint32_t> vb((size_t)(c.grp_cap_rows / 32 + 16), 0u);
    for (int64_t r = 0; r < c.grp_rows; ++r)
        if (sorted[(size_t)r] >= 0) vb[(size_t)(r >> 5)] |= 1u << (r & 31);
    if (c.grp_rows > 0)
        mcopy(c, c.d_sorted_slot, sorted.data(), sizeof(int32_t) * c.grp_rows,
                           cudaMemcpyHostToDevice);
    mcopy(c, c.d_sorted_vbits, vb.data(), sizeof(uint32_t) * vb.size(),
                       cudaMemcpyHostToDevice);
    std::vector<int32_t> t0v(kMaxCentroids, 0), ntv(kMaxCentroids, 0);
    std::copy(c.grp_tile0.begin(), c.grp_tile0.end(), t0v.begin());
    std::copy(c.grp_ntiles.begin(), c.grp_ntiles.end(), ntv.begin());
    mcopy(c, c.d_list_tile0, t0v.data(), 4 * kMaxCentroids, cudaMemcpyHostToDevice);
    mcopy(c, c.d_list_ntiles, ntv.data(), 4 * kMaxCentroids, cudaMemcpyHostToDevice);
    if (c.grp_rows > 0) {
        k_sort_rows<<<(unsigned)((c.grp_rows + 7) / 8), 256, 0, c.mstream>>>(
            c.d_sorted_slot, c.grp_rows, c.rows_bf, c.Dp, c.d_rows_sorted);
        SW_CUDA(cudaGetLastError());
    }
    SW_CUDA(cudaStreamSynchronize(c.mstream));
    c.grp_C = C;
    c.grp_max_chunks = c.grp_ch;
    c.grp_dirty = false;
}

int64_t ivf_group_prepare(Ctx& c, int B, cudaStream_t st) {
    static const bool enabled = [] {
        const char* e = getenv("SW_IVF_GROUPED");
        return !(e && e[0] == '0');
    }();
    if (!enabled || !c.ivf || c.ivf_C == 0 || c.Rp != 1 || !c.tc_ok) return 0;
    const int np = std::min(eff_nprobe(c), c.ivf_C);
    if (np >= c.ivf_C) return 0;
    if (c.grp_dirty || c.grp_C != c.ivf_C) build_sorted(c);
    if (c.grp_rows == 0) return 0;
    // SW_IVF_PAIR=1: items of two query blocks on CTA pairs. Measured (1M x 512, 64/8, B = 1024):
    // DRAM per launch 1.35 -> 1.07 GB (each tile once per 256 queries) but slower, 0.285 ->
    // 0.329 ms: the kernel is not HBM-bound at this size (tensor 39%, 4.6 TB/s), and a list with
    // one query block occupies two SMs for one block's work. Off by default.
    static const bool pair_ok = [] {
        const char* e = getenv("SW_IVF_PAIR");
        return e && e[0] == '1';
    }();
    c.grp_pair = pair_ok && c.num_sms >= 2;
    // blocks of 128 gathered queries: every list rounds up (and to an even count with pairs)
    const int64_t blocks = ((int64_t)B * np + 127) / 128 + (c.grp_pair ? 2 : 1) * c.ivf_C;
    const int64_t max_items = blocks * c.grp_ch;
    if (np * c.grp_ch > kMaxSlices) return 0;
    if (blocks * 128 > c.qg_cap) {
        cudaFree(c.d_qg);
        cudaFree(c.d_qmap);
        c.qg_cap = blocks * 128;
        SW_CUDA(cudaMalloc(&c.d_qg, sizeof(__nv_bfloat16) * c.qg_cap * c.Dp));
        SW_CUDA(cudaMalloc(&c.d_qmap, sizeof(int32_t) * c.qg_cap));
        SW_REQUIRE(encode_2d_map(&c.tm_qg, c.d_qg, (uint64_t)c.Dp, (uint64_t)c.qg_cap, 128),
                   "grouped IVF: tensor map encode failed");
    }
    if (max_items > c.items_cap) {
        cudaFree(c.d_items);
        c.items_cap = max_items;
        SW_CUDA(cudaMalloc(&c.d_items, sizeof(int4) * c.items_cap));
    }
    SW_CUDA(cudaMemsetAsync(c.d_qcnt, 0, sizeof(int32_t) * kMaxCentroids, st));
    SW_CUDA(cudaMemsetAsync(c.d_items, 0, sizeof(int4) * max_items, st));
    k_group_count<<<B, kMaxCentroids, 0, st>>>(c.prank, c.ivf_C, np, c.d_qcnt, c.d_qlist, c.Bmax);
    k_group_plan<<<1, kMaxCentroids, 0, st>>>(c.d_qcnt, c.ivf_C, c.d_list_tile0, c.d_list_ntiles,
                                              c.grp_tpc, c.grp_pair ? 1 : 0, ivf_lpt() ? 1 : 0,
                                              c.d_qbase, c.d_items);
    k_group_gather<<<(unsigned)((blocks * 128 + 7) / 8), 256, 0, st>>>(
        c.d_qcnt, c.d_qlist, c.d_qbase, c.ivf_C, c.Bmax, c.q_bf, c.Dp, c.d_qg, c.d_qmap,
        blocks * 128);
    const int n_chunks = np * c.grp_ch;
    k_fill_slices<<<(unsigned)(((int64_t)B * n_chunks + 255) / 256), 256, 0, st>>>(
        B, n_chunks, kMaxTopK, c.slice_cnt, c.cta_topk);
    SW_CUDA(cudaGetLastError());
    return max_items;
}

// Search-time probe ranking; returns true when lists restrict the search (nprobe < C).
bool launch_probe_rank(Ctx& c, const float* d_q, int B, cudaStream_t st) {
    if (!c.ivf) return false;
    if (c.ivf_C == 0) {  // no centroids: the reference search returns nothing (index.cpp:292)
        SW_CUDA(cudaMemsetAsync(c.prank, 0xFF, (size_t)B * kMaxCentroids, st));
        SW_CUDA(cudaMemsetAsync(c.pmask, 0, sizeof(uint64_t) * 4 * (size_t)B, st));
        return true;
    }
    const int np = std::min(eff_nprobe(c), c.ivf_C);
    if (np >= c.ivf_C) return false;  // every list probed == exhaustive
    const int cp = c.ivf_C <= 32 ? 32 : c.ivf_C <= 64 ? 64 : c.ivf_C <= 128 ? 128 : 256;
    {
        const int G = 256 / cp, DH = cp <= 64 ? 192 : cp == 128 ? 96 : 48;
        const size_t smem = sizeof(double) * ((size_t)DH * (cp + 1) + (size_t)G * DH + 256);
        auto launch = [&](auto kern) {
            ensure_smem_attr(c, kern, (size_t)200 * 1024);  // per context (= per device)
            kern<<<(B + G - 1) / G, 256, smem, st>>>(d_q, B, c.D, c.cent, c.Df, c.ivf_C, np,
                                                     c.prank, c.pmask);
        };
        if (cp == 32) launch(k_probe_rank_smem<32>);
        else if (cp == 64) launch(k_probe_rank_smem<64>);
        else if (cp == 128) launch(k_probe_rank_smem<128>);
        else launch(k_probe_rank_smem<256>);
    }
    SW_CUDA(cudaGetLastError());
    return true;
}

}  // namespace sw
