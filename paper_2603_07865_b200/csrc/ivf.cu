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

// Probe ranking per query (index.cpp:295-304): thread j computes dot(q, c_j) sequentially, its
// rank = #{i : s_i > s_j or (s_i == s_j and i < j)} is its position in the partial sort. Writes
// the rank (255 when not among the first nprobe) and the probed-list bitmask.
__global__ void k_probe_rank(const float* __restrict__ q, int D, const float* __restrict__ cent,
                             int Df, int C, int nprobe, uint8_t* __restrict__ prank,
                             uint64_t* __restrict__ pmask) {
    __shared__ double s[kMaxCentroids];
    __shared__ float qs[1024];
    const int b = blockIdx.x, j = threadIdx.x;
    const float* qb = q + (int64_t)b * D;
    for (int d = j; d < D && d < 1024; d += blockDim.x) qs[d] = qb[d];
    __syncthreads();
    if (j < C) {
        const float* c = cent + (int64_t)j * Df;
        double a = 0.0;
        for (int d = 0; d < D; ++d) a = fma((double)(d < 1024 ? qs[d] : qb[d]), (double)c[d], a);
        s[j] = a;
    }
    __syncthreads();
    if (j < kMaxCentroids) {
        uint8_t r = kNotProbed;
        if (j < C) {
            int rank = 0;
            for (int i = 0; i < C; ++i) rank += (s[i] > s[j] || (s[i] == s[j] && i < j)) ? 1 : 0;
            if (rank < nprobe) r = (uint8_t)rank;
        }
        prank[(int64_t)b * kMaxCentroids + j] = r;
        const unsigned ballot = __ballot_sync(0xffffffffu, r != kNotProbed);
        if ((j & 31) == 0) {
            uint32_t* pm32 = reinterpret_cast<uint32_t*>(pmask + (int64_t)b * 4);
            pm32[j >> 5] = ballot;
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
        SW_CUDA(cudaMemcpy(c.cent, pad.data(), sizeof(float) * pad.size(), cudaMemcpyHostToDevice));
}

void fetch_row(Ctx& c, int64_t row, float* out) {
    SW_CUDA(cudaMemcpy(out, c.rows + row * c.Df, sizeof(float) * c.D, cudaMemcpyDeviceToHost));
}

// kmeans (index.cpp:59-184) over the rows perm[0..n) (arena row indices, reference input order).
void kmeans(Ctx& c, const std::vector<int64_t>& perm, int cnum, uint64_t seed) {
    const int64_t n = (int64_t)perm.size();
    const int D = c.D;
    cudaStream_t st = c.mstream;
    MtRng rng(seed);
    DBuf<int64_t> d_perm((size_t)n);
    SW_CUDA(cudaMemcpy(d_perm.p, perm.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice));
    std::vector<float> cent((size_t)cnum * D);
    auto crow = [&](int j) { return cent.data() + (size_t)j * D; };

    // ---- k-means++ seeding with a running minimum distance (index.cpp:79-107)
    const uint64_t first = rng.uniform_int((uint64_t)n);
    fetch_row(c, perm[first], crow(0));
    DBuf<double> d_d2((size_t)n);
    DBuf<float> d_c((size_t)D);
    std::vector<double> d2((size_t)n);
    const int TB = 256;
    const int nb = (int)((n + TB - 1) / TB);
    auto d2_pass = [&](int j, int init) {
        SW_CUDA(cudaMemcpy(d_c.p, crow(j), sizeof(float) * D, cudaMemcpyHostToDevice));
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
    DBuf<int32_t> d_assign((size_t)n);
    DBuf<int32_t> d_mem((size_t)n);
    DBuf<int64_t> d_moff((size_t)cnum + 1);
    DBuf<double> d_sums((size_t)cnum * D);
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
                DBuf<double> bv((size_t)fb);
                DBuf<int64_t> bi((size_t)fb);
                k_farthest<<<fb, 256, 0, st>>>(c.rows, c.Df, D, d_perm.p, n, d_assign.p, c.cent,
                                               bv.p, bi.p);
                SW_CUDA(cudaGetLastError());
                std::vector<double> hv((size_t)fb);
                std::vector<int64_t> hi((size_t)fb);
                SW_CUDA(cudaMemcpy(hv.data(), bv.p, sizeof(double) * fb, cudaMemcpyDeviceToHost));
                SW_CUDA(cudaMemcpy(hi.data(), bi.p, sizeof(int64_t) * fb, cudaMemcpyDeviceToHost));
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
    DBuf<int64_t> d_s(slots.size());
    DBuf<int32_t> d_n(nr.size());
    SW_CUDA(cudaMemcpy(d_s.p, slots.data(), sizeof(int64_t) * slots.size(), cudaMemcpyHostToDevice));
    SW_CUDA(cudaMemcpy(d_n.p, nr.data(), sizeof(int32_t) * nr.size(), cudaMemcpyHostToDevice));
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
        SW_CUDA(cudaMemcpy(segs.data(), c.segs + slot * c.Rp, sizeof(sw_segment) * nr,
                           cudaMemcpyDeviceToHost));
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
    DBuf<int64_t> d_perm(perm.size());
    SW_CUDA(cudaMemcpy(d_perm.p, perm.data(), sizeof(int64_t) * perm.size(), cudaMemcpyHostToDevice));
    argmax_rows(c, d_perm.p, (int64_t)perm.size(), c.ivf_C, c.row_list, nullptr, c.mstream);
    SW_CUDA(cudaStreamSynchronize(c.mstream));
}

// IvfIndex::insert (index.cpp:224-234) for entries just written to the arena, in order: entry e
// added rows [base[e], base[e] + nr[e]) of slot[e]. Rebuilds trigger between entries exactly
// where the reference's per-entry insert calls trigger them.
void ivf_on_insert(Ctx& c, const std::vector<int64_t>& slot, const std::vector<int32_t>& base,
                   const std::vector<int32_t>& nr) {
    const size_t n = slot.size();
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
            DBuf<int64_t> d_rows(rows.size());
            SW_CUDA(cudaMemcpy(d_rows.p, rows.data(), sizeof(int64_t) * rows.size(),
                               cudaMemcpyHostToDevice));
            argmax_rows(c, d_rows.p, (int64_t)rows.size(), c.ivf_C, c.row_list, nullptr, c.mstream);
            SW_CUDA(cudaStreamSynchronize(c.mstream));
        }
        if (c.ivf_mutations >= c.ivf_interval) ivf_rebuild(c);
        e0 = e1 + 1;
    }
}

// IvfIndex::remove (index.cpp:236-255), after the slot was cleared.
void ivf_on_remove(Ctx& c, int64_t slot) {
    c.ivf_mutations += (uint64_t)c.ivf_rows[(size_t)slot];
    c.ivf_rows[(size_t)slot] = 0;
    if (c.ivf_mutations >= c.ivf_interval) ivf_rebuild(c);
}

void ivf_set_centroids(Ctx& c, const float* h, int C) {
    c.h_cent.assign(h, h + (size_t)C * c.D);
    c.ivf_C = C;
    upload_centroids(c, c.h_cent, C);
    // reassign every stored row (list membership follows the centroids)
    std::vector<int64_t> rows;
    for (auto& kv : c.slot_of)
        for (int r = 0; r < c.ivf_rows[(size_t)kv.second]; ++r) rows.push_back(kv.second * c.Rp + r);
    if (!rows.empty() && C > 0) {
        DBuf<int64_t> d_rows(rows.size());
        SW_CUDA(cudaMemcpy(d_rows.p, rows.data(), sizeof(int64_t) * rows.size(), cudaMemcpyHostToDevice));
        argmax_rows(c, d_rows.p, (int64_t)rows.size(), C, c.row_list, nullptr, c.mstream);
        SW_CUDA(cudaStreamSynchronize(c.mstream));
    }
}

// Search-time probe ranking; returns true when lists restrict the search (nprobe < C).
bool launch_probe_rank(Ctx& c, const float* d_q, int B, cudaStream_t st) {
    if (!c.ivf) return false;
    if (c.ivf_C == 0) {  // no centroids: the reference search returns nothing (index.cpp:292)
        SW_CUDA(cudaMemsetAsync(c.prank, 0xFF, (size_t)B * kMaxCentroids, st));
        SW_CUDA(cudaMemsetAsync(c.pmask, 0, sizeof(uint64_t) * 4 * (size_t)B, st));
        return true;
    }
    const int np = std::min(c.ivf_nprobe, c.ivf_C);
    if (np >= c.ivf_C) return false;  // every list probed == exhaustive
    k_probe_rank<<<B, kMaxCentroids, 0, st>>>(d_q, c.D, c.cent, c.Df, c.ivf_C, np, c.prank,
                                              c.pmask);
    SW_CUDA(cudaGetLastError());
    return true;
}

}  // namespace sw
