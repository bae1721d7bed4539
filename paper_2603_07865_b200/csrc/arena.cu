// K5 — arena updates: the device data plane of the Cache Manager.
//
// Replaces the per-row std::vector<float> storage of IvfIndex lists (index.hpp:19-23,
// index.cpp:226-255) and CacheEntry::segment_vectors (cache.hpp:21) with one SoA arena:
//   rows    [S*Rp][Df]  fp32 master rows            (exact fp64 rescoring reads these)
//   rows_bf [S*Rp][Dp]  bf16 shadow, K zero-padded  (tcgen05 scoring streams these via TMA)
//   sneg    [S*Rp]      fp64 clamp01(cos(row, negative)) precomputed at insert (selector.cpp:41-42)
//   segs    [S*Rp]      PyramidDescriptor per row
// An entry owns Rp = next_pow2(rows_per_entry) consecutive rows; unused rows of the shadow
// repeat row 0 so the tensor-core per-entry max needs no mask.
#include <cmath>

#include "sw_internal.cuh"

namespace sw {

namespace {

__device__ __forceinline__ double seq_dot(const float* __restrict__ a,
                                          const float* __restrict__ b, int D) {
    // Sum_i (double)a_i * (double)b_i in order i = 0..D-1 (core.cpp:26-30). The fp32 x fp32
    // product is exact in fp64, so the fused multiply-add rounds exactly like mul-then-add.
    double s = 0.0;
    for (int i = 0; i < D; ++i) s = fma((double)a[i], (double)b[i], s);
    return s;
}

__device__ __forceinline__ double clamp01(double v) { return fmin(1.0, fmax(0.0, v)); }

__device__ __forceinline__ double clamp_cos(double v) {  // core.cpp:35-36
    if (v > 1.0) v = 1.0;
    if (v < -1.0) v = -1.0;
    return v;
}

// One block per inserted entry. Rows land at [row_base, row_base + n) of the entry's slot.
__global__ void k_insert_rows(int64_t n, const int64_t* __restrict__ slot_of,
                              const int32_t* __restrict__ row_base,
                              const int64_t* __restrict__ row_off, const uint64_t* __restrict__ ids,
                              const float* __restrict__ src, const sw_segment* __restrict__ src_segs,
                              float* __restrict__ rows, __nv_bfloat16* __restrict__ rows_bf,
                              double* __restrict__ sneg, sw_segment* __restrict__ segs,
                              uint64_t* __restrict__ slot_ids, int32_t* __restrict__ slot_nrows,
                              uint8_t* __restrict__ valid, uint32_t* __restrict__ valid_bits,
                              uint32_t* __restrict__ norms,
                              const float* __restrict__ neg, int have_neg, int D, int Df, int Dp,
                              int Rp) {
    int64_t e = blockIdx.x;
    if (e >= n) return;
    const int64_t slot = slot_of[e];
    const int64_t r0 = row_off[e], r1 = row_off[e + 1];
    const int nr = (int)(r1 - r0);
    const int base = row_base ? row_base[e] : 0;
    for (int r = 0; r < nr; ++r) {
        const float* s = src + (r0 + r) * (int64_t)D;
        const int64_t dst = slot * Rp + base + r;
        float* df = rows + dst * Df;
        __nv_bfloat16* db = rows_bf + dst * Dp;
        for (int d = threadIdx.x; d < Dp; d += blockDim.x) {
            float v = d < D ? s[d] : 0.0f;
            if (d < Df) df[d] = v;
            db[d] = __float2bfloat16_rn(v);
        }
        if (threadIdx.x == 0) segs[dst] = src_segs[r0 + r];
    }
    __syncthreads();
    // per-row scalars: thread r owns row r (sequential fp64 sums keep the reference's order)
    for (int r = threadIdx.x; r < nr; r += blockDim.x) {
        const int64_t dst = slot * Rp + base + r;
        const float* df = rows + dst * Df;
        // |e|, |e - bf16(e)|, |bf16(e)|: the data-dependent terms of the tcgen05 error bound
        double nn = 0.0, dd = 0.0, bb = 0.0;
        for (int d = 0; d < D; ++d) {
            const double x = (double)df[d];
            const double xb = (double)__bfloat162float(__float2bfloat16_rn(df[d]));
            nn = fma(x, x, nn);
            dd = fma(x - xb, x - xb, dd);
            bb = fma(xb, xb, bb);
        }
        atomicMax(&norms[0], f2ord((float)sqrt(nn) * (1.0f + 1e-6f)));
        atomicMax(&norms[1], f2ord((float)sqrt(dd) * (1.0f + 1e-6f)));
        atomicMax(&norms[2], f2ord((float)sqrt(bb) * (1.0f + 1e-6f)));
        sneg[dst] = have_neg ? clamp01(clamp_cos(seq_dot(df, neg, D))) : 0.0;
    }
    // pad rows repeat row 0 in the bf16 shadow (approximate per-entry max unaffected)
    const int total = base + nr;
    for (int r = total; r < Rp; ++r) {
        const __nv_bfloat16* s0 = rows_bf + (slot * Rp) * Dp;
        __nv_bfloat16* dd = rows_bf + (slot * Rp + r) * Dp;
        for (int d = threadIdx.x; d < Dp; d += blockDim.x) dd[d] = s0[d];
    }
    if (threadIdx.x == 0) {
        slot_ids[slot] = ids[e];
        slot_nrows[slot] = total;
        valid[slot] = 1;
        atomicOr(&valid_bits[slot >> 5], 1u << (slot & 31));
    }
}

__global__ void k_clear_slot(int64_t slot, uint8_t* valid, uint32_t* valid_bits, int32_t* nrows) {
    valid[slot] = 0;
    nrows[slot] = 0;
    atomicAnd(&valid_bits[slot >> 5], ~(1u << (slot & 31)));
}

__global__ void k_copy_latents(int64_t n, const int64_t* __restrict__ slot_of,
                               const float* __restrict__ src, const int64_t* __restrict__ lat_off,
                               const int32_t* __restrict__ tsrc_in, float* __restrict__ latent,
                               int32_t* __restrict__ tsrc, int64_t Lslots, int C, int Tmax,
                               int F) {
    int64_t e = blockIdx.y;
    if (e >= n) return;
    const int64_t slot = slot_of[e];
    const int ts = min(tsrc_in[e], Tmax);
    const float* s = src + lat_off[e];
    float* d = latent + (slot % Lslots) * (int64_t)C * Tmax * F;
    const int64_t total = (int64_t)C * ts * F;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t c = i / ((int64_t)ts * F);
        int64_t rem = i - c * ts * F;
        d[c * (int64_t)Tmax * F + rem] = s[c * (int64_t)tsrc_in[e] * F + rem];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) tsrc[slot] = ts;
}

__global__ void k_recompute_sneg(int64_t n_rows_total, int Rp, const int32_t* __restrict__ nrows,
                                 const uint8_t* __restrict__ valid, const float* __restrict__ rows,
                                 const float* __restrict__ neg, double* __restrict__ sneg, int D,
                                 int Df) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_rows_total) return;
    int64_t slot = i / Rp;
    int r = (int)(i - slot * Rp);
    if (!valid[slot] || r >= nrows[slot]) return;
    sneg[i] = clamp01(clamp_cos(seq_dot(rows + i * Df, neg, D)));
}

// ---------------------------------------------------------------- synthetic fill (benchmark)
__device__ __forceinline__ void philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
        uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
        uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}
__device__ __forceinline__ float u01(uint32_t x) { return (float)((x >> 8) | 1u) * 0x1.0p-24f; }

// One block per entry: full row = normalise(N(0,1)^D) (core.cpp:110-114 shape); pyramid rows =
// normalise(full + 0.1 dir) (index.cpp:33-46 shape). Written to a packed staging buffer.
__global__ void k_synth_rows(int64_t n, uint64_t seed, uint64_t first_id, int D, int R,
                             double delta_floor_levels, float* __restrict__ out,
                             sw_segment* __restrict__ segs, uint64_t* __restrict__ ids_out,
                             double* __restrict__ dur_out) {
    extern __shared__ double sh[];  // [D] doubles
    __shared__ double red[32];
    int64_t e = blockIdx.x;
    if (e >= n) return;
    const uint64_t id = first_id + (uint64_t)e;
    for (int r = 0; r < R; ++r) {
        // normals for this (entry, row)
        for (int d4 = threadIdx.x; d4 * 4 < D; d4 += blockDim.x) {
            uint32_t c[4] = {(uint32_t)d4, (uint32_t)r, (uint32_t)id, (uint32_t)(id >> 32)};
            philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
            float rr0 = sqrtf(-2.0f * logf(u01(c[0]))), t0 = 6.2831853f * u01(c[1]);
            float rr1 = sqrtf(-2.0f * logf(u01(c[2]))), t1 = 6.2831853f * u01(c[3]);
            float z[4] = {rr0 * cosf(t0), rr0 * sinf(t0), rr1 * cosf(t1), rr1 * sinf(t1)};
            for (int j = 0; j < 4 && d4 * 4 + j < D; ++j) {
                float g = z[j];
                double v = (double)g;
                if (r > 0) v = (double)out[(e * R) * (int64_t)D + d4 * 4 + j] + 0.1 * v;
                sh[d4 * 4 + j] = v;
            }
        }
        __syncthreads();
        double s = 0.0;
        for (int d = threadIdx.x; d < D; d += blockDim.x) s += sh[d] * sh[d];
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
            red[0] = sqrt(t);
        }
        __syncthreads();
        double nrm = red[0];
        for (int d = threadIdx.x; d < D; d += blockDim.x)
            out[(e * R + r) * (int64_t)D + d] = (float)(sh[d] / nrm);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        uint32_t c[4] = {0xD0u, 0u, (uint32_t)id, (uint32_t)(id >> 32)};
        philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
        double dur = 4.0 + 8.0 * ((double)(c[0] >> 11) * 0x1.0p-21);
        ids_out[e] = id;
        dur_out[e] = dur;
        int row = 0;
        for (int level = 0; row < R; ++level) {
            int tiles = 1 << level;
            double len = dur / tiles;
            for (int i = 0; i < tiles && row < R; ++i, ++row) {
                sw_segment sg;
                sg.level = level;
                sg.reserved = 0;
                sg.start_s = i * len;
                sg.length_s = len;
                segs[e * R + row] = sg;
            }
        }
    }
}

__global__ void k_synth_latents(int64_t slot0, int64_t n, uint64_t seed,
                                const double* __restrict__ dur, float* __restrict__ latent,
                                int32_t* __restrict__ tsrc, int64_t Lslots, int C, int Tmax, int F,
                                double fps) {
    int64_t e = blockIdx.y;
    if (e >= n) return;
    const int64_t slot = slot0 + e;
    int ts = (int)llround(dur[e] * fps);
    ts = min(max(ts, 1), Tmax);
    if (slot >= Lslots) {  // slots beyond the latent arena share (slot % Lslots)
        if (blockIdx.x == 0 && threadIdx.x == 0) tsrc[slot] = ts;
        return;
    }
    float4* d = reinterpret_cast<float4*>(latent + slot * (int64_t)C * Tmax * F);
    const int64_t total4 = (int64_t)C * Tmax * F / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total4;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t c[4] = {(uint32_t)i, 0x1A7u, (uint32_t)slot, (uint32_t)(slot >> 32)};
        philox(c, (uint32_t)seed ^ 0x5A5Au, (uint32_t)(seed >> 32));
        float r0 = sqrtf(-2.0f * logf(u01(c[0]))), t0 = 6.2831853f * u01(c[1]);
        float r1 = sqrtf(-2.0f * logf(u01(c[2]))), t1 = 6.2831853f * u01(c[3]);
        d[i] = make_float4(r0 * cosf(t0), r0 * sinf(t0), r1 * cosf(t1), r1 * sinf(t1));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) tsrc[slot] = ts;
}

}  // namespace

// Insert launcher used by capi.cu (ids + row_base travel with the slots).
void launch_insert_rows_full(Ctx& c, int64_t n, const int64_t* d_slot, const int32_t* d_base,
                             const int64_t* d_row_off, const uint64_t* d_ids, const float* d_rows,
                             const sw_segment* d_segs, cudaStream_t st) {
    if (n <= 0) return;
    for (int64_t off = 0; off < n; off += 65535 * 16) {
        int64_t m = std::min<int64_t>(n - off, 65535LL * 16);
        k_insert_rows<<<(unsigned)m, 128, 0, st>>>(
            m, d_slot + off, d_base ? d_base + off : nullptr, d_row_off + off, d_ids + off,
            d_rows, d_segs, c.rows, c.rows_bf, c.sneg, c.segs, c.ids, c.nrows, c.valid,
            c.valid_bits, c.norms, c.neg, c.have_neg ? 1 : 0, c.D, c.Df, c.Dp, c.Rp);
    }
    SW_CUDA(cudaGetLastError());
}

void launch_clear_slot(Ctx& c, int64_t slot, cudaStream_t st) {
    k_clear_slot<<<1, 1, 0, st>>>(slot, c.valid, c.valid_bits, c.nrows);
    SW_CUDA(cudaGetLastError());
}

void launch_copy_latents(Ctx& c, int64_t n, const int64_t* d_slot, const float* d_lat,
                         const int64_t* d_lat_off, const int32_t* d_tsrc, cudaStream_t st) {
    if (n <= 0) return;
    for (int64_t off = 0; off < n; off += 65535) {
        int64_t m = std::min<int64_t>(n - off, 65535);
        dim3 grid(8, (unsigned)m);
        k_copy_latents<<<grid, 256, 0, st>>>(m, d_slot + off, d_lat, d_lat_off + off,
                                             d_tsrc + off, c.latent, c.tsrc, c.Lslots, c.C,
                                             c.Tmax, c.F);
    }
    SW_CUDA(cudaGetLastError());
}

void launch_recompute_sneg(Ctx& c, cudaStream_t st) {
    int64_t total = c.high_water * c.Rp;
    if (total == 0) return;
    k_recompute_sneg<<<(unsigned)((total + 127) / 128), 128, 0, st>>>(
        total, c.Rp, c.nrows, c.valid, c.rows, c.neg, c.sneg, c.D, c.Df);
    SW_CUDA(cudaGetLastError());
}

void launch_fill_synthetic(Ctx& c, int64_t slot0, int64_t n, uint64_t first_id, uint64_t seed,
                           double delta, cudaStream_t st) {
    (void)delta;
    const int R = c.R;
    const int64_t chunk = 32768;  // grid.y of the latent fill must stay <= 65535
    float* stage = nullptr;
    sw_segment* segs = nullptr;
    uint64_t* ids = nullptr;
    double* dur = nullptr;
    int64_t* slots = nullptr;
    int64_t* offs = nullptr;
    SW_CUDA(cudaMallocAsync(&stage, sizeof(float) * chunk * R * c.D, st));
    SW_CUDA(cudaMallocAsync(&segs, sizeof(sw_segment) * chunk * R, st));
    SW_CUDA(cudaMallocAsync(&ids, sizeof(uint64_t) * chunk, st));
    SW_CUDA(cudaMallocAsync(&dur, sizeof(double) * chunk, st));
    SW_CUDA(cudaMallocAsync(&slots, sizeof(int64_t) * chunk, st));
    SW_CUDA(cudaMallocAsync(&offs, sizeof(int64_t) * (chunk + 1), st));
    std::vector<int64_t> h_slots(chunk), h_offs(chunk + 1);
    for (int64_t done = 0; done < n; done += chunk) {
        int64_t m = std::min(chunk, n - done);
        for (int64_t i = 0; i < m; ++i) h_slots[i] = slot0 + done + i;
        for (int64_t i = 0; i <= m; ++i) h_offs[i] = i * R;
        SW_CUDA(cudaMemcpyAsync(slots, h_slots.data(), sizeof(int64_t) * m, cudaMemcpyHostToDevice, st));
        SW_CUDA(cudaMemcpyAsync(offs, h_offs.data(), sizeof(int64_t) * (m + 1), cudaMemcpyHostToDevice, st));
        k_synth_rows<<<(unsigned)m, 128, sizeof(double) * c.D, st>>>(
            m, seed, first_id + done, c.D, R, 0.0, stage, segs, ids, dur);
        SW_CUDA(cudaGetLastError());
        launch_insert_rows_full(c, m, slots, nullptr, offs, ids, stage, segs, st);
        if (c.latent) {
            dim3 grid(16, (unsigned)m);
            k_synth_latents<<<grid, 256, 0, st>>>(slot0 + done, m, seed, dur, c.latent, c.tsrc,
                                                  c.Lslots, c.C, c.Tmax, c.F, c.cfg.latent_fps);
            SW_CUDA(cudaGetLastError());
        }
        SW_CUDA(cudaStreamSynchronize(st));  // h_slots/h_offs are reused next chunk
    }
    cudaFreeAsync(stage, st);
    cudaFreeAsync(segs, st);
    cudaFreeAsync(ids, st);
    cudaFreeAsync(dur, st);
    cudaFreeAsync(slots, st);
    cudaFreeAsync(offs, st);
}

namespace {
// chosen segment row of each request (slot * Rp + segment.reserved), zeros on a miss
__global__ void k_choice_rows(const sw_choice* __restrict__ ch, int B, const float* __restrict__ rows,
                              int Rp, int Df, int D, float* __restrict__ out) {
    const int b = blockIdx.x;
    if (b >= B) return;
    const sw_choice c = ch[b];
    const float* src = c.hit ? rows + ((int64_t)c.slot * Rp + c.segment.reserved) * Df : nullptr;
    for (int d = threadIdx.x; d < D; d += blockDim.x) out[(int64_t)b * D + d] = src ? src[d] : 0.0f;
}
}  // namespace

void launch_choice_rows(Ctx& c, const sw_choice* d_ch, int B, float* d_rows, cudaStream_t st) {
    if (B <= 0) return;
    k_choice_rows<<<B, 128, 0, st>>>(d_ch, B, c.rows, c.Rp, c.Df, c.D, d_rows);
    SW_CUDA(cudaGetLastError());
}

}  // namespace sw
