// Microbenchmark of k_finish's phase-B chain in isolation: one warp, `lanes` lanes each running
// the sequential fp64 dot (core.cpp:26-30) of a query (doubles in smem) with one 2 KiB fp32 row
// (random rows of a 2 GiB arena, pre-touched so they sit in L2), for several load strategies.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/_uc tools/ubench_chain.cu
#include <cstdint>
#include <cstdio>

constexpr int D = 512, N4 = D / 4;

template <int PF>
__device__ double chain_ring(const float4* __restrict__ rp, const double* qd) {
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

// query doubles software-pipelined through registers too: the two LDS.128 of step i + QA are
// issued at step i, so the shared-memory latency is off the DFMA chain
template <int PF, int QA>
__device__ double chain_ring_q(const float4* __restrict__ rp, const double* qd) {
    float4 ring[PF];
    double2 qa[QA], qb[QA];
    const double2* q2 = reinterpret_cast<const double2*>(qd);
#pragma unroll
    for (int i = 0; i < PF; ++i) ring[i] = __ldg(rp + i);
#pragma unroll
    for (int i = 0; i < QA; ++i) {
        qa[i] = q2[2 * i];
        qb[i] = q2[2 * i + 1];
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N4; ++i) {
        const float4 x = ring[i % PF];
        if (i + PF < N4) ring[i % PF] = __ldg(rp + i + PF);
        const double2 a = qa[i % QA], b = qb[i % QA];
        if (i + QA < N4) {
            qa[i % QA] = q2[2 * (i + QA)];
            qb[i % QA] = q2[2 * (i + QA) + 1];
        }
        s = fma(a.x, (double)x.x, s);
        s = fma(a.y, (double)x.y, s);
        s = fma(b.x, (double)x.z, s);
        s = fma(b.y, (double)x.w, s);
    }
    return s;
}

__device__ __forceinline__ float4 ld_plain(const float4* p) {
    float4 v;
    asm volatile("ld.global.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
template <int PF>
__device__ double chain_plain(const float4* __restrict__ rp, const double* qd) {
    float4 ring[PF];
#pragma unroll
    for (int i = 0; i < PF; ++i) ring[i] = ld_plain(rp + i);
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N4; ++i) {
        const float4 x = ring[i % PF];
        if (i + PF < N4) ring[i % PF] = ld_plain(rp + i + PF);
        s = fma(qd[4 * i + 0], (double)x.x, s);
        s = fma(qd[4 * i + 1], (double)x.y, s);
        s = fma(qd[4 * i + 2], (double)x.z, s);
        s = fma(qd[4 * i + 3], (double)x.w, s);
    }
    return s;
}

// per-lane cp.async (LDGSTS, no register scoreboards) of its own row into a private smem ring of
// NS stages x CH float4, completion by cp.async.wait_group
template <int NS, int CH>
__device__ double chain_cpasync(const float4* __restrict__ rp, const double* qd, float4* mine) {
    auto issue = [&](int c) {
        if (c < N4 / CH) {
#pragma unroll
            for (int u = 0; u < CH; ++u)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                 (uint32_t)__cvta_generic_to_shared(mine + (c % NS) * CH + u)),
                             "l"(rp + c * CH + u)
                             : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int c = 0; c < NS - 1; ++c) issue(c);
    double s = 0.0;
    for (int c = 0; c < N4 / CH; ++c) {
        issue(c + NS - 1);
        asm volatile("cp.async.wait_group %0;" ::"n"(NS - 1) : "memory");
        const float4* x4 = mine + (c % NS) * CH;
        const double* q = qd + c * CH * 4;
#pragma unroll
        for (int u = 0; u < CH; ++u) {
            const float4 x = x4[u];
            s = fma(q[4 * u + 0], (double)x.x, s);
            s = fma(q[4 * u + 1], (double)x.y, s);
            s = fma(q[4 * u + 2], (double)x.z, s);
            s = fma(q[4 * u + 3], (double)x.w, s);
        }
    }
    return s;
}

// conversions pipelined: the doubles of float4 i + CA are formed at step i
template <int PF, int CA>
__device__ double chain_conv_ahead(const float4* __restrict__ rp, const double* qd) {
    float4 ring[PF];
    double xd[CA][4];
#pragma unroll
    for (int i = 0; i < PF; ++i) ring[i] = __ldg(rp + i);
#pragma unroll
    for (int i = 0; i < CA; ++i) {
        xd[i][0] = ring[i].x; xd[i][1] = ring[i].y; xd[i][2] = ring[i].z; xd[i][3] = ring[i].w;
        ring[i] = __ldg(rp + i + PF);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N4; ++i) {
        const double a0 = xd[i % CA][0], a1 = xd[i % CA][1], a2 = xd[i % CA][2], a3 = xd[i % CA][3];
        if (i + CA < N4) {
            const int j = i + CA;
            const float4 x = ring[j % PF];
            if (j + PF < N4) ring[j % PF] = __ldg(rp + j + PF);
            xd[i % CA][0] = x.x; xd[i % CA][1] = x.y; xd[i % CA][2] = x.z; xd[i % CA][3] = x.w;
        }
        s = fma(qd[4 * i + 0], a0, s);
        s = fma(qd[4 * i + 1], a1, s);
        s = fma(qd[4 * i + 2], a2, s);
        s = fma(qd[4 * i + 3], a3, s);
    }
    return s;
}
// exact fp32 -> fp64 by bit manipulation on the integer pipe for normal floats (sign | exponent
// rebias | mantissa shift); any zero / subnormal / inf / nan in the warp's float4 falls back to
// F2F for that float4
__device__ __forceinline__ double f2d_bits(float x) {
    const uint32_t u = __float_as_uint(x);
    const uint32_t hi = ((u & 0x7FFFFFFFu) >> 3) + ((u & 0x80000000u) | 0x38000000u);
    return __hiloint2double((int)hi, (int)(u << 29));
}
__device__ __forceinline__ bool normal4(float4 x) {
    const float m = fminf(fminf(fabsf(x.x), fabsf(x.y)), fminf(fabsf(x.z), fabsf(x.w)));
    const float M = fmaxf(fmaxf(fabsf(x.x), fabsf(x.y)), fmaxf(fabsf(x.z), fabsf(x.w)));
    return m >= 1.17549435e-38f && M <= 3.40282347e38f;  // false for nan too
}
template <int PF>
__device__ double chain_bits(const float4* __restrict__ rp, const double* qd) {
    float4 ring[PF];
#pragma unroll
    for (int i = 0; i < PF; ++i) ring[i] = __ldg(rp + i);
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N4; ++i) {
        const float4 x = ring[i % PF];
        if (i + PF < N4) ring[i % PF] = __ldg(rp + i + PF);
        double a0, a1, a2, a3;
        if (__all_sync(__activemask(), normal4(x))) {
            a0 = f2d_bits(x.x); a1 = f2d_bits(x.y); a2 = f2d_bits(x.z); a3 = f2d_bits(x.w);
        } else {
            a0 = x.x; a1 = x.y; a2 = x.z; a3 = x.w;
        }
        s = fma(qd[4 * i + 0], a0, s);
        s = fma(qd[4 * i + 1], a1, s);
        s = fma(qd[4 * i + 2], a2, s);
        s = fma(qd[4 * i + 3], a3, s);
    }
    return s;
}
template <int PF>
__device__ double chain_bits_nocheck(const float4* __restrict__ rp, const double* qd) {
    float4 ring[PF];
#pragma unroll
    for (int i = 0; i < PF; ++i) ring[i] = __ldg(rp + i);
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N4; ++i) {
        const float4 x = ring[i % PF];
        if (i + PF < N4) ring[i % PF] = __ldg(rp + i + PF);
        s = fma(qd[4 * i + 0], f2d_bits(x.x), s);
        s = fma(qd[4 * i + 1], f2d_bits(x.y), s);
        s = fma(qd[4 * i + 2], f2d_bits(x.z), s);
        s = fma(qd[4 * i + 3], f2d_bits(x.w), s);
    }
    return s;
}

// x already doubles in shared memory (no conversion on the chain)
__device__ double chain_dd(const double* xd, const double* qd) {
    double s = 0.0;
#pragma unroll 16
    for (int i = 0; i < D; ++i) s = fma(qd[i], xd[i], s);
    return s;
}

// the whole row staged into shared memory first (coalesced by the warp), then the chain
__device__ double chain_smem(const float* __restrict__ row0, const int64_t* rows, int lanes,
                             const double* qd, float* stage) {
    const int lane = threadIdx.x & 31;
    for (int r = 0; r < lanes; ++r) {
        const float4* src = reinterpret_cast<const float4*>(row0 + rows[r] * D);
        for (int i = lane; i < N4; i += 32)
            reinterpret_cast<float4*>(stage + r * (D + 4))[i] = __ldg(src + i);
    }
    __syncwarp();
    double s = 0.0;
    if (lane < lanes) {
        const float* x = stage + lane * (D + 4);
#pragma unroll 16
        for (int i = 0; i < D; ++i) s = fma(qd[i], (double)x[i], s);
    }
    return s;
}

__global__ void k_chain(const float* rows_base, const int64_t* rows, int lanes, int mode,
                        double* out, long long* cyc) {
    extern __shared__ double sm[];
    double* qd = sm;
    float* stage = reinterpret_cast<float*>(sm + D);
    for (int i = threadIdx.x; i < D; i += 32) qd[i] = 1.0 / (i + 1);
    __syncwarp();
    const int lane = threadIdx.x & 31;
    const float4* rp = reinterpret_cast<const float4*>(rows_base + rows[lane % lanes] * D);
    const long long t0 = clock64();
    double s = 0.0;
    if (mode == 3) {
        s = chain_smem(rows_base, rows, lanes, qd, stage);
    } else if (lane < lanes) {
        if (mode == 0) s = chain_ring<8>(rp, qd);
        if (mode == 1) s = chain_ring<16>(rp, qd);
        if (mode == 2) s = chain_ring<32>(rp, qd);
        if (mode == 4) s = chain_ring_q<16, 2>(rp, qd);
        if (mode == 5) s = chain_ring_q<16, 4>(rp, qd);
        if (mode == 6) s = chain_plain<16>(rp, qd);
        if (mode == 7)
            s = chain_cpasync<4, 4>(rp, qd, reinterpret_cast<float4*>(stage) + lane * 16);
        if (mode == 8)
            s = chain_cpasync<4, 8>(rp, qd, reinterpret_cast<float4*>(stage) + lane * 32);
        if (mode == 9) s = chain_conv_ahead<16, 2>(rp, qd);
        if (mode == 10) s = chain_conv_ahead<16, 4>(rp, qd);
        if (mode == 11) s = chain_dd(qd, qd);
        if (mode == 12) s = chain_bits<16>(rp, qd);
        if (mode == 13) s = chain_bits_nocheck<16>(rp, qd);
    }
    __syncwarp();
    const long long t1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_touch(const float* p, int64_t n, float* sink) {
    float a = 0;
    for (int64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a += p[i];
    if (a == 12345.f) *sink = a;
}

int main() {
    const int64_t nrows = 1 << 20;
    float* rows;
    cudaMalloc(&rows, (size_t)nrows * D * 4);
    cudaMemset(rows, 0x3f, (size_t)nrows * D * 4);  // 0x3f3f3f3f = 0.747 (normal)
    int64_t h[32];
    for (int i = 0; i < 32; ++i) h[i] = (int64_t)((uint64_t)(i + 1) * 0x9E3779B97F4A7C15ull % nrows);
    int64_t* d_rows;
    cudaMalloc(&d_rows, sizeof(h));
    cudaMemcpy(d_rows, h, sizeof(h), cudaMemcpyHostToDevice);
    double* out;
    cudaMalloc(&out, 32 * 8);
    long long* cyc;
    cudaMallocManaged(&cyc, 8);
    float* sink;
    cudaMalloc(&sink, 4);
    const size_t smem = D * 8 + 32 * (D + 4) * 4;
    cudaFuncSetAttribute(k_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const char* names[] = {"reg ring PF=8", "reg ring PF=16", "reg ring PF=32", "smem staged",
                           "ring16 + q 2 ahead", "ring16 + q 4 ahead", "plain ld ring16",
                           "cp.async 4x4", "cp.async 4x8", "conv 2 ahead", "conv 4 ahead",
                           "x doubles in smem", "int-pipe convert+check", "int-pipe convert"};
    for (int lanes : {1, 15, 32})
        for (int mode = 0; mode < 14; ++mode) {
            for (int rep = 0; rep < 3; ++rep) {
                // rows hot in L2: touch exactly the rows used
                for (int i = 0; i < lanes; ++i)
                    k_touch<<<4, 128>>>(rows + h[i] * D, D, sink);
                k_chain<<<1, 32, smem>>>(rows, d_rows, lanes, mode, out, cyc);
                cudaDeviceSynchronize();
            }
            printf("lanes %2d %-16s: %6lld cycles (%.1f / element)\n", lanes, names[mode], *cyc,
                   *cyc / 512.0);
        }
    return 0;
}
