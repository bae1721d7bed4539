// Microbenchmark for the exact-rescoring row fetch (k_finish phase B): 1024 CTAs x 64 threads,
// lanes 0..16 of warp 0 each run a sequential fp64 chain over one random 2 KiB fp32 row of a
// 2 GiB arena, with the row either cold, bulk-prefetched to L2 (cp.async.bulk.prefetch.L2)
// some time before, or line-prefetched (prefetch.global.L2) right before. Prints cycles per row.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o /tmp/ub tools/ubench_rowfetch.cu
#include <cstdio>
#include <cstdint>

constexpr int D = 512;

template <int PF>
__device__ double chain(const float4* __restrict__ rp, const double* qd) {
    float4 ring[PF];
#pragma unroll
    for (int i = 0; i < PF; ++i) ring[i] = __ldg(rp + i);
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < D / 4; ++i) {
        const float4 x = ring[i % PF];
        if (i + PF < D / 4) ring[i % PF] = __ldg(rp + i + PF);
        s = fma(qd[4 * i + 0], (double)x.x, s);
        s = fma(qd[4 * i + 1], (double)x.y, s);
        s = fma(qd[4 * i + 2], (double)x.z, s);
        s = fma(qd[4 * i + 3], (double)x.w, s);
    }
    return s;
}

__global__ void __launch_bounds__(64, 7) k_rows(const float* rows, int64_t nrows, int mode,
                                                int spin, double* out, long long* cyc) {
    __shared__ double qd[D];
    for (int i = threadIdx.x; i < D; i += 64) qd[i] = 1.0 / (i + 1);
    const int lane = threadIdx.x & 31;
    const bool active = threadIdx.x < 17;
    uint64_t h = (uint64_t)(blockIdx.x * 17 + lane) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 29;
    const int64_t row = (int64_t)(h % (uint64_t)nrows);
    const float* rp = rows + row * D;
    if (active && mode == 1)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(rp), "r"(D * 4) : "memory");
    __syncthreads();
    const long long t0 = clock64();
    if (spin) {  // time between the bulk prefetch and the first use (phase A's work)
        while (clock64() - t0 < spin) {
        }
    }
    const long long t1 = clock64();
    if (active && mode == 2)
        for (int j = 0; j < D * 4 / 128; ++j)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(rp + 32 * j));
    double s = 0.0;
    if (active) s = mode == 3 ? chain<32>(reinterpret_cast<const float4*>(rp), qd)
                              : chain<16>(reinterpret_cast<const float4*>(rp), qd);
    const long long t2 = clock64();
    if (active) out[blockIdx.x * 17 + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t2 - t1;
}

int main() {
    const int64_t nrows = 1 << 20;
    float* rows;
    double* out;
    long long* cyc;
    cudaMalloc(&rows, (size_t)nrows * D * 4);
    cudaMemset(rows, 0, (size_t)nrows * D * 4);
    cudaMalloc(&out, 1024 * 17 * 8);
    cudaMallocManaged(&cyc, 1024 * 8);
    void* flush;
    cudaMalloc(&flush, 256 << 20);
    const char* names[] = {"cold (PF16)", "bulk prefetch L2", "line prefetch L2", "cold (PF32)"};
    for (int mode = 0; mode < 4; ++mode)
        for (int spin : {0, 4000, 16000}) {
            if (spin && mode != 1) continue;
            cudaMemset(flush, mode, 256 << 20);  // evict the arena from L2
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            k_rows<<<1024, 64>>>(rows, nrows, mode, spin, out, cyc);
            cudaEventRecord(b);
            cudaDeviceSynchronize();
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            double m = 0, mx = 0;
            for (int i = 0; i < 1024; ++i) {
                m += cyc[i];
                mx = cyc[i] > mx ? cyc[i] : mx;
            }
            printf("%-18s spin %5d: chain cycles mean %.0f max %.0f, kernel %.1f us\n",
                   names[mode], spin, m / 1024, mx, ms * 1e3);
        }
    return 0;
}
