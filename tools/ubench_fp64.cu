// Microbenchmark: latency of the exact-rescoring chain's building blocks on this GPU
// (dependent DFMA, F2F.F64.F32 + DFMA, LDS.64 broadcast + DFMA). Prints cycles per step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o /tmp/ubench tools/ubench_fp64.cu
#include <cstdio>

__global__ void k_chain(const float* x, double* out, long long* cyc, int mode) {
    __shared__ double qd[512];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) qd[i] = 1.0 + i * 1e-3;
    __syncthreads();
    float xr[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) xr[i] = x[threadIdx.x * 16 + i];
    double s = 0.0, a = 1.000001;
    const long long t0 = clock64();
    if (mode == 0) {  // dependent DFMA only
#pragma unroll 16
        for (int i = 0; i < 512; ++i) s = fma(a, s, 1e-3);
    } else if (mode == 1) {  // + F2F of a register float (independent of the chain)
#pragma unroll 16
        for (int i = 0; i < 512; ++i) s = fma(a, (double)xr[i & 15], s);
    } else if (mode == 2) {  // + LDS.64 of the query + F2F
#pragma unroll 16
        for (int i = 0; i < 512; ++i) s = fma(qd[i], (double)xr[i & 15], s);
    } else {  // dependent DADD
#pragma unroll 16
        for (int i = 0; i < 512; ++i) s = s + a;
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    float* x;
    double* out;
    long long* cyc;
    cudaMalloc(&x, 1 << 20);
    cudaMemset(x, 0, 1 << 20);
    cudaMalloc(&out, 1 << 20);
    cudaMallocManaged(&cyc, 8 * 2048);
    const char* names[] = {"dfma chain", "dfma + f2f", "dfma + lds + f2f", "dadd chain"};
    for (int mode = 0; mode < 4; ++mode) {
        for (int warps : {1, 8}) {
            for (int rep = 0; rep < 2; ++rep) k_chain<<<1, 32 * warps>>>(x, out, cyc, mode);
            cudaDeviceSynchronize();
            printf("%-18s warps/SM %d: %.2f cycles/step\n", names[mode], warps, cyc[0] / 512.0);
        }
        // 8 CTAs per SM x 148 SMs, one warp each (the finish kernel's phase-B shape)
        k_chain<<<148 * 8, 32>>>(x, out, cyc, mode);
        cudaDeviceSynchronize();
        double m = 0;
        for (int i = 0; i < 148 * 8; ++i) m += cyc[i];
        printf("%-18s 1184 CTAs x 1 warp: %.2f cycles/step\n", names[mode], m / (148 * 8) / 512.0);
    }
    return 0;
}
