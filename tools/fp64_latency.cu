// Microbenchmark: dependent-chain latency of fp64 DADD / DFMA / DMUL and F2F on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, float* fin, int n) {
    double s = out[0], a = out[1], b = out[2];
    float f = fin[threadIdx.x];
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) s = __dadd_rn(s, a);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) s = fma(s, a, b);
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) s = __dmul_rn(s, a);
    long long t3 = clock64();
    double acc = 0.0;
    for (int i = 0; i < n; ++i) { acc = __dadd_rn(acc, (double)f); f = (float)acc; }
    long long t4 = clock64();
    float x = f;
    for (int i = 0; i < n; ++i) x = fmaf(x, 1.0001f, 0.5f);
    long long t5 = clock64();
    out[3 + threadIdx.x] = s + acc + x;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
    double* d; long long* c; float* f;
    cudaMalloc(&d, 4096); cudaMalloc(&c, 64); cudaMalloc(&f, 4096);
    double h[3] = {1.0, 1.0000001, 1e-9};
    cudaMemcpy(d, h, 24, cudaMemcpyHostToDevice);
    cudaMemset(f, 0, 4096);
    const int n = 4096;
    for (int threads : {32, 128, 1024}) {
        k<<<1, threads>>>(d, c, f, n);
        k<<<1, threads>>>(d, c, f, n);
        long long hc[5];
        cudaMemcpy(hc, c, 40, cudaMemcpyDeviceToHost);
        printf("threads=%d  cycles/op: dadd %.1f  dfma %.1f  dmul %.1f  f2f+dadd+f2f %.1f  ffma %.1f\n", threads,
               hc[0] / (double)n, hc[1] / (double)n, hc[2] / (double)n, hc[3] / (double)n, hc[4] / (double)n);
    }
    // throughput: many warps per SM
    k<<<148, 1024>>>(d, c, f, n);
    cudaDeviceSynchronize();
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
