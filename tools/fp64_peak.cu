// fp64_peak.cu -- measured fp64 FMA throughput and DADD issue rate of this B200
// ("measure an fp64 FMA peak on the box"; the ALU roofline of
// the ExBLAS dot).  8 independent dependency chains per thread, 148*k CTAs.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double *out, int iters, double a, double b) {
    double c[8];
    for (int j = 0; j < 8; ++j) c[j] = threadIdx.x * 1e-9 + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) c[j] = __fma_rn(c[j], a, b);
    }
    double s = 0;
    for (int j = 0; j < 8; ++j) s += c[j];
    if (s == 12345.678) out[0] = s;
}
__global__ void dadd_loop(double *out, int iters, double a) {
    double c[8];
    for (int j = 0; j < 8; ++j) c[j] = threadIdx.x * 1e-9 + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) c[j] = __dadd_rn(c[j], a);
    }
    double s = 0;
    for (int j = 0; j < 8; ++j) s += c[j];
    if (s == 12345.678) out[0] = s;
}
int lat_main();
int main(int argc, char **argv) {
    if (argc > 1) return lat_main();
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double *d; cudaMalloc(&d, 8);
    int iters = 20000, bs = 256, grid = nsm * 8;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int k = 0; k < 2; ++k) {
        for (int w = 0; w < 3; ++w) { if (k == 0) dfma_loop<<<grid, bs>>>(d, iters, 0.999999, 1e-7); else dadd_loop<<<grid, bs>>>(d, iters, 1e-7); }
        cudaEventRecord(e0);
        if (k == 0) dfma_loop<<<grid, bs>>>(d, iters, 0.999999, 1e-7); else dadd_loop<<<grid, bs>>>(d, iters, 1e-7);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)grid * bs * iters * 8;
        printf("{\"op\": \"%s\", \"Gop_per_s\": %.1f, \"per_sm_per_clk_at_1965MHz\": %.2f, \"ms\": %.3f}\n",
               k == 0 ? "DFMA" : "DADD", ops / ms / 1e6, ops / (ms * 1e-3) / nsm / 1.965e9, ms);
    }
    return 0;
}
// ---- latency probe (single thread, dependent chains), run with argv[1] == "lat"
__global__ void lat_kernel(double *out, long long *cyc, double a, int n) {
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, a);
    long long t1 = clock64();
    double y = a;
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) y = __fma_rn(y, a, a);
    long long t3 = clock64();
    out[0] = x + y;
    cyc[0] = t1 - t0;
    cyc[1] = t3 - t2;
}
int lat_main() {
    double *d; long long *c; cudaMalloc(&d, 8); cudaMalloc(&c, 16);
    int n = 4096;
    lat_kernel<<<1, 1>>>(d, c, 1e-9, n);
    lat_kernel<<<1, 1>>>(d, c, 1e-9, n);
    long long h[2]; cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
    printf("{\"DADD_latency_cycles\": %.2f, \"DFMA_latency_cycles\": %.2f}\n", (double)h[0] / n, (double)h[1] / n);
    return 0;
}
