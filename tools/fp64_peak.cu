// fp64_peak.cu -- microbenchmark: DFMA pipe vs fp64 mma.sync (DMMA m8n8k4)
// throughput on this GPU (MEASURED_PEAKS.json has no fp64 entry).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b)
{
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dmma_loop(double* out, int iters, double a)
{
    double A = a * (threadIdx.x + 1), B = a * (threadIdx.x + 2);
    double c[8][2];
    for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(A), "d"(B));
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[threadIdx.x] = s;
}

int main()
{
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double* out;
    cudaMalloc(&out, 1 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int blocksPerSm : {4, 8}) {
        const int grid = sms * blocksPerSm, bs = 256;
        dfma_loop<<<grid, bs>>>(out, 100, 1.0000001, 1e-9);
        cudaEventRecord(e0);
        dfma_loop<<<grid, bs>>>(out, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * iters * (double)grid * bs;
        printf("{\"kernel\":\"dfma\",\"blocks_per_sm\":%d,\"tflops\":%.2f}\n", blocksPerSm, flops / ms / 1e9);
        dmma_loop<<<grid, bs>>>(out, 100, 1e-3);
        cudaEventRecord(e0);
        dmma_loop<<<grid, bs>>>(out, iters, 1e-3);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        // per warp-mma: 8*8*4 FMAs = 512 flops
        flops = 512.0 * 8 * iters * (double)grid * (bs / 32);
        printf("{\"kernel\":\"dmma_m8n8k4\",\"blocks_per_sm\":%d,\"tflops\":%.2f}\n", blocksPerSm, flops / ms / 1e9);
    }
    printf("{\"sms\":%d,\"clock_khz\":%d,\"err\":\"%s\"}\n", sms, clk, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
