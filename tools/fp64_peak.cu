// fp64_peak.cu — measure the B200 FP64 (DFMA) issue rate: the ALU roofline
// denominator of the FP64-bound stage kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu
// Prints one JSON line: DFMA/s per GPU, TFLOP/s (2 flops per DFMA), SM clock.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
    double x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; i++) x[i] = threadIdx.x * 1e-9 + i;
    for (int n = 0; n < iters; n++) {
#pragma unroll
        for (int i = 0; i < ILP; i++) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; i++) s += x[i];
    if (s == 12345.678) out[0] = s;  // keep the loop alive
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);  // kHz
    double* out;
    cudaMalloc(&out, 8);
    const int iters = 1 << 14;
    const int threads = 256, blocks = sms * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dfma_loop<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);  // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0);
        dfma_loop<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double dfma = (double)blocks * threads * iters * 8;
    const double rate = dfma / (best * 1e-3);
    printf("{\"dfma_per_s\": %.4e, \"fp64_tflops\": %.3f, \"sms\": %d, \"max_clock_mhz\": %.0f, "
           "\"dfma_per_sm_per_clk_at_max\": %.2f, \"ms\": %.3f}\n",
           rate, 2 * rate / 1e12, sms, clk / 1e3, rate / sms / (clk * 1e3), best);
    return 0;
}
