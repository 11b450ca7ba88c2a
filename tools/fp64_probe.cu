// fp64_probe.cu -- measured FP64 (non-tensor) instruction throughput of this
// B200: independent DMUL/DADD chains (no FMA, like the --fmad=false stage
// kernels), many warps, no memory traffic.  Reports thread-instructions/s and
// the ratio to 64 FP64 lanes x 148 SMs x the SM clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false tools/fp64_probe.cu -o tools/fp64_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void __launch_bounds__(256) probe(double* out, int iters, double a, double b) {
    double x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            x[c] = __dmul_rn(x[c], a);  // 1 DMUL
            x[c] = __dadd_rn(x[c], b);  // 1 DADD
        }
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

template <int CHAINS>
static void run(int blocks_per_sm, int threads) {
    int dev = 0, sms = 0, clk_khz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    double* out;
    cudaMalloc(&out, 8);
    const int iters = 4096;
    const int blocks = sms * blocks_per_sm;
    probe<CHAINS><<<blocks, threads>>>(out, 64, 0.999999, 1e-7);  // warm
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<CHAINS><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double instr = 2.0 * CHAINS * (double)iters * blocks * threads;
    const double rate = instr / (ms * 1e-3);
    const double peak_at_max_clock = 64.0 * sms * clk_khz * 1e3;
    printf("chains %2d  warps/SM %2d  %.3f ms  %.1f G FP64 thread-instr/s  = %.3f of 64 lanes x %d SMs x %.0f MHz (max clock)\n",
           CHAINS, blocks_per_sm * threads / 32, ms, rate / 1e9, rate / peak_at_max_clock, sms, clk_khz / 1e3);
    cudaFree(out);
}

int main() {
    // (chains = independent dependency chains per thread = ILP)
    run<1>(3, 128);  // 12 warps/SM
    run<1>(4, 128);  // 16
    run<1>(5, 128);  // 20
    run<2>(3, 128);
    run<2>(4, 128);
    run<2>(5, 128);
    run<4>(3, 128);
    run<4>(4, 128);
    run<4>(5, 128);
    run<8>(4, 128);
    run<8>(4, 256);
    return 0;
}
