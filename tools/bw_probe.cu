// bw_probe.cu -- HBM bandwidth of the stage kernel's access pattern without
// its arithmetic: NR fields read + NW written per node, 8192^2 fp64.
//  mode 0: flat grid-stride (STREAM-like), mode 1: row march (128-col tiles,
//  R rows per CTA, 1-row register prefetch), mode 2: row march, 2-row prefetch.
#include <cstdio>
#include <cuda_runtime.h>
#define NRMAX 16
struct Ptrs { const double* in[NRMAX]; double* out[5]; };

template <int NR, int NW>
__global__ void flat(Ptrs P, long long n) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        double s = 0;
#pragma unroll
        for (int f = 0; f < NR; ++f) s += __ldg(P.in[f] + k);
#pragma unroll
        for (int f = 0; f < NW; ++f) P.out[f][k] = s + f;
    }
}

template <int NR, int NW, int PF>
__global__ void __launch_bounds__(128) march(Ptrs P, int nx, int ny, int rpb) {
    const int i = blockIdx.x * 128 + threadIdx.x;
    const int j0 = blockIdx.y * rpb, j1 = min(ny, j0 + rpb);
    double buf[PF][NR];
#pragma unroll
    for (int p = 0; p < PF; ++p)
#pragma unroll
        for (int f = 0; f < NR; ++f) buf[p][f] = __ldg(P.in[f] + (unsigned)(j0 + p) * nx + i);
    for (int j = j0; j < j1; j += PF) {
#pragma unroll
        for (int p = 0; p < PF; ++p) {
            double s = 0;
#pragma unroll
            for (int f = 0; f < NR; ++f) s += buf[p][f];
            const int jl = j + p + PF;
            if (jl < j1) {
#pragma unroll
                for (int f = 0; f < NR; ++f) buf[p][f] = __ldg(P.in[f] + (unsigned)jl * nx + i);
            }
            if (j + p < j1) {
#pragma unroll
                for (int f = 0; f < NW; ++f) P.out[f][(unsigned)(j + p) * nx + i] = s + f;
            }
        }
    }
}

int main() {
    const int nx = 8192, ny = 8192;
    const long long n = (long long)nx * ny;
    Ptrs P;
    double* pool;
    cudaMalloc(&pool, sizeof(double) * n * (NRMAX + 5));
    cudaMemset(pool, 0, sizeof(double) * n * (NRMAX + 5));
    for (int f = 0; f < NRMAX; ++f) P.in[f] = pool + f * n;
    for (int f = 0; f < 5; ++f) P.out[f] = pool + (NRMAX + f) * n;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char* name, int nr, int nw, auto launch) {
        launch(); cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
        printf("%-28s R%-2d W%d  %.3f ms  %.0f GB/s\n", name, nr, nw, ms, (nr + nw) * 8.0 * n / ms / 1e6);
    };
    run("flat", 11, 5, [&] { flat<11, 5><<<148 * 16, 256>>>(P, n); });
    run("flat", 6, 5, [&] { flat<6, 5><<<148 * 16, 256>>>(P, n); });
    run("flat", 16, 5, [&] { flat<16, 5><<<148 * 16, 256>>>(P, n); });
    run("flat copy", 1, 1, [&] { flat<1, 1><<<148 * 16, 256>>>(P, n); });
    for (int rpb : {32, 64, 128, 256}) {
        char nm[64];
        snprintf(nm, 64, "march pf1 rpb=%d", rpb);
        run(nm, 11, 5, [&] { march<11, 5, 1><<<dim3(64, ny / rpb), 128>>>(P, nx, ny, rpb); });
        snprintf(nm, 64, "march pf2 rpb=%d", rpb);
        run(nm, 11, 5, [&] { march<11, 5, 2><<<dim3(64, ny / rpb), 128>>>(P, nx, ny, rpb); });
    }
    run("march pf1 rpb=64", 6, 5, [&] { march<6, 5, 1><<<dim3(64, ny / 64), 128>>>(P, nx, ny, 64); });
    run("march pf2 rpb=64", 6, 5, [&] { march<6, 5, 2><<<dim3(64, ny / 64), 128>>>(P, nx, ny, 64); });
    run("march pf1 rpb=64", 16, 5, [&] { march<16, 5, 1><<<dim3(64, ny / 64), 128>>>(P, nx, ny, 64); });
    run("march pf2 rpb=64", 16, 5, [&] { march<16, 5, 2><<<dim3(64, ny / 64), 128>>>(P, nx, ny, 64); });
    return 0;
}
