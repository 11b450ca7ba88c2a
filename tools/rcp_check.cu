// rcp_check.cu -- exhaustive-style check of hsgn_dev::rcp_or_nan against
// __drcp_rn (tests/test_gpu_rcp.py builds and runs it on the B200).
// Inputs: splitmix64-hashed bit patterns over every exponent (plus the
// neighbourhood of powers of two and the range edges).  Required: wherever
// rcp_or_nan is not NaN it equals __drcp_rn bit for bit, and it is NaN
// nowhere inside 2^-930 < |h| < 2^990 (its fast range is [2^-935, 2^993)).
#include <cstdio>
#include <cstdlib>
#include "../paper_2601_02540_b200/csrc/sgn_device.cuh"

__device__ unsigned long long mix(unsigned long long z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__global__ void check(unsigned long long n, unsigned long long seed, unsigned long long* out) {
    unsigned long long bad = 0, nan_in_range = 0, fast = 0;
    for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < n;
         k += (unsigned long long)gridDim.x * blockDim.x) {
        unsigned long long bits = mix(k ^ seed);
        if ((k & 3) == 1) bits = (bits & 0x800fffffffffffffull) | ((unsigned long long)(k >> 2) % 2047 << 52);
        if ((k & 3) == 2) bits = (((unsigned long long)(k >> 2) % 2047) << 52) + ((bits & 7) - 3);  // near 2^e
        const double h = __longlong_as_double((long long)bits);
        const double a = hsgn_dev::rcp_or_nan(h);
        const double b = __drcp_rn(h);
        const double ah = fabs(h);
        if (!isnan(a)) {
            ++fast;
            if (__double_as_longlong(a) != __double_as_longlong(b)) ++bad;
        } else if (ah > 0x1p-930 && ah < 0x1p990) {
            ++nan_in_range;
        }
    }
    atomicAdd(&out[0], bad);
    atomicAdd(&out[1], nan_in_range);
    atomicAdd(&out[2], fast);
}

int main(int argc, char** argv) {
    const unsigned long long n = argc > 1 ? strtoull(argv[1], nullptr, 10) : (1ull << 30);
    unsigned long long* d;
    cudaMalloc(&d, 3 * sizeof(unsigned long long));
    cudaMemset(d, 0, 3 * sizeof(unsigned long long));
    check<<<148 * 8, 256>>>(n, 20261018ull, d);
    unsigned long long h[3];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    if (cudaGetLastError() != cudaSuccess) return 2;
    printf("samples %llu fast %llu mismatches %llu nan_in_range %llu\n", n, h[2], h[0], h[1]);
    return (h[0] || h[1]) ? 1 : 0;
}
