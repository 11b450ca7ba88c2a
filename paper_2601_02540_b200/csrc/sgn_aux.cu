// sgn_aux.cu -- the non-stage kernels of the hot path: SBP-norm weighted
// row reductions (mass / energy / energy rate / L2 error), the depth
// pre-check of the standalone rhs(), state axpy and weighted-RMS (startup
// step estimate), and init_auxiliary.  All fp64, --fmad=false, reference
// association (see sgn_device.cuh).
#include <cuda_runtime.h>

#include "sgn_device.cuh"

namespace hsgn_dev {



// ---- compensated (double-double) accumulation helpers
struct DD {
    double hi, lo;
};
__device__ __forceinline__ DD two_sum(double a, double b) {
    const double s = dadd(a, b);
    const double bb = dsub(s, a);
    const double e = dadd(dsub(a, dsub(s, bb)), dsub(b, bb));
    return {s, e};
}
__device__ __forceinline__ DD dd_add(DD x, DD y) {
    DD s = two_sum(x.hi, y.hi);
    const double lo = dadd(s.lo, dadd(x.lo, y.lo));
    return two_sum(s.hi, lo);
}
__device__ __forceinline__ DD dd_add_d(DD x, double y) {
    DD s = two_sum(x.hi, y);
    return two_sum(s.hi, dadd(s.lo, x.lo));
}

// Pointwise integrands (exact reference association):
//   kind 0: h                                         (model.hpp:77-80)
//   kind 1: energy density                            (model.hpp:63-75)
//   kind 2: <dE/dq, q_t>                              (analysis.hpp:52-65)
//   kind 3: (a_f - b_f)^2                             (analysis.hpp:19-23)
__device__ __forceinline__ double integrand(int kind, const AuxArgs& A, const double* q, const double* qt,
                                            int field, long long off) {
    const long long fs = A.fs;
    if (kind == 0) return q[field * fs + off];
    if (kind == 3) {
        const double d = dsub(q[field * fs + off], qt[field * fs + off]);
        return dmul(d, d);
    }
    const double h = q[off], u = q[fs + off], v = q[2 * fs + off], w = q[3 * fs + off], e = q[4 * fs + off];
    const double b = A.b[off];
    if (kind == 1) {
        const double g_half = dmul(0.5, A.g), lam_sixth = A.lambda / 6.0;
        const double r1 = dsub(e / h, 1.0);
        const double s = dadd(dadd(dadd(dmul(0.5, dadd(dmul(u, u), dmul(v, v))), dmul(w, w) / 6.0),
                                   dmul(g_half, dadd(h, dmul(2.0, b)))),
                              dmul(dmul(lam_sixth, r1), r1));
        return dmul(h, s);
    }
    const double lam_third = A.lambda / 3.0, lam_sixth = A.lambda / 6.0;
    const double r = e / h;
    const double dE_dh = dadd(dadd(dadd(dadd(dmul(0.5, dadd(dmul(u, u), dmul(v, v))), dmul(w, w) / 6.0),
                                        dmul(A.g, h)),
                                   dmul(A.g, b)),
                              dmul(lam_sixth, dsub(1.0, dmul(r, r))));
    const double dE_du = dmul(h, u), dE_dv = dmul(h, v), dE_dw = dmul(h, w) / 3.0;
    const double dE_de = dmul(-lam_third, dsub(1.0, r));
    return dadd(dadd(dadd(dadd(dmul(dE_dh, qt[off]), dmul(dE_du, qt[fs + off])), dmul(dE_dv, qt[2 * fs + off])),
                     dmul(dE_dw, qt[3 * fs + off])),
                dmul(dE_de, qt[4 * fs + off]));
}

// One CTA per row: rows[j] = sum_i wx_i F_ij, compensated (sbp.hpp:225-231).
__global__ void __launch_bounds__(256) row_sum_kernel(const AuxArgs A, int kind, const double* q,
                                                      const double* qt, int field, double* rows) {
    __shared__ double sh[256], sl[256];
    const int j = blockIdx.x;
    const long long base = (long long)j * A.nx;
    DD acc{0.0, 0.0};
    for (int i = threadIdx.x; i < A.nx; i += blockDim.x) {
        const double wx = (A.x_bounded && (i == 0 || i == A.nx - 1)) ? dmul(0.5, A.dx) : A.dx;
        acc = dd_add_d(acc, dmul(wx, integrand(kind, A, q, qt, field, base + i)));
    }
    sh[threadIdx.x] = acc.hi;
    sl[threadIdx.x] = acc.lo;
    __syncthreads();
    if (threadIdx.x == 0) {
        DD t{0.0, 0.0};
        for (int k = 0; k < (int)blockDim.x; ++k) t = dd_add(t, DD{sh[k], sl[k]});
        rows[j] = dadd(t.hi, t.lo);
    }
}

// The recorder's conservation row (io.hpp:137-144) in one pass over q, b and
// q_t: rows[k*ny + j] for k = 0 mass, 1 energy, 2 energy rate, each with
// the accumulation order of row_sum_kernel (so bit-identical to it).
__global__ void __launch_bounds__(256) cons_rows_kernel(const AuxArgs A, const double* q, const double* qt,
                                                        double* rows) {
    __shared__ double sh[3][256], sl[3][256];
    const int j = blockIdx.x;
    const long long base = (long long)j * A.nx;
    DD acc[3] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    for (int i = threadIdx.x; i < A.nx; i += blockDim.x) {
        const double wx = (A.x_bounded && (i == 0 || i == A.nx - 1)) ? dmul(0.5, A.dx) : A.dx;
#pragma unroll
        for (int k = 0; k < 3; ++k) acc[k] = dd_add_d(acc[k], dmul(wx, integrand(k, A, q, qt, 0, base + i)));
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        sh[k][threadIdx.x] = acc[k].hi;
        sl[k][threadIdx.x] = acc[k].lo;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        const int k = threadIdx.x;
        DD t{0.0, 0.0};
        for (int m = 0; m < (int)blockDim.x; ++m) t = dd_add(t, DD{sh[k][m], sl[k][m]});
        rows[(long long)k * A.ny + j] = dadd(t.hi, t.lo);
    }
}

// Gauge samples h + b at the recorder's nodes (io.hpp:131-135).
__global__ void gauge_kernel(const double* h, const double* b, const long long* idx, int n, double* out) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n) out[g] = dadd(h[idx[g]], b[idx[g]]);
}

// Depth pre-check of the standalone rhs() (rhs.hpp:94-97): count !(h > 0).
__global__ void depth_check_kernel(const double* h, long long n, unsigned long long* bad) {
    unsigned long long c = 0;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x)
        if (!(h[k] > 0.0)) ++c;
    if (c) atomicAdd(bad, c);
}

// out = a + c*x over the 5 fields (state_add1, time_integration.hpp:61-75).
__global__ void axpy5_kernel(const double* a, double c, const double* x, double* out, long long n,
                             long long fs) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < 5 * n;
         k += (long long)gridDim.x * blockDim.x) {
        const long long f = k / n, o = f * fs + (k - f * n);
        out[o] = dadd(a[o], dmul(c, x[o]));
    }
}

// Per-block partial sums of (x / (atol + rtol |ref|))^2 (weighted_rms,
// time_integration.hpp:144-162).
__global__ void __launch_bounds__(256) wrms_kernel(const double* x, const double* ref, double atol, double rtol,
                                                   long long n, long long fs, double* part) {
    __shared__ double sh[256];
    double s = 0.0;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < 5 * n;
         k += (long long)gridDim.x * blockDim.x) {
        const long long f = k / n, o = f * fs + (k - f * n);
        const double w = dadd(atol, dmul(rtol, fabs(ref[o])));
        const double r = x[o] / w;
        s = dadd(s, dmul(r, r));
    }
    sh[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < (int)blockDim.x; ++k) t = dadd(t, sh[k]);
        part[blockIdx.x] = t;
    }
}

__device__ __forceinline__ int aux_row(const AuxArgs& A, int jr) {
    if (jr < 0) return A.y_lo == YE_WRAP ? A.ny - 1 : (A.y_lo == YE_CLAMP ? 0 : -1);
    if (jr >= A.ny) return A.y_hi == YE_WRAP ? 0 : (A.y_hi == YE_CLAMP ? A.ny - 1 : A.ny);
    return jr;
}

template <bool POW2>
__device__ __forceinline__ double aux_dx(const AuxArgs& A, const double* f, int i, long long row) {
    const int n = A.nx;
    int il, ir;
    double c = A.cpx;
    if (A.x_bounded && i == 0) {
        il = 0; ir = 1; c = A.c1x;
    } else if (A.x_bounded && i == n - 1) {
        il = n - 2; ir = n - 1; c = A.c1x;
    } else {
        il = i == 0 ? n - 1 : i - 1;
        ir = i == n - 1 ? 0 : i + 1;
    }
    return sbp_d<POW2>(c, f[row + il], f[row + ir]);
}

template <bool POW2>
__device__ __forceinline__ double aux_dy(const AuxArgs& A, const double* f, int i, int j) {
    const long long p = A.nx;
    int jl, jr;
    double c = A.cpy;
    if (A.y_bounded_lo && j == 0) {
        jl = 0; jr = 1; c = A.c1y;
    } else if (A.y_bounded_hi && j == A.ny - 1) {
        jl = A.ny - 2; jr = A.ny - 1; c = A.c1y;
    } else {
        jl = aux_row(A, j - 1);
        jr = aux_row(A, j + 1);
    }
    return sbp_d<POW2>(c, f[jl * p + i], f[jr * p + i]);
}

// init_auxiliary (model.hpp:93-105): eta = h; w = -h (Dx u + Dy v) + 1.5 (u Dx b + v Dy b).
template <bool POW2>
__global__ void init_aux_kernel(const AuxArgs A, double* q) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (i >= A.nx) return;
    const long long fs = A.fs, row = (long long)j * A.nx, off = row + i;
    const double h = q[off], u = q[fs + off], v = q[2 * fs + off];
    const double du = aux_dx<POW2>(A, q + fs, i, row);
    const double dv = aux_dy<POW2>(A, q + 2 * fs, i, j);
    const double dbx = aux_dx<POW2>(A, A.b, i, row);
    const double dby = aux_dy<POW2>(A, A.b, i, j);
    q[3 * fs + off] = dadd(dmul(-h, dadd(du, dv)), dmul(1.5, dadd(dmul(u, dbx), dmul(v, dby))));
    q[4 * fs + off] = h;
}

// ---------------------------------------------------------------- launchers

cudaError_t launch_row_sums(const AuxArgs& A, int kind, const double* q, const double* qt, int field,
                            double* rows, cudaStream_t st) {
    row_sum_kernel<<<A.ny, 256, 0, st>>>(A, kind, q, qt, field, rows);
    return cudaGetLastError();
}

cudaError_t launch_cons_rows(const AuxArgs& A, const double* q, const double* qt, double* rows, cudaStream_t st) {
    cons_rows_kernel<<<A.ny, 256, 0, st>>>(A, q, qt, rows);
    return cudaGetLastError();
}

cudaError_t launch_gauges(const double* h, const double* b, const long long* idx, int n, double* out,
                          cudaStream_t st) {
    gauge_kernel<<<(n + 127) / 128, 128, 0, st>>>(h, b, idx, n, out);
    return cudaGetLastError();
}

cudaError_t launch_depth_check(const double* h, long long n, unsigned long long* bad, cudaStream_t st) {
    const int blocks = (int)((n + 255) / 256 < 148 * 8 ? (n + 255) / 256 : 148 * 8);
    depth_check_kernel<<<blocks, 256, 0, st>>>(h, n, bad);
    return cudaGetLastError();
}

cudaError_t launch_axpy5(const double* a, double c, const double* x, double* out, long long n, long long fs,
                         cudaStream_t st) {
    const long long t = 5 * n;
    const int blocks = (int)((t + 255) / 256 < 148 * 8 ? (t + 255) / 256 : 148 * 8);
    axpy5_kernel<<<blocks, 256, 0, st>>>(a, c, x, out, n, fs);
    return cudaGetLastError();
}

int wrms_blocks() { return 148 * 4; }

cudaError_t launch_wrms(const double* x, const double* ref, double atol, double rtol, long long n, long long fs,
                        double* part, cudaStream_t st) {
    wrms_kernel<<<wrms_blocks(), 256, 0, st>>>(x, ref, atol, rtol, n, fs, part);
    return cudaGetLastError();
}

cudaError_t launch_init_aux(const AuxArgs& A, double* q, cudaStream_t st) {
    dim3 grid((A.nx + 127) / 128, A.ny);
    if (A.pow2)
        init_aux_kernel<true><<<grid, 128, 0, st>>>(A, q);
    else
        init_aux_kernel<false><<<grid, 128, 0, st>>>(A, q);
    return cudaGetLastError();
}

// Factors of the manufactured source term along one grid direction:
// (sin 2pi x, cos 2pi x, sin 4pi x, cos 4pi x) at x = x0 + i dx
// (Grid2D::x, grid.hpp:24-25), read by sgn_stage.cu mms_source.
__global__ void src_factor_kernel(double x0, double dx, int n, double* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double tp = 2.0 * 3.14159265358979323846, fp = 4.0 * 3.14159265358979323846;
    const double x = dadd(x0, dmul((double)i, dx));
    double s1, c1, s2, c2;
    sincos(tp * x, &s1, &c1);
    sincos(fp * x, &s2, &c2);
    out[4 * i] = s1;
    out[4 * i + 1] = c1;
    out[4 * i + 2] = s2;
    out[4 * i + 3] = c2;
}

cudaError_t launch_src_factors(double x0, double dx, int n, double* out, cudaStream_t st) {
    src_factor_kernel<<<(n + 255) / 256, 256, 0, st>>>(x0, dx, n, out);
    return cudaGetLastError();
}

}  // namespace hsgn_dev
