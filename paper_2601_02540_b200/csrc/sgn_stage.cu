// sgn_stage.cu -- the fused fp64 split-form SGN stage kernel for sm_100a.
//
// One launch evaluates the reference's whole tendency (rhs.hpp:77-214:
// products pass, 22 SBP stencil passes, wall SAT, combine pass, optional
// manufactured source) for every node of a slab in ONE pass over HBM, with
// the Bogacki-Shampine stage algebra of time_integration.hpp:277-286 fused
// into its prologue (stage input y + a*k formed on the fly at every stencil
// point) and epilogue (ynew in stage 2, error partials in adaptive mode).
//
// Work decomposition:
//   * a CTA of BX = 128 threads owns BX consecutive columns, i.e. BX-2
//     finished columns plus the left/right halo column (overlapped tiles:
//     every thread does identical product work, the two edge threads skip
//     the combine, so no warp is ever late at the per-row barrier);
//   * the CTA marches down a strip of rows; each thread loads the raw
//     inputs of the NEXT row into registers one row ahead (software
//     pipelining);
//   * the y-stencil uses a register window: the 12 y-differentiated
//     quantities of rows j-1 and j+1 (three named sets whose roles rotate
//     with the 3x-unrolled march, so no register moves);
//   * the x-stencil reads columns i-1, i+1 of a 3-row shared-memory ring
//     that holds only the node's stage inputs and two derived scalars (four
//     16-byte double2 pairs); the neighbours' products are re-formed from
//     them with the identical operations, which costs less than moving them
//     (the kernel is bound by the shared-memory pipe, ncu r1c);
//   * bounded (wall) directions use the same arithmetic form with clamped
//     neighbours and the closure coefficient 1/dx (see sbp_d), plus the SAT
//     face term; periodic x wraps by index, periodic y wraps or reads ghost
//     rows written by the slab halo exchange.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "sgn_device.cuh"

namespace hsgn_dev {

#ifndef HSGN_BX
#define HSGN_BX 128
#endif
constexpr int BX = HSGN_BX;  // threads per CTA == columns touched per tile
constexpr int WX = BX - 2;  // finished columns per tile
#ifndef HSGN_MIN_BLOCKS
#define HSGN_MIN_BLOCKS 0  // 0: per-stage choice in min_blocks()
#endif

template <int MODE>
__host__ __device__ constexpr int npairs() { return MODE == MODE_S2 ? NPAIRS_S2 : NPAIRS; }
#ifndef HSGN_RCP_NOBRANCH
#define HSGN_RCP_NOBRANCH 1  // rcp_or_nan (sgn_device.cuh) instead of __drcp_rn
#endif
#ifndef HSGN_S3_WARPS
#define HSGN_S3_WARPS 20  // resident warps per SM asked of the fixed-step stage-3 kernel
#endif
template <int MODE>
__host__ __device__ constexpr int min_blocks() {
    // measured (r1): S2 (largest ring, 16 raw inputs) is best at 3 CTAs/SM;
    // the other stages fit 96 registers without spills and run best at 5
    // (expressed as resident warps per SM: 12 for S2, 20 for the others)
    return HSGN_MIN_BLOCKS > 0 ? HSGN_MIN_BLOCKS
                               : (MODE == MODE_S2 ? 12 : MODE == MODE_S3A ? 16 : MODE == MODE_S3 ? HSGN_S3_WARPS : 20) /
                                     (BX / 32);
}

// Per-field device pointers (kernel parameters live in the constant bank, so
// every global address is one IMAD.WIDE of the 32-bit node offset).
struct KPtrs {
    const double* y[5];
    const double* k[5];
    const double* kc[5];
    const double* b;
    double* out[5];
    double* part[5];
    const double* yold[5];
    double* out2[5];  // S31: k2 of the next step
};

struct Raw {  // raw stage-input data at one node
    double y[5];
    double k[5];
    double kc[5];  // S2 only: k1 (for the fused ynew)
    double b;
};

struct YQ {  // y-differentiated quantities of one row at this column (rhs.hpp:127-137 + b)
    double h, u, v, w, e, hhb, v2, hv, huv, e2h, hvw, b;
};

// Per-stage kernels: memory row of logical row jr (-1 <= jr <= ny) of the
// slab counted from the ghost row -1 (their KPtrs bases point at row -1, so
// offsets stay non-negative 32-bit values): wrap (periodic, whole grid),
// clamp (wall) or the nearest ghost row (slab edge).
__device__ __forceinline__ int map_row(const StageArgs& A, int jr) {
    if (jr < 0) return A.y_lo == YE_WRAP ? A.ny : (A.y_lo == YE_CLAMP ? 1 : 0);
    if (jr >= A.ny) return A.y_hi == YE_WRAP ? 1 : (A.y_hi == YE_CLAMP ? A.ny : A.ny + 1);
    return jr + 1;
}

template <int MODE>
__device__ __forceinline__ void load_raw(const KPtrs& P, unsigned off, Raw& r) {
#pragma unroll
    for (int f = 0; f < 5; ++f) r.y[f] = __ldg(P.y[f] + off);
    if (MODE == MODE_S1 || MODE == MODE_S2) {
#pragma unroll
        for (int f = 0; f < 5; ++f) r.k[f] = __ldg(P.k[f] + off);
    }
    if (MODE == MODE_S2) {
#pragma unroll
        for (int f = 0; f < 5; ++f) r.kc[f] = __ldg(P.kc[f] + off);
    }
    r.b = __ldg(P.b + off);
}

// Pointwise products of rhs.hpp:99-109 at one node from the stage input q
// (h, u, v, w, eta) and b: stores the ring pairs of the node (S already
// offset by ring row and column), fills the y-quantities; returns h > 0.
template <bool STORE_RH = true>
__device__ __forceinline__ bool products_q(const double q[5], double b, double2* S, YQ& Y, double* rh_out) {
    const double h = q[0], u = q[1], v = q[2], w = q[3], e = q[4];
    const bool ok = h > 0.0;
    const double rh = HSGN_RCP_NOBRANCH ? rcp_or_nan(h) : __drcp_rn(h);
    bool slow = false;
    double r = div_fast(e, h, rh, slow);  // eta/h computed once (rhs.hpp:86-88)
    if (slow) r = e / h;
    const double hpb = dadd(h, b);
    const double hv = dmul(h, v);
    S[P_HU * BX] = make_double2(h, u);
    S[P_VW * BX] = make_double2(v, w);
    S[P_EB * BX] = make_double2(e, b);
    S[P_RHB * BX] = make_double2(r, hpb);
    if (STORE_RH) S[P_RH * BX] = make_double2(rh, 0.0);
    if (rh_out) *rh_out = rh;
    Y.h = h;
    Y.u = u;
    Y.v = v;
    Y.w = w;
    Y.e = e;
    Y.b = b;
    Y.hhb = dmul(h, hpb);
    Y.v2 = dmul(v, v);
    Y.hv = hv;
    Y.huv = dmul(dmul(h, u), v);  // (h*u)*v
    Y.e2h = dmul(e, r);
    Y.hvw = dmul(hv, w);
    return ok;
}

// The same from raw stage data: q = y + a*k (state_add1,
// time_integration.hpp:61-75) for S1/S2, q = y otherwise; S2 also stores
// ((y + c1 k1) + c2 k2), the k3-free part of ynew (state_add3).
template <int MODE, bool STORE_RH = true>
__device__ __forceinline__ bool products(const StageArgs& A, const Raw& raw, double2* S, YQ& Y, double* rh_out = nullptr) {
    double q[5];
#pragma unroll
    for (int f = 0; f < 5; ++f)
        q[f] = (MODE == MODE_S1 || MODE == MODE_S2) ? dadd(raw.y[f], dmul(A.a, raw.k[f])) : raw.y[f];
    const bool ok = products_q<STORE_RH>(q, raw.b, S, Y, rh_out);
    if (MODE == MODE_S2) {
        double yp[5];
#pragma unroll
        for (int f = 0; f < 5; ++f) yp[f] = dadd(dadd(raw.y[f], dmul(A.c1, raw.kc[f])), dmul(A.c2, raw.k[f]));
        S[P_YP01 * BX] = make_double2(yp[0], yp[1]);
        S[P_YP23 * BX] = make_double2(yp[2], yp[3]);
        S[P_YP4 * BX] = make_double2(yp[4], 0.0);
    }
    return ok;
}

// Manufactured source terms S(t, x, y) (scenarios.hpp:179-217 forcing; the
// closed form restated in DESIGN.md section 5 and oracle/hsgn_oracle.c).
__device__ __noinline__ void mms_source(double t, double x, double y, double g, double* s) {
    const double tp = 2.0 * 3.14159265358979323846, fp = 4.0 * 3.14159265358979323846;
    double s1x, c1x, s1y, c1y, s2x, c2x, s2y, c2y, st, ct;
    sincos(tp * x, &s1x, &c1x);
    sincos(tp * y, &s1y, &c1y);
    sincos(fp * x, &s2x, &c2x);
    sincos(fp * y, &s2y, &c2y);
    sincos(tp * t, &st, &ct);
    const double bx = -(2.0 / 25.0) * tp * s1x * c1y - (1.0 / 25.0) * fp * s2x * c2y;
    const double by = -(2.0 / 25.0) * tp * c1x * s1y - (1.0 / 25.0) * fp * c2x * s2y;
    const double bxx = -(2.0 / 25.0) * tp * tp * c1x * c1y - (1.0 / 25.0) * fp * fp * c2x * c2y;
    const double bxy = (2.0 / 25.0) * tp * tp * s1x * s1y + (1.0 / 25.0) * fp * fp * s2x * s2y;
    const double bv = (2.0 / 25.0) * c1x * c1y + (1.0 / 25.0) * c2x * c2y;
    const double h = 2.0 + 0.5 * s1x * s1y * ct - bv;
    const double hx = 0.5 * tp * c1x * s1y * ct - bx;
    const double hy = 0.5 * tp * s1x * c1y * ct - by;
    const double ht = -0.5 * tp * s1x * s1y * st;
    const double A = 0.3;
    const double u = A * s1x * st, ux = A * tp * c1x * st, uxx = -A * tp * tp * s1x * st;
    const double v = A * s1y * st, vy = A * tp * c1y * st, vyy = -A * tp * tp * s1y * st;
    const double ut = A * tp * s1x * ct, uxt = A * tp * tp * c1x * ct;
    const double vt = A * tp * s1y * ct, vyt = A * tp * tp * c1y * ct;
    const double D = ux + vy, Dt = uxt + vyt;
    const double Gx = ux * bx + u * bxx + v * bxy;
    const double Gy = u * bxy + vy * by + v * bxx;
    const double Gt = ut * bx + vt * by;
    const double wx = -hx * D - h * uxx + 1.5 * Gx;
    const double wy = -hy * D - h * vyy + 1.5 * Gy;
    const double wt = -ht * D - h * Dt + 1.5 * Gt;
    const double sh = ht + (hx * u + h * ux) + (hy * v + h * vy);
    s[0] = sh;
    s[1] = ut + u * ux + g * (hx + bx);
    s[2] = vt + v * vy + g * (hy + by);
    s[3] = wt + u * wx + v * wy;
    s[4] = sh;
}

// Adaptive-mode epilogues, kept out of line so they do not raise the register
// pressure of the fixed-step kernels.  (Scalars and base pointers are passed
// by value: taking the address of the kernel-parameter structs would copy
// them to local memory.)
// S2: ((d1 k1 + d2 k2) + d3 k3) (time_integration.hpp:128-129, first 3 terms)
__device__ __noinline__ void s2_error_partial(const double* kc, const double* k, double* part, long long fs,
                                              unsigned off, double d1, double d2, double d3, double o0, double o1,
                                              double o2, double o3, double o4) {
    const double o[5] = {o0, o1, o2, o3, o4};
#pragma unroll
    for (int f = 0; f < 5; ++f) {
        const double k1v = __ldg(kc + f * fs + off);
        const double k2v = __ldg(k + f * fs + off);
        part[f * fs + off] = dadd(dadd(dmul(d1, k1v), dmul(d2, k2v)), dmul(d3, o[f]));
    }
}
__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ------------------------------------------------------------ TMA staging
// Bulk-async (TMA) prefetch of the raw stage inputs into a 3-slot shared
// ring, two rows ahead of use.  One elected thread issues, per row and input
// field, 1-3 cp.async.bulk copies (the tile's columns i0-2 .. i0+127 with the
// periodic wrap split off) completing on the slot's mbarrier; all threads
// wait on the mbarrier phase before reading their column.  Requires nx even
// (16-byte aligned pieces); the host falls back to register prefetch
// otherwise.
constexpr int RW = BX + 2;  // raw row width: logical columns i0-2 .. i0+127
constexpr int RSLOTS = 3;

template <int MODE>
__host__ __device__ constexpr int nraw() { return MODE == MODE_S2 ? 16 : (MODE == MODE_S1 ? 11 : 6); }

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_copy(double* dst, const double* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Issue the raw inputs of logical row jr for the tile starting at column i0
// into ring slot `slot` (layout [field][RW]).  Called by one thread.
template <int MODE>
__device__ __forceinline__ void tma_issue_row(const StageArgs& A, const KPtrs& P, int jr, int i0, double* slot,
                                              unsigned long long* bar) {
    const int nx = A.nx;
    const long long row = (long long)map_row(A, jr) * nx;
    int lo = i0 - 2, hi = i0 + BX;  // logical columns [lo, hi)
    // pieces (smem offset, global column, length), all even
    int po[3], pg[3], pl[3], np = 0;
    if (A.x_bounded) {
        const int a = lo < 0 ? 0 : lo, b = hi > nx ? nx : hi;
        po[np] = a - lo; pg[np] = a; pl[np] = b - a; ++np;
    } else {
        if (hi > nx + 2) hi = nx + 2;  // beyond column nx only idle lanes
        if (lo < 0) { po[np] = 0; pg[np] = nx + lo; pl[np] = -lo; ++np; }
        const int a = lo < 0 ? 0 : lo, b = hi > nx ? nx : hi;
        po[np] = a - lo; pg[np] = a; pl[np] = b - a; ++np;
        if (hi > nx) { po[np] = nx - lo; pg[np] = 0; pl[np] = hi - nx; ++np; }
    }
    int cols = 0;
    for (int k = 0; k < np; ++k) cols += pl[k];
    mbar_expect_tx(bar, (unsigned)(cols * 8 * nraw<MODE>()));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of the slot
#pragma unroll
    for (int f = 0; f < nraw<MODE>(); ++f) {
        const double* base = f < 5 ? P.y[f] : (f == nraw<MODE>() - 1 ? P.b : (f < 10 ? P.k[f - 5] : P.kc[f - 10]));
        for (int k = 0; k < np; ++k)
            tma_copy(slot + f * RW + po[k], base + row + pg[k], (unsigned)(pl[k] * 8), bar);
    }
}

// Read this thread's column of a raw slot into the Raw struct.
template <int MODE>
__device__ __forceinline__ void raw_from_smem(const double* slot, int tid, Raw& r) {
    const double* s = slot + tid + 1;
#pragma unroll
    for (int f = 0; f < 5; ++f) r.y[f] = s[f * RW];
    if (MODE == MODE_S1 || MODE == MODE_S2) {
#pragma unroll
        for (int f = 0; f < 5; ++f) r.k[f] = s[(5 + f) * RW];
    }
    if (MODE == MODE_S2) {
#pragma unroll
        for (int f = 0; f < 5; ++f) r.kc[f] = s[(10 + f) * RW];
    }
    r.b = s[(nraw<MODE>() - 1) * RW];
}

// Per-thread constants and accumulators of one CTA's march.
struct Thr {
    int tid, i, j1;
    bool finish, xl, xr;
    unsigned col;       // memory column this thread loads (wrapped / clamped)
    double cx;          // x-stencil coefficient of this column
    int sl, sr;         // ring columns of aL / aR
    int jc0, jc1;       // rows that use the y closure coefficient (clamped walls)
    unsigned long long bad, my_min;
    double my_err;
    // L2 prefetch (thread f < nraw owns raw field f): field base, tile span
    const double* pf_base;
    int pf_col, pf_bytes;
};

// Distance (rows) of the bulk L2 prefetch ahead of the register loads.
#ifndef HSGN_EARLY_PF  // stages with <= 6 raw inputs issue the next-row loads before products
#define HSGN_EARLY_PF 0
#endif
#ifndef HSGN_L2_PF
#define HSGN_L2_PF 0
#endif

// One cp.async.bulk.prefetch.L2 per raw field and row: the tile's row segment
// is pulled into L2 HSGN_L2_PF rows before the register loads touch it, so
// those loads see L2 instead of DRAM latency.  No registers or shared memory.
template <int MODE>
__device__ __forceinline__ void l2_prefetch_row(const StageArgs& A, const Thr& T, int jr) {
    if (T.pf_bytes > 0) {
        const double* p = T.pf_base + (long long)map_row(A, jr) * A.nx + T.pf_col;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(T.pf_bytes) : "memory");
    }
}

// x-quantities of a neighbour column re-formed from its ring pairs, with the
// operations of products() / rhs.hpp:99-109 (bit-identical).
struct XQ {
    double h, u, v, w, e, b, hhb, u2, hu, huv, e2h, huw;
};
__device__ __forceinline__ void neighbour_x(const double2* S, XQ& X) {
    const double2 p0 = S[P_HU * BX], p1 = S[P_VW * BX], p2 = S[P_EB * BX], p3 = S[P_RHB * BX];
    X.h = p0.x;
    X.u = p0.y;
    X.v = p1.x;
    X.w = p1.y;
    X.e = p2.x;
    X.b = p2.y;
    X.hhb = dmul(X.h, p3.y);
    X.u2 = dmul(X.u, X.u);
    X.hu = dmul(X.h, X.u);
    X.huv = dmul(X.hu, X.v);
    X.e2h = dmul(X.e, p3.x);
    X.huw = dmul(X.hu, X.w);
}

#ifndef HSGN_YWIN_SMEM
#define HSGN_YWIN_SMEM 1
#endif
#ifndef HSGN_STAGE_SPLITBAR
#define HSGN_STAGE_SPLITBAR 1
#endif
// Split-phase row barrier of the stage-3 kernels (measured: S3 1.235 ->
// 1.219 ms; S1 1.447 -> 1.478, so S1 / RHS keep __syncthreads), as in S12: step j
// arrives on an mbarrier after finishing row j and the next step waits for
// that phase only after forming its next row's products, so a warp that is
// ahead does that work instead of idling at the barrier.  (A 4-slot ring
// with the arrive right after the products -- a whole step of slack --
// measured far slower: 40 KB rings squeeze L1.)
template <int MODE, bool TMA>
__host__ __device__ constexpr bool split_bar() {
    return HSGN_STAGE_SPLITBAR && !TMA && HSGN_YWIN_SMEM && (MODE == MODE_S3 || MODE == MODE_S3A);
}
template <int MODE, bool TMA>
__host__ __device__ constexpr int ring_slots() { return 3; }

// y-quantities of a row re-formed from its own-column ring pairs (same
// operations as products(), so bit-identical to the carried values).
__device__ __forceinline__ void neighbour_y(const double2* S, YQ& Y) {
    const double2 p0 = S[P_HU * BX], p1 = S[P_VW * BX], p2 = S[P_EB * BX], p3 = S[P_RHB * BX];
    Y.h = p0.x;
    Y.u = p0.y;
    Y.v = p1.x;
    Y.w = p1.y;
    Y.e = p2.x;
    Y.b = p2.y;
    Y.hhb = dmul(Y.h, p3.y);
    Y.v2 = dmul(Y.v, Y.v);
    Y.hv = dmul(Y.h, Y.v);
    Y.huv = dmul(dmul(Y.h, Y.u), Y.v);
    Y.e2h = dmul(Y.e, p3.x);
    Y.hvw = dmul(Y.hv, Y.w);
}

// The combine pass (rhs.hpp:147-213, wall SAT sbp.hpp:272-284, source
// rhs.hpp:212-213) at one node of row j.  S: ring slot of row j (centre at
// S + tid, x-neighbours at S + sl / S + sr); ypr / ynr: the y-quantities of
// rows j-1 / j+1 at this column.  All stage kernels share it.
// SW / SRC: the kernel may see rhs_shallow_water / a source term (the fused
// fixed-step kernels never do: the host launches them only without either).
template <int KIND, bool SW = true, bool SRC = true>
__device__ __forceinline__ void tendency(const StageArgs& A, const double2* S, int tid, int sl, int sr, double cx,
                                         double cy, bool xl, bool xr, int i, int j, const YQ& ypr, const YQ& ynr,
                                         double rh, double o[5]) {
    const double2* Sc = S + tid;  // row j, own column
    // centre values of row j (products re-formed as in rhs.hpp:99-109)
    const double2 c0 = Sc[P_HU * BX], c1 = Sc[P_VW * BX], c2 = Sc[P_EB * BX], c3 = Sc[P_RHB * BX];
    const double h = c0.x, u = c0.y, v = c1.x, w = c1.y, b = c2.y, r = c3.x, hpb = c3.y;
    const double hu = dmul(h, u), u2 = dmul(u, u), hv = dmul(h, v), v2 = dmul(v, v);
    // x-neighbours i-1, i+1
    XQ L, R;
    neighbour_x(S + sl, L);
    neighbour_x(S + sr, R);
#define DX(f) const double d##f##_x = sbp_d<KIND>(cx, L.f, R.f)
#define DY(f) const double d##f##_y = sbp_d<KIND>(cy, ypr.f, ynr.f)
    DX(h); DX(u); DX(v); DX(w); DX(e); DX(b); DX(hhb); DX(u2); DX(hu); DX(huv); DX(e2h); DX(huw);
    DY(h); DY(u); DY(v); DY(w); DY(e); DY(b); DY(hhb); DY(v2); DY(hv); DY(huv); DY(e2h); DY(hvw);
#undef DX
#undef DY
    const double g = A.g;
    // KIND 2: every tendency sum is linear in the (undivided) differences, so
    // the stencil coefficient is applied once per tendency (exact: power of 2)
    auto sc = [&](double x) { return KIND == 2 ? dmul(A.cpx, x) : x; };
    // s + 0.5*G as one rounding: 0.5*G is exact, so fma(0.5, G, s) == RN(s + RN(0.5 G))
    auto add_half = [](double s, double G) { return __fma_rn(0.5, G, s); };
    {  // continuity (rhs.hpp:156-157) + wall SAT (sbp.hpp:272-284)
        const double s = sc(dadd(dadd(dadd(dmul(u, dh_x), dmul(h, du_x)), dmul(v, dh_y)), dmul(h, dv_y)));
        double ht = -s;
        // KIND 2 implies no walls (host-checked); only the fused kernels
        // compile the test out (the per-stage kernels measured slower without it)
        if ((SRC || KIND != 2) && A.walls) {
            double sat = 0.0;
            if (xl) sat = dsub(sat, dmul(A.tdx, hu));
            if (xr) sat = dadd(sat, dmul(A.tdx, hu));
            if (j == 0 && A.sat_y_lo) sat = dsub(sat, dmul(A.tdy, hv));
            if (j == A.ny - 1 && A.sat_y_hi) sat = dadd(sat, dmul(A.tdy, hv));
            ht = dadd(ht, sat);
        }
        o[0] = ht;
    }
    const double ghb = dmul(g, hpb);
    const double ls_rr = dmul(A.lam_sixth, dmul(r, r));
    const double lt_r = dmul(A.lam_third, r);
    const double omr = dsub(1.0, r);
    const double lh_omr = dmul(A.lam_half, omr);
    const double uv = dmul(u, v);
    double nu, nv, nw;  // division numerators (before the common factor in KIND 2)
    {  // x-momentum (rhs.hpp:167-175), 0.5 factored out of the two split groups
        double s = dsub(dmul(g, dhhb_x), dmul(ghb, dh_x));
        s = add_half(s, dsub(dadd(dsub(dmul(h, du2_x), dmul(u2, dh_x)), dmul(u, dhu_x)), dmul(hu, du_x)));
        s = add_half(s, dsub(dadd(dsub(dhuv_y, dmul(uv, dh_y)), dmul(hv, du_y)), dmul(hu, dv_y)));
        s = dadd(s, dadd(dsub(dsub(dadd(dmul(ls_rr, dh_x), dmul(A.lam_third, de_x)), dmul(lt_r, de_x)),
                              dmul(A.lam_sixth, de2h_x)),
                         dmul(lh_omr, db_x)));
        nu = -s;
    }
    {  // y-momentum (rhs.hpp:180-188)
        double s = dsub(dmul(g, dhhb_y), dmul(ghb, dh_y));
        s = add_half(s, dsub(dadd(dsub(dmul(h, dv2_y), dmul(v2, dh_y)), dmul(v, dhv_y)), dmul(hv, dv_y)));
        s = add_half(s, dsub(dadd(dsub(dhuv_x, dmul(uv, dh_x)), dmul(hu, dv_x)), dmul(hv, du_x)));
        s = dadd(s, dadd(dsub(dsub(dadd(dmul(ls_rr, dh_y), dmul(A.lam_third, de_y)), dmul(lt_r, de_y)),
                              dmul(A.lam_sixth, de2h_y)),
                         dmul(lh_omr, db_y)));
        nv = -s;
    }
    {  // vertical velocity (rhs.hpp:196-200)
        const double hw = dmul(h, w);
        double s = dmul(0.5, dsub(dsub(dadd(dhuw_x, dmul(hu, dw_x)), dmul(dmul(u, w), dh_x)), dmul(hw, du_x)));
        s = add_half(s, dsub(dsub(dadd(dhvw_y, dmul(hv, dw_y)), dmul(dmul(v, w), dh_y)), dmul(hw, dv_y)));
        nw = dsub(dmul(A.lambda, omr), sc(s));
    }
    {  // the three "/h" (rhs.hpp:175,188,200), one range test per node
        bool slow = false;
        double qu = div_fast(nu, h, rh, slow), qv = div_fast(nv, h, rh, slow), qw = div_fast(nw, h, rh, slow);
        if (slow) {
            qu = nu / h;
            qv = nv / h;
            qw = nw / h;
        }
        o[1] = sc(qu);  // RN(c s / h) == c RN(s / h) for c a power of two
        o[2] = sc(qv);
        o[3] = qw;
    }
    {  // auxiliary depth (rhs.hpp:206-208)
        const double s =
            dadd(dadd(dadd(dmul(u, de_x), dmul(v, de_y)), dmul(dmul(1.5, u), db_x)), dmul(dmul(1.5, v), db_y));
        o[4] = dsub(w, sc(s));
    }
    if (SW && A.shallow) {  // rhs_shallow_water zeroes the decoupled tendencies
        o[3] = 0.0;
        o[4] = 0.0;
    }
    if (SRC && A.source) {  // add_manufactured_sources: after assembly (rhs.hpp:212-213)
        const double xg = dadd(A.x_min, dmul((double)i, A.dx));
        const double yg = dadd(A.y_min, dmul((double)(A.j_global0 + j), A.dy));
        double s5[5];
        mms_source(A.t, xg, yg, A.g, s5);
#pragma unroll
        for (int f = 0; f < 5; ++f) o[f] = dadd(o[f], s5[f]);
    }
}

// One row of the march: form row jn = j+1 (ring slot SN, register set yn),
// then finish row j (ring slot SC; row j-1 is register set yp).
template <int MODE, int KIND, bool TMA, int SC>
__device__ __forceinline__ void march_row(const StageArgs& A, const KPtrs& P, Thr& T, double2* ring, double* rawring,
                                          unsigned long long* bars, int j0, int j, const YQ& yp, YQ& yn, Raw& raw,
                                          Raw& raw_next, unsigned long long* sbar) {
    constexpr int NP = npairs<MODE>();
    constexpr int NS = ring_slots<MODE, TMA>();
    constexpr bool SPLIT = split_bar<MODE, TMA>();
    constexpr int SN = (SC + 1) % NS;
    const int jn = j + 1;
    const unsigned nx = (unsigned)A.nx;
    // register prefetch of raw(jn+1), issued after products(jn) so the load is
    // in flight during the finish of row j.  (Issuing it before products(jn)
    // needs two raw register sets and a 6x-unrolled march: measured slower in
    // round 1 -- spills in S1/S2, I-cache in S3 -- so EARLY stays off; raw and
    // raw_next may then alias.)
    constexpr bool EARLY = HSGN_EARLY_PF && nraw<MODE>() <= 6;
    if (!TMA && EARLY && jn < T.j1) load_raw<MODE>(P, (unsigned)map_row(A, jn + 1) * nx + T.col, raw_next);
    if (!TMA && HSGN_L2_PF > 1 && jn + HSGN_L2_PF <= T.j1) l2_prefetch_row<MODE>(A, T, jn + HSGN_L2_PF);
    if (TMA) {  // raw row jn lives in raw slot (SC+2)%3; row j+3 goes into slot (SC+1)%3
        constexpr int RS = (SC + 2) % 3, RI = (SC + 1) % 3;
        mbar_wait(&bars[RS], (unsigned)(((jn - j0 + 1) / 3) & 1));
        raw_from_smem<MODE>(rawring + RS * (nraw<MODE>() * RW), T.tid, raw);
        if (T.tid == 0 && j + 3 <= T.j1)
            tma_issue_row<MODE>(A, P, j + 3, (int)blockIdx.x * WX, rawring + RI * (nraw<MODE>() * RW), &bars[RI]);
    }
    {  // products of row jn (for D_y of row j, and D_x of row jn one step later)
        const bool ok = products<MODE>(A, raw, ring + SN * (NP * BX) + T.tid, yn);
        if (T.finish && jn < T.j1 && !ok) ++T.bad;
    }
    if (!TMA && !EARLY && jn < T.j1) load_raw<MODE>(P, (unsigned)map_row(A, jn + 1) * nx + T.col, raw);
    if (!TMA && EARLY) raw = raw_next;  // (register moves: the 3x unroll cannot alternate two sets)
    // One barrier per row: row j's ring entries (written one step ago) become
    // visible, and this step's writes to slot SN are ordered after the last
    // reads of that slot (finish of row j-2, before the previous barrier).
    const int t = j - j0 + 1;  // step index (the prologue is step 0)
    if (SPLIT) {
        mbar_wait(&sbar[(t - 1) & 1], (unsigned)((t - 1) >> 1) & 1u);
    } else {
        __syncthreads();
    }
    if (!T.finish) {
        if (SPLIT) mbar_arrive(&sbar[t & 1]);
        return;
    }

    const double2* S = ring + SC * (NP * BX);
    const double2* Sc = S + T.tid;  // row j, own column
    const double cy = (j == T.jc0 || j == T.jc1) ? A.c1y : A.cpy;
    // Row j-1: S1/S3/RHS re-form it from its ring entry (slot SP, own
    // column), which frees the carried window's registers (96 instead of
    // ~160) for 6 DMUL + 4 LDS.128 per node; S2 keeps the register window
    // (measured faster for S2, r1: 2.05 vs 2.95 ms).
    constexpr bool ywin_smem = HSGN_YWIN_SMEM && MODE != MODE_S2;
    YQ yprev;
    if (ywin_smem) neighbour_y(ring + ((SC + NS - 1) % NS) * (NP * BX) + T.tid, yprev);
    const YQ& ypr = ywin_smem ? yprev : yp;
    const unsigned off = (unsigned)(j + 1) * nx + T.col;  // bases point at row -1
    // S3A: the error-norm inputs of this node are requested before the
    // tendency so their latency hides behind it
    double e_part[5], e_yold[5];
    if (MODE == MODE_S3A) {
#pragma unroll
        for (int f = 0; f < 5; ++f) {
            e_part[f] = P.part[f][off];
            e_yold[f] = __ldg(P.yold[f] + off);
        }
    }
    double o[5];
    tendency<KIND>(A, S, T.tid, T.sl, T.sr, T.cx, cy, T.xl, T.xr, T.i, j, ypr, yn, Sc[P_RH * BX].x, o);
    // ---- epilogue
    if (MODE == MODE_S2) {
        const double2 y01 = Sc[P_YP01 * BX], y23 = Sc[P_YP23 * BX], y4 = Sc[P_YP4 * BX];
        const double ypart[5] = {y01.x, y01.y, y23.x, y23.y, y4.x};
#pragma unroll
        for (int f = 0; f < 5; ++f) {  // state_add3: ((y + c1 k1) + c2 k2) + c3 k3
            const double yn_f = dadd(ypart[f], dmul(A.c3, o[f]));
            P.out[f][off] = yn_f;
            if (f == 0) {
                const unsigned long long bits = (unsigned long long)__double_as_longlong(yn_f);
                T.my_min = bits < T.my_min ? bits : T.my_min;
            }
        }
        if (A.adaptive)
            s2_error_partial(A.kc - A.nx, A.k - A.nx, A.part - A.nx, A.fs, off, A.d1, A.d2, A.d3, o[0], o[1], o[2],
                             o[3], o[4]);
    } else {
#pragma unroll
        for (int f = 0; f < 5; ++f) P.out[f][off] = o[f];
        if (MODE == MODE_S3A) {  // sum_f (e_f / scale_f)^2 (time_integration.hpp:127-136)
            const double2 c0 = Sc[P_HU * BX], c1 = Sc[P_VW * BX], c2 = Sc[P_EB * BX];
            const double yn5[5] = {c0.x, c0.y, c1.x, c1.y, c2.x};  // ynew = this stage's input
            double acc = 0.0;
#pragma unroll
            for (int f = 0; f < 5; ++f) {
                const double e = dmul(A.dt, dadd(e_part[f], dmul(A.d4, o[f])));
                const double ay = fabs(e_yold[f]), an = fabs(yn5[f]);
                const double scale = dadd(A.atol, dmul(A.rtol, ay < an ? an : ay));
                const double rq = e / scale;
                acc = dadd(acc, dmul(rq, rq));
            }
            T.my_err = dadd(T.my_err, acc);
        }
    }
    if (SPLIT) mbar_arrive(&sbar[t & 1]);  // row j finished: its slot may be reused after the next wait
}

template <int MODE, int KIND, bool TMA>
__global__ void __launch_bounds__(BX, min_blocks<MODE>()) sgn_stage_kernel(const StageArgs A, const KPtrs P) {
    constexpr int NP = npairs<MODE>();
    extern __shared__ __align__(16) double2 ring[];  // 3 x NP x BX pairs
    __shared__ unsigned long long s_min[BX / 32];
    __shared__ double s_err[BX / 32];
    __shared__ int s_skip;

    const int tid = threadIdx.x;
    // ---- graph-level failure protocol: skip all work
    // once an earlier stage of the captured step sequence failed.
    if (A.halt) {
        if (tid == 0) {
            int skip = *A.halt;
            if (!skip && A.chk_bad && *A.chk_bad) skip = 1;
            if (!skip && A.chk_bad2 && *A.chk_bad2) skip = 1;
            if (!skip && A.chk_minh) {
                const unsigned long long mb = *A.chk_minh;
                if (mb != ~0ull && __longlong_as_double((long long)mb) <= A.h_floor) skip = 1;
            }
            if (skip) *A.halt = 1;
            s_skip = skip;
        }
        __syncthreads();
        if (s_skip) return;
    }

    const int nx = A.nx, ny = A.ny;
    Thr T;
    T.tid = tid;
    const int i = (int)blockIdx.x * WX - 1 + tid;  // logical column (may be -1 or >= nx)
    T.i = i;
    T.finish = tid >= 1 && tid <= WX && i < nx;
    // memory column: periodic wrap of the two halo columns, clamp otherwise
    int col = i;
    if (i < 0) col = A.x_bounded ? 0 : nx - 1;
    if (i >= nx) col = (A.x_bounded || i > nx) ? nx - 1 : 0;
    T.col = (unsigned)col;
    T.xl = A.x_bounded && i == 0;
    T.xr = A.x_bounded && i == nx - 1;
    T.cx = (T.xl || T.xr) ? A.c1x : A.cpx;
    T.sl = T.xl ? tid : tid - 1;
    T.sr = T.xr ? tid : tid + 1;
    const int j0 = A.band0 + blockIdx.y * A.rows_per_block;
    T.j1 = min(A.band1 > 0 ? A.band1 : ny, j0 + A.rows_per_block);
    T.jc0 = A.y_lo == YE_CLAMP ? 0 : -2;
    T.jc1 = A.y_hi == YE_CLAMP ? ny - 1 : -2;
    T.bad = 0;
    T.my_min = ~0ull;
    T.my_err = 0.0;
    const unsigned unx = (unsigned)nx;
    T.pf_base = nullptr;
    T.pf_bytes = 0;
    T.pf_col = 0;
    if (!TMA && HSGN_L2_PF > 1 && (nx % 2) == 0 && tid < nraw<MODE>()) {
#pragma unroll
        for (int f = 0; f < nraw<MODE>(); ++f)
            if (tid == f)
                T.pf_base = f < 5 ? P.y[f] : (f == nraw<MODE>() - 1 ? P.b : (f < 10 ? P.k[f - 5] : P.kc[f - 10]));
        const int a = max((int)blockIdx.x * WX - 2, 0), e = min((int)blockIdx.x * WX + BX, nx);
        T.pf_col = a;
        T.pf_bytes = (e - a) * 8;
        for (int r = j0 + 2; r <= min(j0 + HSGN_L2_PF, T.j1); ++r) l2_prefetch_row<MODE>(A, T, r);
    }

    // ---- prologue: row j0-1 -> register set C (ring slot 2), row j0 -> set A (slot 0)
    YQ ya, yb, yc;
    Raw raw;
    double* rawring = reinterpret_cast<double*>(ring + 3 * NP * BX);  // TMA: RSLOTS x nraw x RW
    __shared__ __align__(8) unsigned long long bars[RSLOTS];
    if (TMA) {  // raw row r lives in slot (r - j0 + 1) % 3
        const int i0 = (int)blockIdx.x * WX;
        if (tid == 0) {
            for (int s = 0; s < RSLOTS; ++s) mbar_init(&bars[s], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            for (int s = 0; s < RSLOTS; ++s)
                if (j0 - 1 + s <= T.j1)
                    tma_issue_row<MODE>(A, P, j0 - 1 + s, i0, rawring + s * (nraw<MODE>() * RW), &bars[s]);
        }
        __syncthreads();
        mbar_wait(&bars[0], 0);
        raw_from_smem<MODE>(rawring, tid, raw);
    } else {
        load_raw<MODE>(P, (unsigned)map_row(A, j0 - 1) * unx + T.col, raw);
    }
    constexpr int NS = ring_slots<MODE, TMA>();
    products<MODE>(A, raw, ring + (NS - 1) * (NP * BX) + tid, yc);
    if (TMA) {
        mbar_wait(&bars[1], 0);
        raw_from_smem<MODE>(rawring + nraw<MODE>() * RW, tid, raw);
    } else {
        load_raw<MODE>(P, (unsigned)(j0 + 1) * unx + T.col, raw);
    }
    {
        const bool ok = products<MODE>(A, raw, ring + tid, ya);
        if (T.finish && !ok) ++T.bad;
    }
    if (TMA) {  // slot 0 (row j0-1) is free once every thread has read it
        __syncthreads();
        if (tid == 0 && j0 + 2 <= T.j1)
            tma_issue_row<MODE>(A, P, j0 + 2, (int)blockIdx.x * WX, rawring, &bars[0]);
    } else {
        load_raw<MODE>(P, (unsigned)map_row(A, j0 + 1) * unx + T.col, raw);
    }

    // ---- march, unrolled by 3: row j lives in ring slot (j-j0)%3 and register
    // set {a,b,c}[(j-j0)%3]; step SC reads set SC+2 (row j-1), writes SC+1.
    Raw raw2;  // next-row prefetch target when it overlaps products (EARLY)
    __shared__ __align__(8) unsigned long long sbar[2];
    if (split_bar<MODE, TMA>()) {
        if (tid == 0) {
            mbar_init(&sbar[0], BX);
            mbar_init(&sbar[1], BX);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        mbar_arrive(&sbar[0]);  // step 0: rows j0-1 and j0 written
    }
    for (int j = j0; j < T.j1; j += 3) {
        march_row<MODE, KIND, TMA, 0>(A, P, T, ring, rawring, bars, j0, j, yc, yb, raw, raw2, sbar);
        if (j + 1 >= T.j1) break;
        march_row<MODE, KIND, TMA, 1>(A, P, T, ring, rawring, bars, j0, j + 1, ya, yc, raw, raw2, sbar);
        if (j + 2 >= T.j1) break;
        march_row<MODE, KIND, TMA, 2>(A, P, T, ring, rawring, bars, j0, j + 2, yb, ya, raw, raw2, sbar);
    }

    // ---- block reductions (fixed order inside the block)
    if (T.bad) atomicAdd(A.bad, T.bad);
    const int warp = tid >> 5, lane = tid & 31;
    if (MODE == MODE_S2 && A.minh) {
        const unsigned long long m = warp_min_u64(T.my_min);
        if (lane == 0) s_min[warp] = m;
        __syncthreads();
        if (tid == 0) {
            unsigned long long mm = s_min[0];
            for (int k = 1; k < BX / 32; ++k) mm = s_min[k] < mm ? s_min[k] : mm;
            if (mm != ~0ull) atomicMin(A.minh, mm);
        }
    }
    if (MODE == MODE_S3A) {
        const double s = warp_sum(T.my_err);
        if (lane == 0) s_err[warp] = s;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int k = 0; k < BX / 32; ++k) t = dadd(t, s_err[k]);
            A.err_part[blockIdx.y * gridDim.x + blockIdx.x] = t;
        }
    }
}

// ------------------------------------------------------------ fused S3 + S1
// Stage 3 of step n and stage 1 of step n+1 in one pass (fixed step, FSAL:
// y' = ynew, k1' = k4):  k4 = f(ynew), k2' = f(ynew + a k4).  The S3 half
// runs one row and one column ahead of the S1 half inside the CTA, so the
// stage-1 input at every stencil point comes from registers/shared memory
// instead of a second HBM pass: per step the fixed-step pipeline moves
// 168 (S2) + 128 (S31) = 296 B/node instead of 384.  Arithmetic is the
// unfused S3 and S1 operation for operation (bit-identical).
//
//   * tile: BX threads, columns i0-2 .. i0+BX-3; the S3 half finishes
//     threads 1..BX-2, the S1 half threads 2..BX-3 (WX2 = BX-4 columns);
//   * rows: the S1 half finishes rows [j0, j1) of the CTA; the S3 half
//     rows j0-1 .. j1 (k4 stored for [j0, j1) only); ynew rows j0-2 .. j1+1;
//   * two 3-slot rings of 4 pairs (S3 inputs, S1 inputs; the centre 1/h of
//     each ring row is carried in registers instead), one barrier per row:
//     49 KB per CTA, 4 CTAs per SM;
//   * whole-grid contexts only (y edges WRAP or CLAMP: rows -2 and ny+1
//     exist by wrap/clamp, no ghost rows needed).
constexpr int WX2 = BX - 4;
constexpr int NPF = 4;  // ring pairs of the fused kernel (no P_RH)

// Fused kernels: the same for -GHOST <= jr < ny + GHOST, counted from row
// -GHOST (their KPtrs bases point there).
__device__ __forceinline__ int map_row2(const StageArgs& A, int jr) {
    if (jr < 0) return A.y_lo == YE_WRAP ? jr + A.ny + GHOST : (A.y_lo == YE_CLAMP ? GHOST : jr + GHOST);
    if (jr >= A.ny) return A.y_hi == YE_WRAP ? jr - A.ny + GHOST : (A.y_hi == YE_CLAMP ? A.ny - 1 + GHOST : jr + GHOST);
    return jr + GHOST;
}

struct Thr2 {
    int tid, i, j0, j1, jc0, jc1;
    bool fa, fb;  // finishes the S3 half / the S1 half (and owns the column)
    bool xl, xr;
    unsigned col;
    double cx;
    int sl, sr;
    unsigned long long bad_a, bad_b;
};

// S3 half at row r from ring-A slots (ap: row r-1, ac: row r; yn: the
// y-quantities of row r+1 as products() just formed them, identical to the
// ring re-form; rh: 1/h of row r at this column): k4 (stored when owned) and
// the S1-half input products of row r into ring-B slot bo (their
// y-quantities into yb, 1/h into *rh_b).
template <int KIND>
__device__ __forceinline__ void s31_half3(const StageArgs& A, const KPtrs& P, Thr2& T, const double2* ap,
                                          const double2* ac, const YQ& yn, double rh, double2* bo, YQ& yb,
                                          double* rh_b, int r) {
    if (!T.fa) return;
    YQ yp;
    neighbour_y(ap + T.tid, yp);
    const double cy = (r == T.jc0 || r == T.jc1) ? A.c1y : A.cpy;
    double o[5];
    tendency<KIND, false, false>(A, ac, T.tid, T.sl, T.sr, T.cx, cy, T.xl, T.xr, T.i, r, yp, yn, rh, o);
    const bool own = T.fb && r >= T.j0 && r < T.j1;
    if (own) {
        const unsigned off = (unsigned)(r + GHOST) * (unsigned)A.nx + T.col;
#pragma unroll
        for (int f = 0; f < 5; ++f) P.out[f][off] = o[f];
    }
    // next step's stage-1 input ynew + a k4 (state_add1) and its products
    const double2* Sc = ac + T.tid;
    const double2 p0 = Sc[P_HU * BX], p1 = Sc[P_VW * BX], p2 = Sc[P_EB * BX];
    Raw rb;
    rb.y[0] = p0.x;
    rb.y[1] = p0.y;
    rb.y[2] = p1.x;
    rb.y[3] = p1.y;
    rb.y[4] = p2.x;
    rb.b = p2.y;
#pragma unroll
    for (int f = 0; f < 5; ++f) rb.k[f] = o[f];
    const bool ok = products<MODE_S1, false>(A, rb, bo + T.tid, yb, rh_b);
    if (own && !ok) ++T.bad_b;
}

// S1 half at row j from ring-B slots (bp: row j-1, bc: row j; ynb: the
// y-quantities of row j+1 from the S3 half that just formed them).
template <int KIND>
__device__ __forceinline__ void s31_half1(const StageArgs& A, const KPtrs& P, const Thr2& T, const double2* bp,
                                          const double2* bc, const YQ& ynb, double rh, int j) {
    if (!T.fb) return;
    // a clamped (wall) row reads itself in place of the missing neighbour,
    // exactly the clamped stage input the unfused S1 forms there
    if (j == 0 && A.y_lo == YE_CLAMP) bp = bc;
    YQ yp, yc;
    neighbour_y(bp + T.tid, yp);
    const bool hi = j == A.ny - 1 && A.y_hi == YE_CLAMP;
    if (hi) neighbour_y(bc + T.tid, yc);
    const YQ& yn = hi ? yc : ynb;
    const double cy = (j == T.jc0 || j == T.jc1) ? A.c1y : A.cpy;
    double o[5];
    tendency<KIND, false, false>(A, bc, T.tid, T.sl, T.sr, T.cx, cy, T.xl, T.xr, T.i, j, yp, yn, rh, o);
    const unsigned off = (unsigned)(j + GHOST) * (unsigned)A.nx + T.col;
#pragma unroll
    for (int f = 0; f < 5; ++f) P.out2[f][off] = o[f];
}

#ifndef HSGN_S31_MINB
#define HSGN_S31_MINB (16 / (BX / 32))  // 16 warps per SM (49 KB of rings per 128-thread CTA)
#endif

template <int KIND>
__global__ void __launch_bounds__(BX, HSGN_S31_MINB) sgn_s31_kernel(const StageArgs A, const KPtrs P) {
    extern __shared__ __align__(16) double2 ring[];  // ring A | ring B, each 3 x NPF x BX
    __shared__ int s_skip;
    const int tid = threadIdx.x;
    if (A.halt) {  // failure protocol
        if (tid == 0) {
            int skip = *A.halt;
            if (!skip && A.chk_bad && *A.chk_bad) skip = 1;
            if (!skip && A.chk_minh) {
                const unsigned long long mb = *A.chk_minh;
                if (mb != ~0ull && __longlong_as_double((long long)mb) <= A.h_floor) skip = 1;
            }
            if (skip) *A.halt = 1;
            s_skip = skip;
        }
        __syncthreads();
        if (s_skip) return;
    }
    const int nx = A.nx, ny = A.ny;
    Thr2 T;
    T.tid = tid;
    const int i = (int)blockIdx.x * WX2 - 2 + tid;
    T.i = i;
    T.fb = tid >= 2 && tid <= BX - 3 && i >= 0 && i < nx;
    T.fa = tid >= 1 && tid <= BX - 2 && i >= -1 && i <= nx;
    int col = i;
    if (i < 0) col = A.x_bounded ? 0 : nx + i;
    if (i >= nx) col = (A.x_bounded || i > nx + 1) ? nx - 1 : i - nx;
    T.col = (unsigned)col;
    T.xl = A.x_bounded && i == 0;
    T.xr = A.x_bounded && i == nx - 1;
    T.cx = (T.xl || T.xr) ? A.c1x : A.cpx;
    T.sl = T.xl ? tid : tid - 1;
    T.sr = T.xr ? tid : tid + 1;
    T.j0 = A.band0 + blockIdx.y * A.rows_per_block;
    T.j1 = min(A.band1 > 0 ? A.band1 : ny, T.j0 + A.rows_per_block);
    T.jc0 = A.y_lo == YE_CLAMP ? 0 : INT_MIN;
    T.jc1 = A.y_hi == YE_CLAMP ? ny - 1 : INT_MIN;
    T.bad_a = 0;
    T.bad_b = 0;
    const int j0 = T.j0;
    const unsigned unx = (unsigned)nx;
    constexpr int SLOT = NPF * BX;
    // rotating slot pointers (the march is not unrolled: one copy of each
    // half keeps the kernel inside the instruction cache)
    double2* a0 = ring;             // ring A: rows j, j+1, j+2 at the top of iteration j
    double2* a1 = ring + SLOT;
    double2* a2 = ring + 2 * SLOT;
    double2* b0 = ring + 3 * SLOT;  // ring B: rows j-1, j, j+1
    double2* b1 = ring + 4 * SLOT;
    double2* b2 = ring + 5 * SLOT;
    double rha1, rha2, rhb1, rhb2;  // 1/h carried: ring A rows j+1, j+2; ring B rows j, j+1

    // ---- prologue: ynew rows j0-2 -> a1, j0-1 -> a2, j0 -> a0; S3 half of
    // row j0-1 (-> b0); row j0+1 -> a1; S3 half of row j0 (-> b1).  The
    // pointers then sit as iteration j0 expects.
    Raw raw;
    YQ ya, yb;  // y-quantities just formed for ring A / ring B (the next row of each half)
    double rh_m2, rh_m1, rh_0, rhb0;
    load_raw<MODE_S3>(P, (unsigned)map_row2(A, j0 - 2) * unx + T.col, raw);
    products<MODE_S3, false>(A, raw, a1 + tid, ya, &rh_m2);
    load_raw<MODE_S3>(P, (unsigned)map_row2(A, j0 - 1) * unx + T.col, raw);
    products<MODE_S3, false>(A, raw, a2 + tid, ya, &rh_m1);
    load_raw<MODE_S3>(P, (unsigned)map_row2(A, j0) * unx + T.col, raw);
    if (!products<MODE_S3, false>(A, raw, a0 + tid, ya, &rh_0) && T.fb) ++T.bad_a;
    load_raw<MODE_S3>(P, (unsigned)map_row2(A, j0 + 1) * unx + T.col, raw);
    __syncthreads();
    // S3 half of row j0-1 (ring B row j0-1 -> b0)
    s31_half3<KIND>(A, P, T, a1, a2, ya, rh_m1, b0, yb, &rhb0, j0 - 1);
    // row j0+1 overwrites row j0-2's slot (a1): only this thread's own column
    // of row j0-2 was read (y-window of the S3 half above)
    if (!products<MODE_S3, false>(A, raw, a1 + tid, ya, &rha1) && T.fb && j0 + 1 < T.j1) ++T.bad_a;
    load_raw<MODE_S3>(P, (unsigned)map_row2(A, j0 + 2) * unx + T.col, raw);
    // S3 half of row j0 (ring B row j0 -> b1)
    s31_half3<KIND>(A, P, T, a2, a0, ya, rh_0, b1, yb, &rhb1, j0);
    __syncthreads();  // ring A row j0-1 (a2) is overwritten next; ring B rows j0-1, j0 published

#pragma unroll 1
    for (int j = j0; j < T.j1; ++j) {
        // ynew row j+2 into the slot of row j-1 (a2), last read across
        // threads by the S3 half of row j-1 before the previous barrier
        if (!products<MODE_S3, false>(A, raw, a2 + tid, ya, &rha2) && T.fb && j + 2 < T.j1) ++T.bad_a;
        if (j + 1 < T.j1) load_raw<MODE_S3>(P, (unsigned)map_row2(A, j + 3) * unx + T.col, raw);
        __syncthreads();
        // S3 half of row j+1 -> ring B row j+1 into the slot of row j-2 (b2),
        // last read across threads by the S1 half of row j-2
        s31_half3<KIND>(A, P, T, a0, a1, ya, rha1, b2, yb, &rhb2, j + 1);
        s31_half1<KIND>(A, P, T, b0, b1, yb, rhb1, j);
        // rotate: A rows (j+1, j+2, j) -> (a0, a1, a2); B rows (j, j+1, j-1) -> (b0, b1, b2)
        double2* t = a0;
        a0 = a1;
        a1 = a2;
        a2 = t;
        t = b0;
        b0 = b1;
        b1 = b2;
        b2 = t;
        rha1 = rha2;
        rhb1 = rhb2;
    }
    if (T.bad_a) atomicAdd(A.bad, T.bad_a);
    if (T.bad_b) atomicAdd(A.bad2, T.bad_b);
}

// y-quantities of the row above / below at this column for a finish at row
// j: the ring entry of the neighbour row, or (clamped wall rows) the row's
// own entry, as the unfused kernels' clamped stage input gives.
__device__ __forceinline__ void ywin_prev(const StageArgs& A, int j, const double2* prev, const double2* cur, int tid,
                                          YQ& Y) {
    neighbour_y((j == 0 && A.y_lo == YE_CLAMP ? cur : prev) + tid, Y);
}

// ------------------------------------------------------------ fused S1 + S2
// Stages 1 and 2 of one fixed step in one pass: reads y, k1 (= f(y)) and b,
// writes ynew (+ min h): 128 B/node; stage 3 (k4 = f(ynew), 88 B/node)
// follows as its own kernel, so a step moves 216 B/node.  S2 is the
// HBM-heaviest stage (16 inputs); fusing S1 into it removes the k2 round
// trip and the re-read of y and k1.  Pipeline per iteration r:
//   P1  stage-1 input y + a1 k1 of row r -> ring A   |  barrier
//   H1  k2 at row r-1; stage-2 input y + a2 k2 -> ring B, and
//       ((y + c1 k1) + c2 k2) kept in registers for H2 of the next row
//   H2  k3 at row r-2; ynew = part + c3 k3 (stored, min h)
// Same tile / ring layout as S31 (WX2 = BX-4 columns, 2 x 3 slots x 4
// pairs, 1/h in registers: 49 KB; 3 CTAs per SM at <= 168 registers).
// Whole-grid contexts.
// measured (r1, 8192^2): 3 CTAs/SM at <= 168 registers without spills runs
// S12 in 3.16 ms; forcing 4 CTAs (128 registers) spills ~380 B/thread and
// takes 7.1 ms.  Passing ring A's next-row y-quantities in registers and
// issuing the next raw row before the barrier measured faster (3.16 vs 3.31).
#ifndef HSGN_S12_MINB
#define HSGN_S12_MINB (12 / (BX / 32))
#endif
#ifndef HSGN_S12_PASS_A
#define HSGN_S12_PASS_A 1
#endif
#ifndef HSGN_S12_SPLITBAR
#define HSGN_S12_SPLITBAR 1  // split-phase row barrier (mbarrier arrive after H2, wait after the next P1)
#endif
#ifndef HSGN_S12_EARLY_H1
#define HSGN_S12_EARLY_H1 1
#endif
#ifndef HSGN_S12_UNROLL
#define HSGN_S12_UNROLL 1  // march unroll of S12 (1: one copy of the loop body in the I-cache)
#endif
constexpr int kS12Unroll = HSGN_S12_UNROLL;
#ifndef HSGN_S12_LATE_PF
#define HSGN_S12_LATE_PF 0
#endif

// ADAPT: also store the error partial ((d1 k1 + d2 k2) + d3 k3)
// (time_integration.hpp:128-129, the S2 epilogue of the per-stage path) for
// the adaptive S3's error norm.
template <int KIND, bool ADAPT>
__global__ void __launch_bounds__(BX, HSGN_S12_MINB) sgn_s12_kernel(const StageArgs A, const KPtrs P) {
    extern __shared__ __align__(16) double2 ring[];  // ring A | ring B, each 3 x NPF x BX
    __shared__ unsigned long long s_min[BX / 32];
    __shared__ int s_skip;
    const int tid = threadIdx.x;
    if (A.halt) {  // failure protocol: the previous step's S3 counter and min h
        if (tid == 0) {
            int skip = *A.halt;
            if (!skip && A.chk_bad && *A.chk_bad) skip = 1;
            if (!skip && A.chk_minh) {
                const unsigned long long mb = *A.chk_minh;
                if (mb != ~0ull && __longlong_as_double((long long)mb) <= A.h_floor) skip = 1;
            }
            if (skip) *A.halt = 1;
            s_skip = skip;
        }
        __syncthreads();
        if (s_skip) return;
    }
    const int nx = A.nx, ny = A.ny;
    // KIND 2 (common factor) is only chosen for fully periodic grids without
    // walls (host-checked): the wall / clamp branches compile out
    constexpr bool PER = KIND == 2;
    const int i = (int)blockIdx.x * WX2 - 2 + tid;
    const bool fa = tid >= 1 && tid <= BX - 2 && i >= -1 && i <= nx;  // stage-1 finish
    const bool fb = tid >= 2 && tid <= BX - 3 && i >= 0 && i < nx;    // stage-2 finish (owned column)
    int c = i;
    if (i < 0) c = (!PER && A.x_bounded) ? 0 : nx + i;
    if (i >= nx) c = ((!PER && A.x_bounded) || i > nx + 1) ? nx - 1 : i - nx;
    const unsigned col = (unsigned)c;
    const bool xl = !PER && A.x_bounded && i == 0, xr = !PER && A.x_bounded && i == nx - 1;
    const double cx = (xl || xr) ? A.c1x : A.cpx;
    const int sl = xl ? tid : tid - 1, sr = xr ? tid : tid + 1;
    const int j0 = A.band0 + blockIdx.y * A.rows_per_block;
    const int j1 = min(A.band1 > 0 ? A.band1 : ny, j0 + A.rows_per_block);
    const int jc0 = (!PER && A.y_lo == YE_CLAMP) ? 0 : INT_MIN, jc1 = (!PER && A.y_hi == YE_CLAMP) ? ny - 1 : INT_MIN;
    const bool clamp_lo = !PER && A.y_lo == YE_CLAMP, clamp_hi = !PER && A.y_hi == YE_CLAMP;
    const unsigned unx = (unsigned)nx;
    unsigned long long bad1 = 0, bad2 = 0, my_min = ~0ull;

    constexpr int SLOT = NPF * BX;
    // at iteration r ring A holds rows (r-2, r-1, r) in (pa, pb, pc), ring B
    // rows (r-3, r-2, r-1) in (qa, qb, qc); pc and qc are written now
    double2 *pa = ring, *pb = ring + SLOT, *pc = ring + 2 * SLOT;
    double2 *qa = ring + 3 * SLOT, *qb = ring + 4 * SLOT, *qc = ring + 5 * SLOT;
    double rhap = 0.0, rhbp = 0.0;  // 1/h of ring A row r-1 / ring B row r-2
    double partp[5];                // ((y + c1 k1) + c2 k2) of row r-2
#pragma unroll
    for (int f = 0; f < 5; ++f) partp[f] = 0.0;

    // Split-phase row barrier (HSGN_S12_SPLITBAR): iteration k arrives on
    // s_bar[k & 1] after its H2 and iteration k + 1 waits for that phase only
    // after its P1.  P1(r) needs no wait of its own (it overwrites ring A row
    // r-3, last read across threads in iteration k - 2), so a warp that is
    // ahead forms the next stage-1 input while the others finish.
    // (Measured slower: a second barrier set -- arrive after P1 / wait before
    // H1, arrive after H1 / wait before H2 -- with a 4-slot ring B, 2.68 vs
    // 2.63 ms.)
    __shared__ __align__(8) unsigned long long s_bar[2];
    if (HSGN_S12_SPLITBAR) {
        if (tid == 0) {
            for (int q = 0; q < 2; ++q) mbar_init(&s_bar[q], BX);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    Raw raw;
    load_raw<MODE_S1>(P, (unsigned)map_row2(A, j0 - 2) * unx + col, raw);
    int k = 0;  // iteration index (split barrier phases)
#pragma unroll kS12Unroll
    for (int r = j0 - 2; r <= j1 + 1; ++r, ++k) {
        // ---- P1: stage-1 input of row r (raw of row r+1 loaded right after)
        YQ ya;
        double rhac;
        {
            const bool ok = products<MODE_S1, false>(A, raw, pc + tid, ya, &rhac);
            if (fb && r >= j0 && r < j1 && !ok) ++bad1;
        }
        if (!HSGN_S12_LATE_PF && r + 1 <= j1 + 1) load_raw<MODE_S1>(P, (unsigned)map_row2(A, r + 1) * unx + col, raw);
        // H1's own-column inputs need no barrier: with the split barrier they
        // are requested before the wait (HSGN_S12_EARLY_H1: 1 the reloads,
        // 2 also the y-window of row r-2)
        const bool do1 = r - 1 >= j0 - 1 && fa;
        double yj[5], kj[5];
        YQ yp1;
        if (HSGN_S12_EARLY_H1 >= 1 && do1) {
            const unsigned offj = (unsigned)map_row2(A, r - 1) * unx + col;
#pragma unroll
            for (int f = 0; f < 5; ++f) {
                yj[f] = __ldg(P.y[f] + offj);
                kj[f] = __ldg(P.k[f] + offj);
            }
            if (HSGN_S12_EARLY_H1 >= 2) neighbour_y((clamp_lo && r - 1 == 0 ? pb : pa) + tid, yp1);
        }
        if (HSGN_S12_SPLITBAR) {
            if (k > 0) mbar_wait(&s_bar[(k - 1) & 1], (unsigned)((k - 1) >> 1) & 1u);
        } else {
            __syncthreads();
        }
        // ---- H1: k2 at row r-1 -> stage-2 input -> ring B (qc)
        YQ yb;
        double rhbc = 0.0, partc[5];
        if (do1) {
            const int j = r - 1;
            // y, k1 of row j again (this thread loaded them one row ago: L1/L2)
            const unsigned offj = (unsigned)map_row2(A, j) * unx + col;
            if (HSGN_S12_EARLY_H1 < 1) {
#pragma unroll
                for (int f = 0; f < 5; ++f) {
                    yj[f] = __ldg(P.y[f] + offj);
                    kj[f] = __ldg(P.k[f] + offj);
                }
            }
            YQ yp, yc;
            if (HSGN_S12_EARLY_H1 >= 2)
                yp = yp1;
            else
                neighbour_y((clamp_lo && j == 0 ? pb : pa) + tid, yp);  // ywin_prev
            const bool hi = clamp_hi && j == ny - 1;
            if (hi || !HSGN_S12_PASS_A) neighbour_y((hi ? pb : pc) + tid, yc);
            const double cy = (j == jc0 || j == jc1) ? A.c1y : A.cpy;
            double k2[5];
            tendency<KIND, false, false>(A, pb, tid, sl, sr, cx, cy, xl, xr, i, j, yp, (hi || !HSGN_S12_PASS_A) ? yc : ya, rhap,
                           k2);
            double q[5];
#pragma unroll
            for (int f = 0; f < 5; ++f) {
                q[f] = dadd(yj[f], dmul(A.a2, k2[f]));                                  // state_add1
                partc[f] = dadd(dadd(yj[f], dmul(A.c1, kj[f])), dmul(A.c2, k2[f]));  // state_add3, 2 terms
            }
            if (ADAPT && fb && j >= j0 && j < j1) {  // d1 k1 + d2 k2 of row j, completed by H2 one row later
                const unsigned offe = (unsigned)(j + GHOST) * unx + col;
#pragma unroll
                for (int f = 0; f < 5; ++f) P.part[f][offe] = dadd(dmul(A.d1, kj[f]), dmul(A.d2, k2[f]));
            }
            const bool ok = products_q<false>(q, pb[tid + P_EB * BX].y, qc + tid, yb, &rhbc);
            if (fb && j >= j0 && j < j1 && !ok) ++bad2;
        }
        if (HSGN_S12_LATE_PF && r + 1 <= j1 + 1) load_raw<MODE_S1>(P, (unsigned)map_row2(A, r + 1) * unx + col, raw);
        // ---- H2: k3 at row r-2 -> ynew (stored, min h)
        if (r - 2 >= j0 && fb) {
            const int j = r - 2;
            YQ yp, yc;
            neighbour_y((clamp_lo && j == 0 ? qb : qa) + tid, yp);  // ywin_prev
            const bool hi = clamp_hi && j == ny - 1;
            if (hi) neighbour_y(qb + tid, yc);
            const double cy = (j == jc0 || j == jc1) ? A.c1y : A.cpy;
            const unsigned off = (unsigned)(j + GHOST) * unx + col;
            double e12[5];  // ADAPT: d1 k1 + d2 k2 stored by H1 one row ago (requested before the tendency)
            if (ADAPT) {
#pragma unroll
                for (int f = 0; f < 5; ++f) e12[f] = P.part[f][off];
            }
            double k3[5];
            tendency<KIND, false, false>(A, qb, tid, sl, sr, cx, cy, xl, xr, i, j, yp, hi ? yc : yb, rhbp, k3);
#pragma unroll
            for (int f = 0; f < 5; ++f) P.out[f][off] = dadd(partp[f], dmul(A.c3, k3[f]));  // state_add3
            if (ADAPT) {  // ((d1 k1 + d2 k2) + d3 k3) (time_integration.hpp:128-129)
#pragma unroll
                for (int f = 0; f < 5; ++f) P.part[f][off] = dadd(e12[f], dmul(A.d3, k3[f]));
            }
            const unsigned long long bits =
                (unsigned long long)__double_as_longlong(dadd(partp[0], dmul(A.c3, k3[0])));
            my_min = bits < my_min ? bits : my_min;
        }
        if (HSGN_S12_SPLITBAR) mbar_arrive(&s_bar[k & 1]);
        // ---- rotate
        double2* t = pa;
        pa = pb;
        pb = pc;
        pc = t;
        t = qa;
        qa = qb;
        qb = qc;
        qc = t;
        rhap = rhac;
        rhbp = rhbc;
#pragma unroll
        for (int f = 0; f < 5; ++f) partp[f] = partc[f];
    }
    if (bad1) atomicAdd(A.bad, bad1);
    if (bad2) atomicAdd(A.bad2, bad2);
    if (A.minh) {
        const unsigned long long m = warp_min_u64(my_min);
        if ((tid & 31) == 0) s_min[tid >> 5] = m;
        __syncthreads();
        if (tid == 0) {
            unsigned long long mm = s_min[0];
            for (int k = 1; k < BX / 32; ++k) mm = s_min[k] < mm ? s_min[k] : mm;
            if (mm != ~0ull) atomicMin(A.minh, mm);
        }
    }
}

// ------------------------------------------------------------ whole step
// One fixed BS3 step in one pass (whole-grid contexts): reads y, k1 (= f(y),
// FSAL) and b, writes ynew and k4 = f(ynew): 168 B/node per step.  The three
// stages run as a pipeline inside the CTA, each one row (and one column)
// behind the previous one:
//   iteration r:  P1  stage-1 input y + a1 k1 of row r      -> ring R1
//                 ---- barrier ----
//                 F1  k2 at row r-1; stage-2 input y + a2 k2 -> ring R2
//                     and ((y + c1 k1) + c2 k2) kept in registers
//                 F2  k3 at row r-2; ynew = part + c3 k3 (stored, min h)
//                                                          -> ring R3
//                 F3  k4 at row r-3 (stored)
// Tiles: thread t holds column i0-3+t; F1 finishes threads 1..BX-2, F2
// 2..BX-3, F3 3..BX-4 (WX3 = BX-6 columns per CTA).  Rows: the CTA owns
// [j0, j1); F3 runs those rows, F2 one more above and below, F1 two, P1
// three.  Every operation is the unfused stages' (bit-identical); the rings
// are the S31 layout (4 pairs, 1/h in registers), 72 KB per CTA.
constexpr int WX3 = BX - 6;

#ifndef HSGN_STEP_MINB
#define HSGN_STEP_MINB (12 / (BX / 32))  // 12 warps per SM (3 x 72 KB of rings)
#endif

template <int KIND>
__global__ void __launch_bounds__(BX, HSGN_STEP_MINB) sgn_step_kernel(const StageArgs A, const KPtrs P) {
    extern __shared__ __align__(16) double2 ring[];  // R1 | R2 | R3, each 3 x NPF x BX
    __shared__ unsigned long long s_min[BX / 32];
    __shared__ int s_skip;
    const int tid = threadIdx.x;
    if (A.halt) {  // failure protocol: the previous step's record
        if (tid == 0) {
            int skip = *A.halt;
            if (!skip && A.chk_bad && *A.chk_bad) skip = 1;
            if (!skip && A.chk_bad2 && *A.chk_bad2) skip = 1;
            if (!skip && A.chk_bad3 && *A.chk_bad3) skip = 1;
            if (!skip && A.chk_minh) {
                const unsigned long long mb = *A.chk_minh;
                if (mb != ~0ull && __longlong_as_double((long long)mb) <= A.h_floor) skip = 1;
            }
            if (skip) *A.halt = 1;
            s_skip = skip;
        }
        __syncthreads();
        if (s_skip) return;
    }
    const int nx = A.nx, ny = A.ny;
    const int i = (int)blockIdx.x * WX3 - 3 + tid;
    const bool f1 = tid >= 1 && tid <= BX - 2 && i >= -2 && i <= nx + 1;
    const bool f2 = tid >= 2 && tid <= BX - 3 && i >= -1 && i <= nx;
    const bool f3 = tid >= 3 && tid <= BX - 4 && i >= 0 && i < nx;
    int c = i;
    if (i < 0) c = A.x_bounded ? 0 : nx + i;
    if (i >= nx) c = (A.x_bounded || i > nx + 2) ? nx - 1 : i - nx;
    const unsigned col = (unsigned)c;
    const bool xl = A.x_bounded && i == 0, xr = A.x_bounded && i == nx - 1;
    const double cx = (xl || xr) ? A.c1x : A.cpx;
    const int sl = xl ? tid : tid - 1, sr = xr ? tid : tid + 1;
    const int j0 = A.band0 + blockIdx.y * A.rows_per_block;
    const int j1 = min(A.band1 > 0 ? A.band1 : ny, j0 + A.rows_per_block);
    const int jc0 = A.y_lo == YE_CLAMP ? 0 : INT_MIN, jc1 = A.y_hi == YE_CLAMP ? ny - 1 : INT_MIN;
    const bool clamp_hi = A.y_hi == YE_CLAMP;
    const unsigned unx = (unsigned)nx;
    unsigned long long bad1 = 0, bad2 = 0, bad3 = 0, my_min = ~0ull;

    constexpr int SLOT = NPF * BX;
    // rotating slots: at iteration r, ring k holds rows (c-2, c-1, c) in
    // (pa, pb, pc) where c = r, r-1, r-2 for R1, R2, R3 (pc is written now)
    double2 *p1a = ring, *p1b = ring + SLOT, *p1c = ring + 2 * SLOT;
    double2 *p2a = ring + 3 * SLOT, *p2b = ring + 4 * SLOT, *p2c = ring + 5 * SLOT;
    double2 *p3a = ring + 6 * SLOT, *p3b = ring + 7 * SLOT, *p3c = ring + 8 * SLOT;
    double rh1p = 0.0, rh2p = 0.0, rh3p = 0.0;  // 1/h of R1 row r-1, R2 row r-2, R3 row r-3
    double partp[5];                            // ((y + c1 k1) + c2 k2) of row r-2
#pragma unroll
    for (int f = 0; f < 5; ++f) partp[f] = 0.0;

    Raw raw;
    load_raw<MODE_S1>(P, (unsigned)map_row2(A, j0 - 3) * unx + col, raw);
#pragma unroll 1
    for (int r = j0 - 3; r <= j1 + 2; ++r) {
        // ---- P1: stage-1 input of row r; raw of row r+1 is loaded right away
        // (in flight across the three finishes)
        double rh1c;
        {
            YQ unused;
            const bool ok = products<MODE_S1, false>(A, raw, p1c + tid, unused, &rh1c);
            if (f3 && r >= j0 && r < j1 && !ok) ++bad1;
        }
        if (r + 1 <= j1 + 2) load_raw<MODE_S1>(P, (unsigned)map_row2(A, r + 1) * unx + col, raw);
        __syncthreads();
        // ---- F1: k2 at row r-1 -> stage-2 input -> R2 (slot p2c)
        double rh2c = 0.0, partc[5];
        if (r - 1 >= j0 - 2 && f1) {
            const int j = r - 1;
            // y, k1 of row j again (this thread loaded them one row ago: L1/L2)
            const unsigned offj = (unsigned)map_row2(A, j) * unx + col;
            double yj[5], kj[5];
#pragma unroll
            for (int f = 0; f < 5; ++f) {
                yj[f] = __ldg(P.y[f] + offj);
                kj[f] = __ldg(P.k[f] + offj);
            }
            YQ yp, yn;
            ywin_prev(A, j, p1a, p1b, tid, yp);
            neighbour_y((clamp_hi && j == ny - 1 ? p1b : p1c) + tid, yn);
            const double cy = (j == jc0 || j == jc1) ? A.c1y : A.cpy;
            double k2[5];
            tendency<KIND, false, false>(A, p1b, tid, sl, sr, cx, cy, xl, xr, i, j, yp, yn, rh1p, k2);
            double q[5];
#pragma unroll
            for (int f = 0; f < 5; ++f) {
                q[f] = dadd(yj[f], dmul(A.a2, k2[f]));
                partc[f] = dadd(dadd(yj[f], dmul(A.c1, kj[f])), dmul(A.c2, k2[f]));
            }
            YQ unused;
            const bool ok = products_q<false>(q, p1b[tid + P_EB * BX].y, p2c + tid, unused, &rh2c);
            if (f3 && j >= j0 && j < j1 && !ok) ++bad2;
        }
        // ---- F2: k3 at row r-2 -> ynew (stored) -> R3 (slot p3c)
        YQ y3;
        double rh3c = 0.0;
        if (r - 2 >= j0 - 1 && f2) {
            const int j = r - 2;
            YQ yp, yn;
            ywin_prev(A, j, p2a, p2b, tid, yp);
            neighbour_y((clamp_hi && j == ny - 1 ? p2b : p2c) + tid, yn);
            const double cy = (j == jc0 || j == jc1) ? A.c1y : A.cpy;
            double k3[5];
            tendency<KIND, false, false>(A, p2b, tid, sl, sr, cx, cy, xl, xr, i, j, yp, yn, rh2p, k3);
            double ynw[5];
#pragma unroll
            for (int f = 0; f < 5; ++f) ynw[f] = dadd(partp[f], dmul(A.c3, k3[f]));  // state_add3
            const bool own = f3 && j >= j0 && j < j1;
            if (own) {
                const unsigned off = (unsigned)(j + GHOST) * unx + col;
#pragma unroll
                for (int f = 0; f < 5; ++f) P.out[f][off] = ynw[f];
                const unsigned long long bits = (unsigned long long)__double_as_longlong(ynw[0]);
                my_min = bits < my_min ? bits : my_min;
            }
            const bool ok = products_q<false>(ynw, p2b[tid + P_EB * BX].y, p3c + tid, y3, &rh3c);
            if (own && !ok) ++bad3;
        }
        // ---- F3: k4 at row r-3 (stored)
        if (r - 3 >= j0 && f3) {
            const int j = r - 3;
            YQ yp;
            ywin_prev(A, j, p3a, p3b, tid, yp);
            YQ yc;
            const bool hi = clamp_hi && j == ny - 1;
            if (hi) neighbour_y(p3b + tid, yc);
            const double cy = (j == jc0 || j == jc1) ? A.c1y : A.cpy;
            double k4[5];
            tendency<KIND, false, false>(A, p3b, tid, sl, sr, cx, cy, xl, xr, i, j, yp, hi ? yc : y3, rh3p, k4);
            const unsigned off = (unsigned)(j + GHOST) * unx + col;
#pragma unroll
            for (int f = 0; f < 5; ++f) P.out2[f][off] = k4[f];
        }
        // ---- rotate
        double2* t = p1a;
        p1a = p1b;
        p1b = p1c;
        p1c = t;
        t = p2a;
        p2a = p2b;
        p2b = p2c;
        p2c = t;
        t = p3a;
        p3a = p3b;
        p3b = p3c;
        p3c = t;
        rh1p = rh1c;
        rh2p = rh2c;
        rh3p = rh3c;
#pragma unroll
        for (int f = 0; f < 5; ++f) partp[f] = partc[f];
    }
    if (bad1) atomicAdd(A.bad, bad1);
    if (bad2) atomicAdd(A.bad2, bad2);
    if (bad3) atomicAdd(A.bad3, bad3);
    if (A.minh) {
        const unsigned long long m = warp_min_u64(my_min);
        if ((tid & 31) == 0) s_min[tid >> 5] = m;
        __syncthreads();
        if (tid == 0) {
            unsigned long long mm = s_min[0];
            for (int k = 1; k < BX / 32; ++k) mm = s_min[k] < mm ? s_min[k] : mm;
            if (mm != ~0ull) atomicMin(A.minh, mm);
        }
    }
}

// Deterministic final sum of per-block partials (single CTA, fixed order,
// compensated); result goes to out[0].
__global__ void __launch_bounds__(256) sum_partials_kernel(const double* part, int n, double* out) {
    __shared__ double sh[256], sc[256];
    double s = 0.0, c = 0.0;
    for (int k = threadIdx.x; k < n; k += 256) {  // Kahan per thread, fixed stride order
        const double term = dsub(part[k], c);
        const double t = dadd(s, term);
        c = dsub(dsub(t, s), term);
        s = t;
    }
    sh[threadIdx.x] = s;
    sc[threadIdx.x] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        double S = 0.0, Cc = 0.0;
        for (int k = 0; k < 256; ++k) {
            const double term = dsub(sh[k], dadd(Cc, sc[k]));
            const double t = dadd(S, term);
            Cc = dsub(dsub(t, S), term);
            S = t;
        }
        out[0] = S;
    }
}

// ----------------------------------------------------------------- launch

__host__ __device__ constexpr size_t cmax(size_t a, size_t b) { return a < b ? b : a; }

static int band_rows(const StageArgs& A) { return (A.band1 > 0 ? A.band1 : A.ny) - A.band0; }

template <int MODE, bool TMA>
__host__ __device__ constexpr size_t ring_bytes() {
    // (S2 must keep ~80 KB of L1 beside its rings -- 3 CTAs of 49 KB: its 16
    // misaligned raw streams rely on L1 line reuse between neighbouring warps;
    // at 4 CTAs or with padded rings it measured 2.95 vs 2.05 ms at 8192^2.)
    return sizeof(double2) * ring_slots<MODE, TMA>() * npairs<MODE>() * BX +
           (TMA ? sizeof(double) * RSLOTS * nraw<MODE>() * RW : 0);
}

// Dynamic shared memory above the 48 KB default needs a per-function opt-in,
// and the attribute is per device: opt each kernel in once on every device
// it is launched on (a racing second opt-in from another host thread is
// harmless).
template <class K>
static cudaError_t smem_opt_in(unsigned long long& done, K kernel, size_t bytes) {
    int d = 0;
    cudaGetDevice(&d);
    if (d < 64 && ((done >> d) & 1ull)) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess && d < 64) done |= 1ull << d;
    return e;
}

template <int MODE, int KIND, bool TMA>
static cudaError_t launch_tma(const StageArgs& A, const KPtrs& P, cudaStream_t st) {
    static unsigned long long opted = 0;
    const cudaError_t e = smem_opt_in(opted, sgn_stage_kernel<MODE, KIND, TMA>, ring_bytes<MODE, TMA>());
    if (e != cudaSuccess) return e;
    dim3 grid((A.nx + WX - 1) / WX, (band_rows(A) + A.rows_per_block - 1) / A.rows_per_block);
    sgn_stage_kernel<MODE, KIND, TMA><<<grid, BX, ring_bytes<MODE, TMA>(), st>>>(A, P);
    return cudaGetLastError();
}

template <int MODE, int KIND>
static cudaError_t launch_mode(const StageArgs& A, cudaStream_t st) {
    KPtrs P;  // field bases at the ghost row -1 (see map_row)
    const long long g = A.nx;
    for (int f = 0; f < 5; ++f) {
        P.y[f] = A.y ? A.y + f * A.fs - g : nullptr;
        P.k[f] = A.k ? A.k + f * A.fs - g : nullptr;
        P.kc[f] = A.kc ? A.kc + f * A.fs - g : nullptr;
        P.out[f] = A.out ? A.out + f * A.fs - g : nullptr;
        P.part[f] = A.part ? A.part + f * A.fs - g : nullptr;
        P.yold[f] = A.yold ? A.yold + f * A.fs - g : nullptr;
        P.out2[f] = A.out2 ? A.out2 + f * A.fs - g : nullptr;
    }
    P.b = A.b - g;  // per-stage kernels: bases at row -1 (see map_row)
    // TMA staging needs 16-byte aligned row pieces: nx even (host decides)
    if (A.tma && (A.nx % 2) == 0) return launch_tma<MODE, KIND, true>(A, P, st);
    return launch_tma<MODE, KIND, false>(A, P, st);
}

template <int KIND>
static cudaError_t launch_s31(const StageArgs& A, cudaStream_t st) {
    if (A.source || A.shallow) return cudaErrorInvalidValue;  // fused kernels: neither (see tendency)
    constexpr size_t bytes = sizeof(double2) * 2 * 3 * NPF * BX;
    static unsigned long long opted = 0;
    const cudaError_t e = smem_opt_in(opted, sgn_s31_kernel<KIND>, bytes);
    if (e != cudaSuccess) return e;
    KPtrs P;
    const long long g = A.nx;
    for (int f = 0; f < 5; ++f) {
        P.y[f] = A.y + f * A.fs - GHOST * g;
        P.k[f] = P.kc[f] = P.yold[f] = nullptr;
        P.part[f] = nullptr;
        P.out[f] = A.out + f * A.fs - GHOST * g;
        P.out2[f] = A.out2 + f * A.fs - GHOST * g;
    }
    P.b = A.b - GHOST * g;
    dim3 grid((A.nx + WX2 - 1) / WX2, (band_rows(A) + A.rows_per_block - 1) / A.rows_per_block);
    sgn_s31_kernel<KIND><<<grid, BX, bytes, st>>>(A, P);
    return cudaGetLastError();
}

template <int KIND>
static cudaError_t launch_step(const StageArgs& A, cudaStream_t st) {
    if (A.source || A.shallow) return cudaErrorInvalidValue;  // fused kernels: neither (see tendency)
    constexpr size_t bytes = sizeof(double2) * 3 * 3 * NPF * BX;
    static unsigned long long opted = 0;
    const cudaError_t e = smem_opt_in(opted, sgn_step_kernel<KIND>, bytes);
    if (e != cudaSuccess) return e;
    KPtrs P;
    const long long g = A.nx;
    for (int f = 0; f < 5; ++f) {
        P.y[f] = A.y + f * A.fs - GHOST * g;
        P.k[f] = A.k + f * A.fs - GHOST * g;
        P.kc[f] = P.yold[f] = nullptr;
        P.part[f] = nullptr;
        P.out[f] = A.out + f * A.fs - GHOST * g;
        P.out2[f] = A.out2 + f * A.fs - GHOST * g;
    }
    P.b = A.b - GHOST * g;
    dim3 grid((A.nx + WX3 - 1) / WX3, (band_rows(A) + A.rows_per_block - 1) / A.rows_per_block);
    sgn_step_kernel<KIND><<<grid, BX, bytes, st>>>(A, P);
    return cudaGetLastError();
}

template <int KIND>
static cudaError_t launch_s12(const StageArgs& A, cudaStream_t st) {
    if (A.source || A.shallow) return cudaErrorInvalidValue;  // fused kernels: neither (see tendency)
    constexpr size_t bytes = sizeof(double2) * 2 * 3 * NPF * BX;
    static unsigned long long opted_f = 0, opted_a = 0;
    cudaError_t e = smem_opt_in(opted_f, sgn_s12_kernel<KIND, false>, bytes);
    if (e == cudaSuccess) e = smem_opt_in(opted_a, sgn_s12_kernel<KIND, true>, bytes);
    if (e != cudaSuccess) return e;
    KPtrs P;
    const long long g = A.nx;
    for (int f = 0; f < 5; ++f) {
        P.y[f] = A.y + f * A.fs - GHOST * g;
        P.k[f] = A.k + f * A.fs - GHOST * g;
        P.kc[f] = P.yold[f] = nullptr;
        P.out2[f] = nullptr;
        P.part[f] = A.part ? A.part + f * A.fs - GHOST * g : nullptr;
        P.out[f] = A.out + f * A.fs - GHOST * g;
    }
    P.b = A.b - GHOST * g;
    dim3 grid((A.nx + WX2 - 1) / WX2, (band_rows(A) + A.rows_per_block - 1) / A.rows_per_block);
    if (A.adaptive)
        sgn_s12_kernel<KIND, true><<<grid, BX, bytes, st>>>(A, P);
    else
        sgn_s12_kernel<KIND, false><<<grid, BX, bytes, st>>>(A, P);
    return cudaGetLastError();
}

template <int KIND>
static cudaError_t launch_kind(int mode, const StageArgs& A, cudaStream_t st) {
    switch (mode) {
        case MODE_S12: return launch_s12<KIND>(A, st);
        case MODE_STEP: return launch_step<KIND>(A, st);
        case MODE_S31: return launch_s31<KIND>(A, st);
        case MODE_RHS: return launch_mode<MODE_RHS, KIND>(A, st);
        case MODE_S1: return launch_mode<MODE_S1, KIND>(A, st);
        case MODE_S2: return launch_mode<MODE_S2, KIND>(A, st);
        default: return A.adaptive ? launch_mode<MODE_S3A, KIND>(A, st) : launch_mode<MODE_S3, KIND>(A, st);
    }
}

// A.pow2 carries the stencil kind chosen by the host (see sbp_d).
cudaError_t launch_stage(int mode, const StageArgs& A, cudaStream_t st) {
    if (A.pow2 == 2) return launch_kind<2>(mode, A, st);
    if (A.pow2 == 1) return launch_kind<1>(mode, A, st);
    return launch_kind<0>(mode, A, st);
}

int stage_grid_blocks(const StageArgs& A) {
    return ((A.nx + WX - 1) / WX) * ((A.ny + A.rows_per_block - 1) / A.rows_per_block);
}

cudaError_t launch_sum_partials(const double* part, int n, double* out, cudaStream_t st) {
    sum_partials_kernel<<<1, 256, 0, st>>>(part, n, out);
    return cudaGetLastError();
}

}  // namespace hsgn_dev
