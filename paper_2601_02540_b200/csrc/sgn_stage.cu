// sgn_stage.cu -- the fused fp64 split-form SGN stage kernels for sm_100a.
//
// One launch evaluates the reference's whole tendency (rhs.hpp:77-214:
// products pass, 22 SBP stencil passes, wall SAT, combine pass, optional
// manufactured source) for every node of a slab in ONE pass over HBM, with
// the Bogacki-Shampine stage algebra of time_integration.hpp:277-286 fused
// into its prologue (stage input y + a*k formed on the fly at every stencil
// point) and epilogue (ynew in stage 2, error partials in adaptive mode).
//
// Two kernels (DESIGN.md sections 2, 2b):
//   * sgn_stage_kernel<MODE, KIND, IN>: one tendency per launch (RHS, S1, S2,
//     S3, adaptive S3A).  Used for rhs(), the per-stage structure and stage 3
//     of the default fixed step;
//   * sgn_s12_kernel<KIND, ADAPT, IN>: stages 1 and 2 of a BS3 step in one
//     pass (reads y, k1, b; writes ynew), the dominant kernel.
// Work decomposition: a CTA of BX = 128 threads owns BX consecutive columns
// (overlapped tiles: the halo columns are recomputed by the neighbour tile)
// and marches down a strip of rows; each thread loads the raw inputs of the
// next row into registers one row ahead; the x-stencil reads columns i-1,
// i+1 of a 3-row shared-memory ring holding the node's stage inputs (four
// 16-byte double2 pairs, neighbour products re-formed with the identical
// operations); the y-stencil uses the next row's y-quantities in registers
// and re-forms the previous row's from its ring entry.
//
// Walls (SBP closures + SAT, sbp.hpp:108-117,156-179,267-285) are confined
// to EDGE tiles: the host splits a bounded grid into the tiles that touch a
// closure column / row (IN = false: clamped neighbours, closure coefficient,
// SAT face terms) and the interior tiles (IN = true: none of those
// predicates, the same arithmetic as the periodic interior).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <type_traits>

#include "sgn_device.cuh"

namespace hsgn_dev {

constexpr int BX = 128;     // threads per CTA == columns touched per tile
constexpr int WX = BX - 2;  // finished columns per tile (per-stage kernel)
constexpr int WX2 = BX - 4; // finished columns per tile (S12)
constexpr int NPF = 4;      // ring pairs per row of the fused kernel (1/h carried in registers)

template <int MODE>
__host__ __device__ constexpr int npairs() { return MODE == MODE_S2 ? NPAIRS_S2 : NPAIRS; }
#ifndef HSGN_S1_WARPS
#define HSGN_S1_WARPS 16  // per-stage S1: 4 CTAs at <= 128 registers (r2: 1.91 -> 1.72 ms at 8192^2 against 5 CTAs with spills)
#endif
#ifndef HSGN_S3_WARPS
#define HSGN_S3_WARPS 20  // resident warps per SM asked of the fixed-step stage-3 kernel
#endif
template <int MODE>
__host__ __device__ constexpr int min_blocks() {
    // measured (r1): S2 (largest ring, 16 raw inputs) is best at 3 CTAs/SM;
    // the other stages fit 96 registers without spills and run best at 5
    // (expressed as resident warps per SM: 12 for S2, 20 for the others)
    return (MODE == MODE_S2 ? 12 : MODE == MODE_S3A ? 16 : MODE == MODE_S3 ? HSGN_S3_WARPS : MODE == MODE_S1 ? HSGN_S1_WARPS : 20) /
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

// Tile coordinates of this CTA.  A.tile_mode 0: the
// plain grid (blockIdx = tile); 1: one launch over the edge tiles and then
// the interior tiles of a grid with walls: CTAs [0, n_edge) take the edge
// tiles, enumerated as the leading / trailing edge strips (all column tiles)
// followed by the leading / trailing edge column tiles of every remaining
// strip; CTAs from n_edge on take the interior tiles row by row.
__device__ __forceinline__ bool edge_cta(const StageArgs& A) { return A.tile_mode == 1 && (int)blockIdx.x < A.n_edge; }

__device__ __forceinline__ void tile_of(const StageArgs& A, int& bx, int& by) {
    if (A.tile_mode == 0) {
        bx = blockIdx.x;
        by = blockIdx.y;
        return;
    }
    int k = blockIdx.x;
    const int ntx = A.ntx, nby = A.nby;
    if (k >= A.n_edge) {  // interior tile
        k -= A.n_edge;
        const int gx = ntx - A.ex_lo - A.ex_hi;
        bx = A.ex_lo + k % gx;
        by = A.ey_lo + k / gx;
        return;
    }
    if (k < A.ey_lo * ntx) {
        bx = k % ntx;
        by = k / ntx;
        return;
    }
    k -= A.ey_lo * ntx;
    if (k < A.ey_hi * ntx) {
        bx = k % ntx;
        by = nby - A.ey_hi + k / ntx;
        return;
    }
    k -= A.ey_hi * ntx;
    const int per = A.ex_lo + A.ex_hi;  // edge column tiles of every remaining strip
    const int r = k % per;
    by = A.ey_lo + k / per;
    bx = r < A.ex_lo ? r : ntx - A.ex_hi + (r - A.ex_lo);
}

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
// offset by ring row and column), fills the y-quantities and the node's
// magnitude guard (guard_add); returns h > 0.
template <int KIND, bool LIT, bool STORE_RH = true>
__device__ __forceinline__ bool products_q(const double q[5], double b, double2* S, YQ& Y, double* rh_out,
                                           Guard& gd) {
    const double h = q[0], u = q[1], v = q[2], w = q[3], e = q[4];
    const bool ok = h > 0.0;
    guard_add<KIND>(gd, q);
    const double rh = rcp_or_nan(h);
    bool slow = false;
    double r = div_fast(e, h, rh, slow);  // eta/h computed once (rhs.hpp:86-88)
    if (LIT && slow) r = e / h;  // fast pass: deferred to the literal pass (guard_mark)
    guard_mark(gd, slow);
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
template <int MODE, int KIND, bool LIT, bool STORE_RH = true>
__device__ __forceinline__ bool products(const StageArgs& A, const Raw& raw, double2* S, YQ& Y, Guard& gd,
                                         double* rh_out = nullptr) {
    double q[5];
#pragma unroll
    for (int f = 0; f < 5; ++f)
        q[f] = (MODE == MODE_S1 || MODE == MODE_S2) ? dadd(raw.y[f], dmul(A.a, raw.k[f])) : raw.y[f];
    const bool ok = products_q<KIND, LIT, STORE_RH>(q, raw.b, S, Y, rh_out, gd);
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
// closed form restated in DESIGN.md section 5 and oracle/hsgn_oracle.c),
// from precomputed factors: xf = (sin 2pi x, cos 2pi x, sin 4pi x, cos 4pi x)
// of the node's column (srcx table), yf the same of its row (srcy table),
// tsc = (sin 2pi t, cos 2pi t) of the stage time (shared memory, once per
// launch).  The tables hold the grid's own nodes, so a halo row / column of
// a tile takes the factors of the row / column it wraps to.
struct Src5 {
    double v[5];
};
static __device__ __noinline__ Src5 mms_source(const double* xf, const double* yf, const double* tsc, double g) {
    const double tp = 2.0 * 3.14159265358979323846, fp = 4.0 * 3.14159265358979323846;
    const double s1x = xf[0], c1x = xf[1], s2x = xf[2], c2x = xf[3];
    const double s1y = yf[0], c1y = yf[1], s2y = yf[2], c2y = yf[3];
    const double st = tsc[0], ct = tsc[1];
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
    Src5 s;  // returned in registers (an output array would go through local memory)
    s.v[0] = sh;
    s.v[1] = ut + u * ux + g * (hx + bx);
    s.v[2] = vt + v * vy + g * (hy + by);
    s.v[3] = wt + u * wx + v * wy;
    s.v[4] = sh;
    return s;
}

// (sin 2pi t, cos 2pi t) of a stage time into shared memory (one thread).
__device__ __forceinline__ void stage_time_factors(double t, double* tsc) {
    sincos(2.0 * 3.14159265358979323846 * t, &tsc[0], &tsc[1]);
}

// Adaptive-mode epilogue, kept out of line so it does not raise the register
// pressure of the fixed-step kernels.  (Scalars and base pointers are passed
// by value: taking the address of the kernel-parameter structs would copy
// them to local memory.)
// S2: ((d1 k1 + d2 k2) + d3 k3) (time_integration.hpp:128-129, first 3 terms)
static __device__ __noinline__ void s2_error_partial(const double* kc, const double* k, double* part, long long fs,
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

// ------------------------------------------------------------ mbarriers
// Split-phase row barriers: a thread arrives when it has finished a row and
// waits for the phase only when it next needs other threads' ring entries.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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

// Graph-level failure protocol: thread 0 decides
// whether this launch is skipped because an earlier stage of the captured
// step sequence failed; returns the CTA-uniform decision.
__device__ __forceinline__ bool halted(const StageArgs& A, int* s_skip) {
    if (!A.halt) return false;
    if (threadIdx.x == 0) {
        int skip = *A.halt;
#pragma unroll
        for (int k = 0; k < 3; ++k)
            if (!skip && A.chk_bad[k] && *A.chk_bad[k]) skip = 1;
        if (!skip && A.chk_minh) {
            const unsigned long long mb = *A.chk_minh;
            if (mb != ~0ull && __longlong_as_double((long long)mb) <= A.h_floor) skip = 1;
        }
        if (skip) *A.halt = 1;
        *s_skip = skip;
    }
    __syncthreads();
    return *s_skip != 0;
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
    Guard gd;           // fast pass: magnitude guard over the stage inputs this thread formed
    int t0;             // split-barrier step index of this pass's prologue
    const double* tsc;  // shared (sin, cos)(2 pi t) of the stage time (sources)
};

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

// Split-phase row barrier of the stage-3 kernels (measured: S3 1.235 ->
// 1.219 ms; S1 1.447 -> 1.478, so S1 / RHS keep __syncthreads), as in S12: step j
// arrives on an mbarrier after finishing row j and the next step waits for
// that phase only after forming its next row's products, so a warp that is
// ahead does that work instead of idling at the barrier.
template <int MODE>
__host__ __device__ constexpr bool split_bar() {
    return MODE == MODE_S3 || MODE == MODE_S3A;
}

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
// IN: interior tile of a grid with walls -- no node of the tile is a
// closure or SAT node, so the continuity sum adds the SAT field's zero
// exactly as the reference does ((-s) + 0.0) without the face predicates.
// LIT: the literal association of rhs.hpp:147-210 (every 0.5 where the
// reference has it, the stencil coefficient inside every derivative: KIND 2
// runs as KIND 1, which is exact for every input).  The fast association
// (LIT = false) factors 0.5 out of the split groups and, for KIND 2, the
// common stencil factor out of each tendency; it is used only where the
// magnitude guard (lit_node) proves it bit-identical.
template <int KIND, bool SW, bool SRC, bool IN, bool LIT>
__device__ __forceinline__ void tendency(const StageArgs& A, const double2* S, int tid, int sl, int sr, double cx,
                                         double cy, bool xl, bool xr, int i, int j, const YQ& ypr, const YQ& ynr,
                                         double rh, double o[5], Guard& gd, const double* tsc = nullptr) {
    constexpr int KD = (LIT && KIND == 2) ? 1 : KIND;  // derivative form
    constexpr bool CF = KD == 2;                       // common factor applied once per tendency
    const double2* Sc = S + tid;  // row j, own column
    // centre values of row j (products re-formed as in rhs.hpp:99-109)
    const double2 c0 = Sc[P_HU * BX], c1 = Sc[P_VW * BX], c2 = Sc[P_EB * BX], c3 = Sc[P_RHB * BX];
    const double h = c0.x, u = c0.y, v = c1.x, w = c1.y, r = c3.x, hpb = c3.y;
    const double hu = dmul(h, u), u2 = dmul(u, u), hv = dmul(h, v), v2 = dmul(v, v);
    // x-neighbours i-1, i+1
    XQ L, R;
    neighbour_x(S + sl, L);
    neighbour_x(S + sr, R);
    // interior tiles: the interior coefficients straight from the parameter
    // bank (no closure row or column), not kept in registers
    const double cxe = IN ? A.cpx : cx, cye = IN ? A.cpy : cy;
#define DX(f) const double d##f##_x = sbp_d<KD>(cxe, L.f, R.f)
#define DY(f) const double d##f##_y = sbp_d<KD>(cye, ypr.f, ynr.f)
    DX(h); DX(u); DX(v); DX(w); DX(e); DX(b); DX(hhb); DX(u2); DX(hu); DX(huv); DX(e2h); DX(huw);
    DY(h); DY(u); DY(v); DY(w); DY(e); DY(b); DY(hhb); DY(v2); DY(hv); DY(huv); DY(e2h); DY(hvw);
#undef DX
#undef DY
    const double g = A.g;
    // KIND 2 (fast): every tendency sum is linear in the (undivided)
    // differences, so the stencil coefficient is applied once per tendency
    auto sc = [&](double x) { return CF ? dmul(A.cpx, x) : x; };
    // s + 0.5*G as one rounding: 0.5*G is exact, so fma(0.5, G, s) == RN(s + RN(0.5 G))
    auto add_half = [](double s, double G) { return __fma_rn(0.5, G, s); };
    {  // continuity (rhs.hpp:156-157) + wall SAT (sbp.hpp:272-284)
        const double s = sc(dadd(dadd(dadd(dmul(u, dh_x), dmul(h, du_x)), dmul(v, dh_y)), dmul(h, dv_y)));
        double ht = -s;
        // KIND 2 implies no walls (host-checked); the per-stage kernels with
        // sources keep the runtime test (measured faster for them)
        if ((SRC || KIND != 2) && A.walls) {
            double sat = 0.0;
            if (!IN) {
                if (xl) sat = dsub(sat, dmul(A.tdx, hu));
                if (xr) sat = dadd(sat, dmul(A.tdx, hu));
                if (j == 0 && A.sat_y_lo) sat = dsub(sat, dmul(A.tdy, hv));
                if (j == A.ny - 1 && A.sat_y_hi) sat = dadd(sat, dmul(A.tdy, hv));
            }
            ht = dadd(ht, sat);
        }
        o[0] = ht;
    }
    const double ghb = dmul(g, hpb);
    const double ls_rr = dmul(A.lam_sixth, dmul(r, r));
    const double lt_r = dmul(A.lam_third, r);
    const double omr = dsub(1.0, r);
    const double lh_omr = dmul(A.lam_half, omr);
    // relaxation groups (rhs.hpp:172-174, 185-187), formed where they are added
    auto g3 = [&](double d_h, double d_e, double d_e2h, double d_b) {
        return dadd(dsub(dsub(dadd(dmul(ls_rr, d_h), dmul(A.lam_third, d_e)), dmul(lt_r, d_e)),
                         dmul(A.lam_sixth, d_e2h)),
                    dmul(lh_omr, d_b));
    };
    double nu, nv, nw;  // division numerators (before the common factor in KIND 2)
    if (LIT) {
        // rhs.hpp:167-200 as written: (0.5*h), (0.5*u), (0.5*hu) ... formed first
        const double h5 = dmul(0.5, h), u5 = dmul(0.5, u), v5 = dmul(0.5, v);
        const double hu5 = dmul(0.5, hu), hv5 = dmul(0.5, hv), uv5 = dmul(u5, v);
        {  // x-momentum
            double s = dsub(dmul(g, dhhb_x), dmul(ghb, dh_x));
            s = dadd(s, dsub(dadd(dsub(dmul(h5, du2_x), dmul(dmul(0.5, u2), dh_x)), dmul(u5, dhu_x)),
                             dmul(hu5, du_x)));
            s = dadd(s, dsub(dadd(dsub(dmul(0.5, dhuv_y), dmul(uv5, dh_y)), dmul(hv5, du_y)), dmul(hu5, dv_y)));
            nu = -dadd(s, g3(dh_x, de_x, de2h_x, db_x));
        }
        {  // y-momentum
            double s = dsub(dmul(g, dhhb_y), dmul(ghb, dh_y));
            s = dadd(s, dsub(dadd(dsub(dmul(h5, dv2_y), dmul(dmul(0.5, v2), dh_y)), dmul(v5, dhv_y)),
                             dmul(hv5, dv_y)));
            s = dadd(s, dsub(dadd(dsub(dmul(0.5, dhuv_x), dmul(uv5, dh_x)), dmul(hu5, dv_x)), dmul(hv5, du_x)));
            nv = -dadd(s, g3(dh_y, de_y, de2h_y, db_y));
        }
        {  // vertical velocity
            const double hw5 = dmul(h5, w);
            double s = dsub(dsub(dadd(dmul(0.5, dhuw_x), dmul(hu5, dw_x)), dmul(dmul(u5, w), dh_x)), dmul(hw5, du_x));
            s = dadd(s, dsub(dsub(dadd(dmul(0.5, dhvw_y), dmul(hv5, dw_y)), dmul(dmul(v5, w), dh_y)),
                             dmul(hw5, dv_y)));
            nw = dsub(dmul(A.lambda, omr), s);
        }
    } else {
        const double uv = dmul(u, v);
        {  // x-momentum (rhs.hpp:167-175), 0.5 factored out of the two split groups
            double s = dsub(dmul(g, dhhb_x), dmul(ghb, dh_x));
            s = add_half(s, dsub(dadd(dsub(dmul(h, du2_x), dmul(u2, dh_x)), dmul(u, dhu_x)), dmul(hu, du_x)));
            s = add_half(s, dsub(dadd(dsub(dhuv_y, dmul(uv, dh_y)), dmul(hv, du_y)), dmul(hu, dv_y)));
            nu = -dadd(s, g3(dh_x, de_x, de2h_x, db_x));
        }
        {  // y-momentum (rhs.hpp:180-188)
            double s = dsub(dmul(g, dhhb_y), dmul(ghb, dh_y));
            s = add_half(s, dsub(dadd(dsub(dmul(h, dv2_y), dmul(v2, dh_y)), dmul(v, dhv_y)), dmul(hv, dv_y)));
            s = add_half(s, dsub(dadd(dsub(dhuv_x, dmul(uv, dh_x)), dmul(hu, dv_x)), dmul(hv, du_x)));
            nv = -dadd(s, g3(dh_y, de_y, de2h_y, db_y));
        }
        {  // vertical velocity (rhs.hpp:196-200)
            const double hw = dmul(h, w);
            double s =
                dmul(0.5, dsub(dsub(dadd(dhuw_x, dmul(hu, dw_x)), dmul(dmul(u, w), dh_x)), dmul(hw, du_x)));
            s = add_half(s, dsub(dsub(dadd(dhvw_y, dmul(hv, dw_y)), dmul(dmul(v, w), dh_y)), dmul(hw, dv_y)));
            nw = dsub(dmul(A.lambda, omr), sc(s));
        }
    }
    {  // the three "/h" (rhs.hpp:175,188,200), one range test per node
        bool slow = false;
        double qu = div_fast(nu, h, rh, slow), qv = div_fast(nv, h, rh, slow), qw = div_fast(nw, h, rh, slow);
        guard_mark(gd, slow);  // fast pass: the literal pass redoes the tile
        if (LIT && slow) {
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
        // the node's grid column / global row (halo nodes wrap or clamp like the grid)
        int ig = i, jg = A.j_global0 + j;
        if (ig < 0) ig = A.x_bounded ? 0 : ig + A.nx;
        if (ig >= A.nx) ig = A.x_bounded ? A.nx - 1 : ig - A.nx;
        if (jg < 0) jg = A.y_bounded ? 0 : jg + A.ny_global;
        if (jg >= A.ny_global) jg = A.y_bounded ? A.ny_global - 1 : jg - A.ny_global;
        const Src5 s5 = mms_source(A.srcx + 4 * ig, A.srcy + 4 * jg, tsc, A.g);
#pragma unroll
        for (int f = 0; f < 5; ++f) o[f] = dadd(o[f], s5.v[f]);
    }
}

// Two-pass tiles: a CTA marches its tile with the
// fast association and records whether any stage input it formed failed
// the magnitude guard (lit_node).  If one did (rare: wavefronts entering
// water at rest), the CTA marches the tile again with the literal
// association and overwrites its outputs; its inputs are never written by
// the launch, so the second pass sees the same data.  The counters and
// reductions are taken from the pass that produced the outputs.  Keeping
// the literal code in a second loop (not a branch inside the first) leaves
// the fast loop's register allocation untouched.

// One row of the march: form row jn = j+1 (ring slot SN, register set yn),
// then finish row j (ring slot SC; row j-1 is register set yp for S2, its
// ring entry otherwise).
template <int MODE, int KIND, bool IN, bool LIT, int SC, bool SRC>
__device__ __forceinline__ void march_row(const StageArgs& A, const KPtrs& P, Thr& T, double2* ring, int j0, int j,
                                          const YQ& yp, YQ& yn, Raw& raw, unsigned long long* sbar) {
    constexpr int NP = npairs<MODE>();
    constexpr bool SPLIT = split_bar<MODE>();
    constexpr int SN = (SC + 1) % 3;
    const int jn = j + 1;
    const unsigned nx = (unsigned)A.nx;
    {  // products of row jn (for D_y of row j, and D_x of row jn one step later)
        const bool ok = products<MODE, KIND, LIT>(A, raw, ring + SN * (NP * BX) + T.tid, yn, T.gd);
        if (T.finish && jn < T.j1 && !ok) ++T.bad;
    }
    // register prefetch of raw(jn+1), in flight during the finish of row j
    if (jn < T.j1) load_raw<MODE>(P, (unsigned)map_row(A, jn + 1) * nx + T.col, raw);
    // One barrier per row: row j's ring entries (written one step ago) become
    // visible, and this step's writes to slot SN are ordered after the last
    // reads of that slot (finish of row j-2, before the previous barrier).
    const int t = T.t0 + j - j0 + 1;  // step index (the prologue is step t0)
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
    const double cy = (!IN && (j == T.jc0 || j == T.jc1)) ? A.c1y : A.cpy;
    // Row j-1: S1/S3/RHS re-form it from its ring entry (slot SP, own
    // column), which frees the carried window's registers (96 instead of
    // ~160) for 6 DMUL + 4 LDS.128 per node; S2 keeps the register window
    // (measured faster for S2, r1: 2.05 vs 2.95 ms).
    constexpr bool ywin_smem = MODE != MODE_S2;
    YQ yprev;
    if (ywin_smem) neighbour_y(ring + ((SC + 2) % 3) * (NP * BX) + T.tid, yprev);
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
    tendency<KIND, true, SRC, IN, LIT>(A, S, T.tid, T.sl, T.sr, T.cx, cy, T.xl, T.xr, T.i, j, ypr, yn,
                                        Sc[P_RH * BX].x, o, T.gd, T.tsc);
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

// Per-thread geometry of this CTA's tile (recomputed by each pass, so
// that only the accumulators are live across the two passes).
template <bool IN>
__device__ __forceinline__ int tile_geo(const StageArgs& A, Thr& T) {
    const int tid = threadIdx.x, nx = A.nx, ny = A.ny;
    int bx, by;
    tile_of(A, bx, by);
    T.tid = tid;
    const int i = bx * WX - 1 + tid;  // logical column (may be -1 or >= nx)
    T.i = i;
    T.finish = tid >= 1 && tid <= WX && i < nx;
    // memory column: periodic wrap of the two halo columns, clamp otherwise
    int col = i;
    if (i < 0) col = (!IN && A.x_bounded) ? 0 : nx - 1;
    if (i >= nx) col = ((!IN && A.x_bounded) || i > nx) ? nx - 1 : 0;
    T.col = (unsigned)col;
    T.xl = !IN && A.x_bounded && i == 0;
    T.xr = !IN && A.x_bounded && i == nx - 1;
    T.cx = (T.xl || T.xr) ? A.c1x : A.cpx;
    T.sl = T.xl ? tid : tid - 1;
    T.sr = T.xr ? tid : tid + 1;
    const int j0 = A.band0 + by * A.rows_per_block;
    T.j1 = min(A.band1 > 0 ? A.band1 : ny, j0 + A.rows_per_block);
    T.jc0 = A.y_lo == YE_CLAMP ? 0 : -2;
    T.jc1 = A.y_hi == YE_CLAMP ? ny - 1 : -2;
    return j0;
}

// One pass over the tile: prologue (rows j0-1, j0) and the march.
template <int MODE, int KIND, bool IN, bool LIT, bool SRC>
__device__ __forceinline__ void march_tile(const StageArgs& A, const KPtrs& P, Thr& T, double2* ring,
                                           unsigned long long* sbar) {
    constexpr int NP = npairs<MODE>();
    const int j0 = tile_geo<IN>(A, T);
    const unsigned unx = (unsigned)A.nx;
    // ---- prologue: row j0-1 -> register set C (ring slot 2), row j0 -> set A (slot 0)
    YQ ya, yb, yc;
    Raw raw;
    load_raw<MODE>(P, (unsigned)map_row(A, j0 - 1) * unx + T.col, raw);
    products<MODE, KIND, LIT>(A, raw, ring + 2 * (NP * BX) + T.tid, yc, T.gd);
    load_raw<MODE>(P, (unsigned)(j0 + 1) * unx + T.col, raw);
    {
        const bool ok = products<MODE, KIND, LIT>(A, raw, ring + T.tid, ya, T.gd);
        if (T.finish && !ok) ++T.bad;
    }
    load_raw<MODE>(P, (unsigned)map_row(A, j0 + 1) * unx + T.col, raw);
    if (split_bar<MODE>()) mbar_arrive(&sbar[T.t0 & 1]);  // step t0: rows j0-1 and j0 written
    // ---- march, unrolled by 3: row j lives in ring slot (j-j0)%3 and register
    // set {a,b,c}[(j-j0)%3]; step SC reads set SC+2 (row j-1), writes SC+1.
    for (int j = j0; j < T.j1; j += 3) {
        march_row<MODE, KIND, IN, LIT, 0, SRC>(A, P, T, ring, j0, j, yc, yb, raw, sbar);
        if (j + 1 >= T.j1) break;
        march_row<MODE, KIND, IN, LIT, 1, SRC>(A, P, T, ring, j0, j + 1, ya, yc, raw, sbar);
        if (j + 2 >= T.j1) break;
        march_row<MODE, KIND, IN, LIT, 2, SRC>(A, P, T, ring, j0, j + 2, yb, ya, raw, sbar);
    }
    T.t0 += T.j1 - j0 + 1;  // a second pass continues the barrier phases
}

template <int MODE, int KIND, bool IN, bool SRC>
__device__ __forceinline__ void stage_body(const StageArgs& A, const KPtrs& P, double2* ring, unsigned long long* s_min,
                                           double* s_err, unsigned long long* sbar, double* s_tsc) {
    const int tid = threadIdx.x;
    Thr T;
    T.bad = 0;
    T.my_min = ~0ull;
    T.my_err = 0.0;
    T.t0 = 0;
    T.tsc = s_tsc;
    if (SRC && A.source && tid == 0) stage_time_factors(A.t, s_tsc);  // read after the first row barrier

    if (split_bar<MODE>()) {
        if (tid == 0) {
            mbar_init(&sbar[0], BX);
            mbar_init(&sbar[1], BX);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    // literal-pass hint of this tile (set when its last launch needed the
    // literal pass: a front stays in a tile for many steps)
    int* hint = A.hint_stage ? A.hint_stage + blockIdx.y * gridDim.x + blockIdx.x : nullptr;
    const bool hinted = !A.lit_all && hint && *hint;
    bool redo = A.lit_all || hinted;
    if (!redo) {
        march_tile<MODE, KIND, IN, false, SRC>(A, P, T, ring, sbar);
        redo = __syncthreads_or(guard_fail(T.gd));
    }
    bool need = false;
    if (redo) {  // literal pass (outputs, counters and partials replaced)
        T.bad = 0;
        T.my_min = ~0ull;
        T.my_err = 0.0;
        T.gd = Guard();
        march_tile<MODE, KIND, IN, true, SRC>(A, P, T, ring, sbar);
        if (hint) need = __syncthreads_or(guard_fail(T.gd));
    }
    if (hint && tid == 0 && need != hinted) *hint = need;

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

// TILES 0: every tile general (IN = false); 1: every tile interior (no
// walls, or KIND 2); 2: one launch over edge tiles (general) and interior
// tiles (tile_mode 1, see tile_of).
template <int MODE, int KIND, int TILES, bool SRC = true>
__global__ void __launch_bounds__(BX, min_blocks<MODE>()) sgn_stage_kernel(const StageArgs A, const KPtrs P) {
    extern __shared__ __align__(16) double2 ring[];  // 3 x NP x BX pairs
    __shared__ unsigned long long s_min[BX / 32];
    __shared__ double s_err[BX / 32];
    __shared__ __align__(8) unsigned long long sbar[2];
    __shared__ double s_tsc[2];
    __shared__ int s_skip;
    if (halted(A, &s_skip)) return;
    if (TILES == 1 || (TILES == 2 && !edge_cta(A)))
        stage_body<MODE, KIND, true, SRC>(A, P, ring, s_min, s_err, sbar, s_tsc);
    else
        stage_body<MODE, KIND, false, SRC>(A, P, ring, s_min, s_err, sbar, s_tsc);
}

// Fused kernels: memory row of -GHOST <= jr < ny + GHOST, counted from row
// -GHOST (their KPtrs bases point there).
__device__ __forceinline__ int map_row2(const StageArgs& A, int jr) {
    if (jr < 0) return A.y_lo == YE_WRAP ? jr + A.ny + GHOST : (A.y_lo == YE_CLAMP ? GHOST : jr + GHOST);
    if (jr >= A.ny) return A.y_hi == YE_WRAP ? jr - A.ny + GHOST : (A.y_hi == YE_CLAMP ? A.ny - 1 + GHOST : jr + GHOST);
    return jr + GHOST;
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
// Tile: BX threads, columns i0-2 .. i0+BX-3; stage 1 finishes threads
// 1..BX-2, stage 2 threads 2..BX-3 (WX2 = BX-4 columns).  Rows: stage 2
// finishes [j0, j1), stage 1 one more row above and below, the stage-1
// input two.  Two 3-slot rings of 4 pairs (1/h in registers): 49 KB, 3 CTAs
// per SM at <= 168 registers.
// measured (r1, 8192^2): 3 CTAs/SM at <= 168 registers without spills runs
// S12 in 3.16 ms; forcing 4 CTAs (128 registers) spills ~380 B/thread and
// takes 7.1 ms.
#ifndef HSGN_S12_MINB
#define HSGN_S12_MINB (12 / (BX / 32))
#endif

// March unrolled by 2 (r2: S12 2.88 -> 2.81 ms periodic, 3.25 -> 3.20 walls;
// by 3 within noise of 2; not unrolled, the slot pointers rotate in registers)
#ifndef HSGN_S12_UNROLL
#define HSGN_S12_UNROLL 2
#endif
constexpr int S12_UNROLL = HSGN_S12_UNROLL;
#ifndef HSGN_S12_FLAT
#define HSGN_S12_FLAT 2
#endif
// FLAT: one branch-free iteration body (H1 and H2 evaluated on every thread
// and iteration, stores / counters / guard predicated on valid rows).
// HSGN_S12_FLAT 0: no instance; 1: every instance; 2 (default): the adaptive
// and sourced instances.  Measured (r2): it removes most of the spills of the
// adaptive / sourced instances (e.g. 592 -> 0 B) and makes the sourced
// config-2 attempt 4-5 % faster (4096^2: 2.50-2.55 -> 2.37 ms); adaptive
// neutral; the plain fixed-step instances are 2-3 % slower flat (S12 2.81 ->
// 2.87 ms periodic, 3.12 -> 3.21 walls), so they keep the branched body.
template <bool ADAPT, bool SRC>
__host__ __device__ constexpr bool s12_flat() { return HSGN_S12_FLAT == 1 || (HSGN_S12_FLAT == 2 && (ADAPT || SRC)); }

// Per-thread constants of an S12 tile.
struct S12Geo {
    int tid, i, j0, j1, jc0, jc1, sl, sr;
    bool fa, fb, xl, xr, clamp_lo, clamp_hi;
    unsigned col;
    double cx;
};

struct S12Acc {
    unsigned* bad;        // shared per-CTA depth-failure counters of stages 1, 2 (incremented on failure only)
    unsigned long long my_min;
    bool any;  // fast pass: a stage input failed the magnitude guard
};

// Per-thread geometry of this CTA's S12 tile.  No wall / clamp logic when
// PER: KIND 2 (common factor, only chosen for fully periodic grids without
// walls, host-checked) or an interior tile of a grid with walls.
template <int KIND, bool IN>
__device__ __forceinline__ S12Geo s12_geo(const StageArgs& A) {
    constexpr bool PER = KIND == 2 || IN;
    const int tid = threadIdx.x, nx = A.nx, ny = A.ny;
    int bx, by;
    tile_of(A, bx, by);
    S12Geo G;
    G.tid = tid;
    const int i = bx * WX2 - 2 + tid;
    G.i = i;
    G.fa = tid >= 1 && tid <= BX - 2 && i >= -1 && i <= nx;  // stage-1 finish
    G.fb = tid >= 2 && tid <= BX - 3 && i >= 0 && i < nx;    // stage-2 finish (owned column)
    int c = i;
    if (i < 0) c = (!PER && A.x_bounded) ? 0 : nx + i;
    if (i >= nx) c = ((!PER && A.x_bounded) || i > nx + 1) ? nx - 1 : i - nx;
    G.col = (unsigned)c;
    G.xl = !PER && A.x_bounded && i == 0;
    G.xr = !PER && A.x_bounded && i == nx - 1;
    G.cx = (G.xl || G.xr) ? A.c1x : A.cpx;
    // (clamped at the tile edge: the edge threads never finish a node, and
    // the steady march reads their ring columns in bounds)
    G.sl = (G.xl || tid == 0) ? tid : tid - 1;
    G.sr = (G.xr || tid == BX - 1) ? tid : tid + 1;
    G.j0 = A.band0 + by * A.rows_per_block;
    G.j1 = min(A.band1 > 0 ? A.band1 : ny, G.j0 + A.rows_per_block);
    G.jc0 = (!PER && A.y_lo == YE_CLAMP) ? 0 : INT_MIN;
    G.jc1 = (!PER && A.y_hi == YE_CLAMP) ? ny - 1 : INT_MIN;
    G.clamp_lo = !PER && A.y_lo == YE_CLAMP;
    G.clamp_hi = !PER && A.y_hi == YE_CLAMP;
    return G;
}

// One pass of S12 over the tile.  k: iteration index (split barrier
// phases), continued by a second pass (which therefore waits from its first
// iteration on: the fast pass's last phase).
// ADAPT: also store the error partial ((d1 k1 + d2 k2) + d3 k3)
// (time_integration.hpp:128-129, the S2 epilogue of the per-stage path) for
// the adaptive S3's error norm.
template <int KIND, bool ADAPT, bool SRC, bool IN, bool LIT>
__device__ __forceinline__ void s12_march(const StageArgs& A, const KPtrs& P, double2* ring,
                                          unsigned long long* s_bar, int& k, S12Acc& acc, const double* s_tsc) {
    constexpr bool FLAT = s12_flat<ADAPT, SRC>();
    const S12Geo G = s12_geo<KIND, IN>(A);
    const int tid = G.tid, i = G.i, j0 = G.j0, j1 = G.j1, ny = A.ny;
    const unsigned unx = (unsigned)A.nx, col = G.col;
    constexpr int SLOT = NPF * BX;
    // at iteration r ring A holds rows (r-2, r-1, r) in (pa, pb, pc), ring B
    // rows (r-3, r-2, r-1) in (qa, qb, qc); pc and qc are written now
    double2 *pa = ring, *pb = ring + SLOT, *pc = ring + 2 * SLOT;
    double2 *qa = ring + 3 * SLOT, *qb = ring + 4 * SLOT, *qc = ring + 5 * SLOT;
    double rhap = 0.0, rhbp = 0.0;  // 1/h of ring A row r-1 / ring B row r-2
    double partp[5];                // ((y + c1 k1) + c2 k2) of row r-2
#pragma unroll
    for (int f = 0; f < 5; ++f) partp[f] = 0.0;
    Guard gd;

    // Split-phase row barrier: iteration k arrives on s_bar[k & 1] after its
    // H2 and iteration k + 1 waits for that phase only after its P1.  P1(r)
    // needs no wait of its own (it overwrites ring A row r-3, last read
    // across threads in iteration k - 2), so a warp that is ahead forms the
    // next stage-1 input while the others finish.  (Measured slower: a
    // second barrier set with a 4-slot ring B, 2.68 vs 2.63 ms.)
    Raw raw;
    unsigned n1 = 0u, n2 = 0u;  // FLAT: depth failures of stage inputs 1, 2 on this thread's finished nodes
    // memory offsets of rows r and r-1 (mapped once, when row r is prefetched)
    unsigned off_r = (unsigned)map_row2(A, j0 - 2) * unx + col, off_rm1 = 0u;
    load_raw<MODE_S1>(P, off_r, raw);
#pragma unroll S12_UNROLL
    for (int r = j0 - 2; r <= j1 + 1; ++r, ++k) {
        // ---- P1: stage-1 input of row r (raw of row r+1 loaded right after)
        YQ ya;
        double rhac;
        {
            const bool ok = products<MODE_S1, KIND, LIT, false>(A, raw, pc + tid, ya, gd, &rhac);
            if (FLAT)
                n1 += (G.fb && r >= j0 && r < j1 && !ok) ? 1u : 0u;
            else if (G.fb && r >= j0 && r < j1 && !ok)
                atomicAdd(&acc.bad[0], 1u);
        }
        unsigned off_rp1 = 0u;
        if (FLAT) {  // the last iteration reloads row j1 + 1 (never read)
            off_rp1 = (unsigned)map_row2(A, min(r + 1, j1 + 1)) * unx + col;
            load_raw<MODE_S1>(P, off_rp1, raw);
        } else if (r + 1 <= j1 + 1) {
            off_rp1 = (unsigned)map_row2(A, r + 1) * unx + col;
            load_raw<MODE_S1>(P, off_rp1, raw);
        }
        // H1's own-column inputs need no barrier: they are requested before
        // the wait (this thread loaded them one row ago: L1/L2 hits)
        const bool do1 = r - 1 >= j0 - 1 && G.fa;
        double yj[5], kj[5];
        if (FLAT || do1) {
            const unsigned offj = off_rm1;
#pragma unroll
            for (int f = 0; f < 5; ++f) {
                yj[f] = __ldg(P.y[f] + offj);
                kj[f] = __ldg(P.k[f] + offj);
            }
        }
        if (k > 0) mbar_wait(&s_bar[(k - 1) & 1], (unsigned)((k - 1) >> 1) & 1u);
        // ---- H1: k2 at row r-1 -> stage-2 input -> ring B (qc)
        YQ yb;
        double rhbc = 0.0, partc[5];
        if (FLAT || do1) {
            const int j = r - 1;
            YQ yp, yc;
            neighbour_y((G.clamp_lo && j == 0 ? pb : pa) + tid, yp);  // a clamped wall row reads itself
            const bool hi = G.clamp_hi && j == ny - 1;
            if (hi) neighbour_y(pb + tid, yc);
            const double cy = (j == G.jc0 || j == G.jc1) ? A.c1y : A.cpy;
            double k2[5];
            Guard g1;
            tendency<KIND, false, SRC, IN, LIT>(A, pb, tid, G.sl, G.sr, G.cx, cy, G.xl, G.xr, i, j, yp,
                                                hi ? yc : ya, rhap, k2, FLAT ? g1 : gd, s_tsc);
            double q[5];
#pragma unroll
            for (int f = 0; f < 5; ++f) {
                q[f] = dadd(yj[f], dmul(A.a2, k2[f]));                                  // state_add1
                partc[f] = dadd(dadd(yj[f], dmul(A.c1, kj[f])), dmul(A.c2, k2[f]));  // state_add3, 2 terms
            }
            if (ADAPT && G.fb && j >= j0 && j < j1) {  // d1 k1 + d2 k2 of row j, completed by H2 one row later
                const unsigned offe = (unsigned)(j + GHOST) * unx + col;
#pragma unroll
                for (int f = 0; f < 5; ++f) P.part[f][offe] = dadd(dmul(A.d1, kj[f]), dmul(A.d2, k2[f]));
            }
            const bool ok =
                products_q<KIND, LIT, false>(q, pb[tid + P_EB * BX].y, qc + tid, yb, &rhbc, FLAT ? g1 : gd);
            if (FLAT) {
                n2 += (G.fb && j >= j0 && j < j1 && !ok) ? 1u : 0u;
                guard_merge(gd, g1, do1);
            } else if (G.fb && j >= j0 && j < j1 && !ok) {
                atomicAdd(&acc.bad[1], 1u);
            }
        }
        // ---- H2: k3 at row r-2 -> ynew (stored, min h)
        const bool do2 = r - 2 >= j0 && G.fb;
        if (FLAT || do2) {
            const int j = r - 2;
            YQ yp, yc;
            neighbour_y((G.clamp_lo && j == 0 ? qb : qa) + tid, yp);
            const bool hi = G.clamp_hi && j == ny - 1;
            if (hi) neighbour_y(qb + tid, yc);
            const double cy = (j == G.jc0 || j == G.jc1) ? A.c1y : A.cpy;
            const unsigned off = (unsigned)(j + GHOST) * unx + col;
            double e12[5];  // ADAPT: d1 k1 + d2 k2 stored by H1 one row ago (requested before the tendency)
            if (ADAPT && do2) {
#pragma unroll
                for (int f = 0; f < 5; ++f) e12[f] = P.part[f][off];
            }
            double k3[5];
            Guard g2;
            tendency<KIND, false, SRC, IN, LIT>(A, qb, tid, G.sl, G.sr, G.cx, cy, G.xl, G.xr, i, j, yp,
                                                hi ? yc : yb, rhbp, k3, FLAT ? g2 : gd, s_tsc + 2);
            if (FLAT) guard_merge(gd, g2, do2);
            double yn[5];
#pragma unroll
            for (int f = 0; f < 5; ++f) yn[f] = dadd(partp[f], dmul(A.c3, k3[f]));  // state_add3
            if (do2) {
#pragma unroll
                for (int f = 0; f < 5; ++f) P.out[f][off] = yn[f];
                if (ADAPT) {  // ((d1 k1 + d2 k2) + d3 k3) (time_integration.hpp:128-129)
#pragma unroll
                    for (int f = 0; f < 5; ++f) P.part[f][off] = dadd(e12[f], dmul(A.d3, k3[f]));
                }
            }
            const unsigned long long bits = (unsigned long long)__double_as_longlong(yn[0]);
            acc.my_min = (do2 && bits < acc.my_min) ? bits : acc.my_min;
        }
        mbar_arrive(&s_bar[k & 1]);
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
        off_rm1 = off_r;
        off_r = off_rp1;
#pragma unroll
        for (int f = 0; f < 5; ++f) partp[f] = partc[f];
    }
    if (FLAT) {
        if (n1) atomicAdd(&acc.bad[0], n1);
        if (n2) atomicAdd(&acc.bad[1], n2);
    }
    acc.any = guard_fail(gd);
}

template <int KIND, bool ADAPT, bool SRC, bool IN>
__device__ __forceinline__ void s12_body(const StageArgs& A, const KPtrs& P, double2* ring, unsigned long long* s_min,
                                         unsigned long long* s_bar) {
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int q = 0; q < 2; ++q) mbar_init(&s_bar[q], BX);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    __shared__ unsigned s_bad[2];
    __shared__ double s_tsc[4];  // SRC: (sin, cos)(2 pi t) of the stage-1 and stage-2 times
    if (tid < 2) s_bad[tid] = 0u;
    if (SRC && tid == 0) {
        stage_time_factors(A.t, s_tsc);
        stage_time_factors(A.t2, s_tsc + 2);
    }
    __syncthreads();
    S12Acc acc{s_bad, ~0ull, false};
    int k = 0;
    // literal-pass hint of this tile (see stage_body)
    int* hint = A.hint_s12 ? A.hint_s12 + blockIdx.y * gridDim.x + blockIdx.x : nullptr;
    const bool hinted = !A.lit_all && hint && *hint;
    bool redo = A.lit_all || hinted;
    if (!redo) {
        s12_march<KIND, ADAPT, SRC, IN, false>(A, P, ring, s_bar, k, acc, s_tsc);
        redo = __syncthreads_or(acc.any);
        if (redo) {  // the fast pass's counts are discarded
            if (tid < 2) s_bad[tid] = 0u;
            __syncthreads();
        }
    }
    bool need = false;
    if (redo) {  // literal pass (outputs, counters and min replaced)
        acc = S12Acc{s_bad, ~0ull, false};
        s12_march<KIND, ADAPT, SRC, IN, true>(A, P, ring, s_bar, k, acc, s_tsc);
        if (hint) need = __syncthreads_or(acc.any);
    }
    if (hint && tid == 0 && need != hinted) *hint = need;
    __syncthreads();
    if (tid == 0 && s_bad[0]) atomicAdd(A.bad, (unsigned long long)s_bad[0]);
    if (tid == 0 && s_bad[1]) atomicAdd(A.bad2, (unsigned long long)s_bad[1]);
    if (A.minh) {
        const unsigned long long m = warp_min_u64(acc.my_min);
        if ((tid & 31) == 0) s_min[tid >> 5] = m;
        __syncthreads();
        if (tid == 0) {
            unsigned long long mm = s_min[0];
            for (int q = 1; q < BX / 32; ++q) mm = s_min[q] < mm ? s_min[q] : mm;
            if (mm != ~0ull) atomicMin(A.minh, mm);
        }
    }
}

template <int KIND, bool ADAPT, bool SRC, int TILES>
__global__ void __launch_bounds__(BX, HSGN_S12_MINB) sgn_s12_kernel(const StageArgs A, const KPtrs P) {
    extern __shared__ __align__(16) double2 ring[];  // ring A | ring B, each 3 x NPF x BX
    __shared__ unsigned long long s_min[BX / 32];
    __shared__ __align__(8) unsigned long long s_bar[2];
    __shared__ int s_skip;
    if (halted(A, &s_skip)) return;
    if (TILES == 1 || (TILES == 2 && !edge_cta(A)))
        s12_body<KIND, ADAPT, SRC, true>(A, P, ring, s_min, s_bar);
    else
        s12_body<KIND, ADAPT, SRC, false>(A, P, ring, s_min, s_bar);
}

// ----------------------------------------------------------------- launch

static int band_rows(const StageArgs& A) { return (A.band1 > 0 ? A.band1 : A.ny) - A.band0; }

template <int MODE>
__host__ __device__ constexpr size_t ring_bytes() {
    // (S2 must keep ~80 KB of L1 beside its rings -- 3 CTAs of 49 KB: its 16
    // misaligned raw streams rely on L1 line reuse between neighbouring warps;
    // at 4 CTAs or with padded rings it measured 2.95 vs 2.05 ms at 8192^2.)
    return sizeof(double2) * 3 * npairs<MODE>() * BX;
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

// Tile split of a launch: with walls and KIND < 2,
// the tiles that evaluate a tendency on a closure column / row or load a
// clamped column run the general (IN = false) instance, the others the
// interior one; without walls every tile is interior.  `wx`: finished
// columns per tile; `hx`: columns loaded beyond them on each side (1
// per-stage, 2 S12); `reach`: rows beyond its strip on which the kernel
// evaluates a tendency (0 per-stage, 1 S12: stage 1 runs one row above and
// below).  A column tile is interior when its loaded columns lie inside
// [0, nx): it then evaluates tendencies on [1, nx-2] only.
struct TileSplit {
    int ntx, nby;
    int ex_lo, ex_hi;  // number of leading / trailing column tiles that are edge tiles
    int ey_lo, ey_hi;  // number of leading / trailing strips that are edge strips
    int n_edge;        // edge tiles; -1: no separable interior (general instance everywhere)
};

static TileSplit tile_split(const StageArgs& A, int wx, int hx, int reach) {
    TileSplit s{};
    s.ntx = (A.nx + wx - 1) / wx;
    s.nby = (band_rows(A) + A.rows_per_block - 1) / A.rows_per_block;
    if (A.pow2 == 2 || !A.walls) return s;  // no closure nodes anywhere
    const int rb = A.rows_per_block, b0 = A.band0, b1 = A.band1 > 0 ? A.band1 : A.ny;
    if (A.x_bounded) {
        auto edge_tile = [&](int bx) { return bx * wx - hx < 0 || bx * wx + wx - 1 + hx > A.nx - 1; };
        while (s.ex_lo < s.ntx && edge_tile(s.ex_lo)) ++s.ex_lo;
        while (s.ex_hi < s.ntx - s.ex_lo && edge_tile(s.ntx - 1 - s.ex_hi)) ++s.ex_hi;
    }
    auto edge_strip = [&](int k) {
        const int j0 = b0 + k * rb, j1 = std::min(b1, j0 + rb);
        return (A.y_lo == YE_CLAMP && j0 - reach <= 0) || (A.y_hi == YE_CLAMP && j1 - 1 + reach >= A.ny - 1);
    };
    while (s.ey_lo < s.nby && edge_strip(s.ey_lo)) ++s.ey_lo;
    while (s.ey_hi < s.nby - s.ey_lo && edge_strip(s.nby - 1 - s.ey_hi)) ++s.ey_hi;
    const int nx_in = s.ntx - s.ex_lo - s.ex_hi, ny_in = s.nby - s.ey_lo - s.ey_hi;
    if (nx_in <= 0 || ny_in <= 0) {
        s.n_edge = -1;
        return s;
    }
    s.n_edge = (s.ey_lo + s.ey_hi) * s.ntx + (s.ex_lo + s.ex_hi) * ny_in;
    return s;
}

// Tile plan of one launch: 0 every tile general,
// 1 every tile interior, 2 edge tiles then interior tiles (tile_mode 1).
static int tile_plan(StageArgs& A, int wx, int hx, int reach, dim3& grid) {
    const TileSplit s = tile_split(A, wx, hx, reach);
    A.ntx = s.ntx;
    A.nby = s.nby;
    A.tile_mode = 0;
    grid = dim3(s.ntx, s.nby);
    if (s.n_edge < 0) return 0;   // no separable interior: the general instance everywhere
    if (s.n_edge == 0) return 1;  // no closure nodes
    A.ex_lo = s.ex_lo;
    A.ex_hi = s.ex_hi;
    A.ey_lo = s.ey_lo;
    A.ey_hi = s.ey_hi;
    A.n_edge = s.n_edge;
    A.tile_mode = 1;
    grid = dim3(s.ntx * s.nby, 1);  // edge CTAs first: the slower tiles start in the first wave
    return 2;
}

// Launch kernel instance K<plan> for the tile plan of these arguments,
// opting each instance in to its dynamic shared memory on first use.  KIND 2
// grids have no closure nodes (host-checked), so only plan 1 exists for them.
template <int KIND, class K0, class K1, class K2>
static cudaError_t launch_planned(const StageArgs& A, const KPtrs& P, K0 k0, K1 k1, K2 k2, unsigned long long* opted,
                                  size_t smem, int wx, int hx, int reach, cudaStream_t st) {
    StageArgs B = A;
    dim3 grid;
    const int plan = tile_plan(B, wx, hx, reach, grid);
    cudaError_t e = cudaSuccess;
    if (plan == 1 || KIND == 2) {
        e = smem_opt_in(opted[1], k1, smem);
        if (e == cudaSuccess) k1<<<grid, BX, smem, st>>>(B, P);
    } else if (plan == 0) {
        e = smem_opt_in(opted[0], k0, smem);
        if (e == cudaSuccess) k0<<<grid, BX, smem, st>>>(B, P);
    } else {
        e = smem_opt_in(opted[2], k2, smem);
        if (e == cudaSuccess) k2<<<grid, BX, smem, st>>>(B, P);
    }
    return e != cudaSuccess ? e : cudaGetLastError();
}

template <int MODE, int KIND>
static cudaError_t launch_mode(const StageArgs& A, cudaStream_t st) {
    static unsigned long long opted[3] = {0, 0, 0};
    constexpr size_t bytes = ring_bytes<MODE>();
    KPtrs P;  // field bases at the ghost row -1 (see map_row)
    const long long g = A.nx;
    for (int f = 0; f < 5; ++f) {
        P.y[f] = A.y ? A.y + f * A.fs - g : nullptr;
        P.k[f] = A.k ? A.k + f * A.fs - g : nullptr;
        P.kc[f] = A.kc ? A.kc + f * A.fs - g : nullptr;
        P.out[f] = A.out ? A.out + f * A.fs - g : nullptr;
        P.part[f] = A.part ? A.part + f * A.fs - g : nullptr;
        P.yold[f] = A.yold ? A.yold + f * A.fs - g : nullptr;
    }
    P.b = A.b - g;
    constexpr int T0 = KIND == 2 ? 1 : 0, T2 = KIND == 2 ? 1 : 2;  // KIND 2: one instance
    // the fixed-step stage 3 without a source term: an instance without the
    // source call region (the other modes keep the runtime test)
    if (MODE == MODE_S3 && !A.source) {
        static unsigned long long opted_ns[3] = {0, 0, 0};
        return launch_planned<KIND>(A, P, sgn_stage_kernel<MODE, KIND, T0, false>,
                                    sgn_stage_kernel<MODE, KIND, 1, false>, sgn_stage_kernel<MODE, KIND, T2, false>,
                                    opted_ns, bytes, WX, 1, 0, st);
    }
    return launch_planned<KIND>(A, P, sgn_stage_kernel<MODE, KIND, T0>, sgn_stage_kernel<MODE, KIND, 1>,
                                sgn_stage_kernel<MODE, KIND, T2>, opted, bytes, WX, 1, 0, st);
}

template <int KIND, bool ADAPT, bool SRC>
static cudaError_t launch_s12_k(const StageArgs& A, const KPtrs& P, cudaStream_t st) {
    constexpr size_t bytes = sizeof(double2) * 2 * 3 * NPF * BX;
    static unsigned long long opted[3] = {0, 0, 0};
    constexpr int T0 = KIND == 2 ? 1 : 0, T2 = KIND == 2 ? 1 : 2;
    return launch_planned<KIND>(A, P, sgn_s12_kernel<KIND, ADAPT, SRC, T0>, sgn_s12_kernel<KIND, ADAPT, SRC, 1>,
                                sgn_s12_kernel<KIND, ADAPT, SRC, T2>, opted, bytes, WX2, 2, 1, st);
}

template <int KIND>
static cudaError_t launch_s12(const StageArgs& A, cudaStream_t st) {
    if (A.shallow) return cudaErrorInvalidValue;  // rhs_shallow_water: per-stage kernels only
    KPtrs P;
    const long long g = A.nx;
    for (int f = 0; f < 5; ++f) {
        P.y[f] = A.y + f * A.fs - GHOST * g;
        P.k[f] = A.k + f * A.fs - GHOST * g;
        P.kc[f] = P.yold[f] = nullptr;
        P.part[f] = A.part ? A.part + f * A.fs - GHOST * g : nullptr;
        P.out[f] = A.out + f * A.fs - GHOST * g;
    }
    P.b = A.b - GHOST * g;
    if (A.source)
        return A.adaptive ? launch_s12_k<KIND, true, true>(A, P, st) : launch_s12_k<KIND, false, true>(A, P, st);
    return A.adaptive ? launch_s12_k<KIND, true, false>(A, P, st) : launch_s12_k<KIND, false, false>(A, P, st);
}

// Instantiation units: build.py compiles this file once per stencil kind and
// kernel family (-DHSGN_INST_KIND=k -DHSGN_INST_S12=0|1), so the kernel
// instances compile in parallel; the plain compile (no HSGN_INST_KIND) holds
// the dispatcher and the non-template kernels.
#define HSGN_CAT2(a, b) a##b
#define HSGN_CAT(a, b) HSGN_CAT2(a, b)
cudaError_t launch_s12_k0(const StageArgs& A, cudaStream_t st);
cudaError_t launch_s12_k1(const StageArgs& A, cudaStream_t st);
cudaError_t launch_s12_k2(const StageArgs& A, cudaStream_t st);
cudaError_t launch_mode_k0(int mode, const StageArgs& A, cudaStream_t st);
cudaError_t launch_mode_k1(int mode, const StageArgs& A, cudaStream_t st);
cudaError_t launch_mode_k2(int mode, const StageArgs& A, cudaStream_t st);

#if defined(HSGN_INST_KIND) && HSGN_INST_S12
cudaError_t HSGN_CAT(launch_s12_k, HSGN_INST_KIND)(const StageArgs& A, cudaStream_t st) {
    return launch_s12<HSGN_INST_KIND>(A, st);
}
#elif defined(HSGN_INST_KIND)
cudaError_t HSGN_CAT(launch_mode_k, HSGN_INST_KIND)(int mode, const StageArgs& A, cudaStream_t st) {
    constexpr int KIND = HSGN_INST_KIND;
    switch (mode) {
        case MODE_RHS: return launch_mode<MODE_RHS, KIND>(A, st);
        case MODE_S1: return launch_mode<MODE_S1, KIND>(A, st);
        case MODE_S2: return launch_mode<MODE_S2, KIND>(A, st);
        default: return A.adaptive ? launch_mode<MODE_S3A, KIND>(A, st) : launch_mode<MODE_S3, KIND>(A, st);
    }
}
#else
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

// A.pow2 carries the stencil kind chosen by the host (see sbp_d).
cudaError_t launch_stage(int mode, const StageArgs& A, cudaStream_t st) {
    if (mode == MODE_S12) {
        if (A.pow2 == 2) return launch_s12_k2(A, st);
        if (A.pow2 == 1) return launch_s12_k1(A, st);
        return launch_s12_k0(A, st);
    }
    if (A.pow2 == 2) return launch_mode_k2(mode, A, st);
    if (A.pow2 == 1) return launch_mode_k1(mode, A, st);
    return launch_mode_k0(mode, A, st);
}

// Kernel launches launch_stage() makes for these arguments (edge and
// interior tiles share one launch).
int stage_launches(int, const StageArgs&) { return 1; }

// CTAs of one per-stage launch (edge + interior tiles), the size of the S3A
// error-partial array.
int stage_grid_blocks(const StageArgs& A) {
    return ((A.nx + WX - 1) / WX) * ((band_rows(A) + A.rows_per_block - 1) / A.rows_per_block);
}

cudaError_t launch_sum_partials(const double* part, int n, double* out, cudaStream_t st) {
    sum_partials_kernel<<<1, 256, 0, st>>>(part, n, out);
    return cudaGetLastError();
}
#endif

}  // namespace hsgn_dev
