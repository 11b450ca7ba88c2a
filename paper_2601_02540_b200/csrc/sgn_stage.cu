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
//   * a CTA owns a BX-column tile and marches down a strip of rows;
//   * each thread owns one column: stage inputs of the NEXT row are loaded
//     into registers one row ahead (software pipelining), pointwise products
//     are formed once per node and parked in a 3-row shared-memory ring
//     (x-neighbours are read from there), while the y-neighbours live in a
//     register rolling window (prev / next row of the 12 y-quantities);
//   * the two halo columns of the tile are fetched with cp.async (LDGSTS)
//     straight into shared memory one row ahead, so no register is spent on
//     them;
//   * bounded (wall) directions use the same arithmetic form with clamped
//     neighbours and the closure coefficient 1/dx (see sbp_d), plus the SAT
//     face term; periodic x wraps by index, periodic y wraps or reads ghost
//     rows written by the slab halo exchange.
#include <cuda_runtime.h>

#include <cstdint>

#include "sgn_device.cuh"

namespace hsgn_dev {

constexpr int BX = 128;   // columns per CTA tile == threads per CTA
constexpr int SW = BX + 2;  // smem row width incl. 2 halo columns

struct Raw {              // raw stage-input data at one node
    double y[5];
    double k[5];
    double kc[5];         // S2 only: k1 (for the fused ynew)
    double b;
};

struct YQ {               // y-differentiated quantities at one node (rhs.hpp:127-137 + b)
    double h, u, v, w, e, hhb, v2, hv, huv, e2h, hvw, b;
};

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Memory row index of logical row jr (may be -1 or ny) of the slab.
__device__ __forceinline__ int map_row(const StageArgs& A, int jr) {
    if (jr < 0) return A.y_lo == YE_WRAP ? A.ny - 1 : (A.y_lo == YE_CLAMP ? 0 : -1);
    if (jr >= A.ny) return A.y_hi == YE_WRAP ? 0 : (A.y_hi == YE_CLAMP ? A.ny - 1 : A.ny);
    return jr;
}

template <int MODE>
__device__ __forceinline__ void load_raw(const StageArgs& A, long long off, Raw& r) {
#pragma unroll
    for (int f = 0; f < 5; ++f) r.y[f] = __ldg(A.y + f * A.fs + off);
    if (MODE == MODE_S1 || MODE == MODE_S2) {
#pragma unroll
        for (int f = 0; f < 5; ++f) r.k[f] = __ldg(A.k + f * A.fs + off);
    }
    if (MODE == MODE_S2) {
#pragma unroll
        for (int f = 0; f < 5; ++f) r.kc[f] = __ldg(A.kc + f * A.fs + off);
    }
    r.b = __ldg(A.b + off);
}

// Stage input q = y + a*k (state_add1, time_integration.hpp:61-75).
template <int MODE>
__device__ __forceinline__ void stage_input(const StageArgs& A, const Raw& r, double q[5]) {
#pragma unroll
    for (int f = 0; f < 5; ++f)
        q[f] = (MODE == MODE_S1 || MODE == MODE_S2) ? dadd(r.y[f], dmul(A.a, r.k[f])) : r.y[f];
}

// Pointwise products of rhs.hpp:99-109.  Writes the 12 x-quantities (and the
// centre extras when `centre`) to smem column `col` of ring slot `S`, and
// fills the y-quantities.  Returns false when !(h > 0).
__device__ __forceinline__ bool products(const double q[5], double b, double* S, int col, bool store,
                                         bool centre, YQ& Y) {
    const double h = q[0], u = q[1], v = q[2], w = q[3], e = q[4];
    const bool ok = h > 0.0;
    const double rh = __drcp_rn(h);
    const double r = div_by(e, h, rh);
    const double hu = dmul(h, u);
    const double hv = dmul(h, v);
    const double huv = dmul(hu, v);  // (h*u)*v
    const double u2 = dmul(u, u);
    const double v2 = dmul(v, v);
    const double hhb = dmul(h, dadd(h, b));
    const double e2h = dmul(e, r);
    const double huw = dmul(hu, w);
    const double hvw = dmul(hv, w);
    if (store) {
    S[XH * SW + col] = h;
    S[XU * SW + col] = u;
    S[XV * SW + col] = v;
    S[XW * SW + col] = w;
    S[XE * SW + col] = e;
    S[XHHB * SW + col] = hhb;
    S[XU2 * SW + col] = u2;
    S[XHU * SW + col] = hu;
    S[XHUV * SW + col] = huv;
    S[XE2H * SW + col] = e2h;
    S[XHUW * SW + col] = huw;
    S[XB * SW + col] = b;
    if (centre) {
        S[CR * SW + col] = r;
        S[CRH * SW + col] = rh;
    }
    }
    Y.h = h; Y.u = u; Y.v = v; Y.w = w; Y.e = e; Y.hhb = hhb;
    Y.v2 = v2; Y.hv = hv; Y.huv = huv; Y.e2h = e2h; Y.hvw = hvw; Y.b = b;
    return ok;
}

// Manufactured source terms S(t, x, y) (scenarios.hpp:179-217 forcing; the
// closed form restated in DESIGN.md section 5 and oracle/hsgn_oracle.c).
__device__ void mms_source(double t, double x, double y, double g, double s[5]) {
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

template <int MODE, bool POW2>
__global__ void __launch_bounds__(BX, 3) sgn_stage_kernel(const StageArgs A) {
    extern __shared__ __align__(16) double dyn_smem[];
#define RING(k) (dyn_smem + (k) * (NSMEM * SW))
    __shared__ __align__(16) double halo_raw[2][2][11];  // [slot][left/right][fields]
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
    const int i0 = blockIdx.x * BX;
    const int i = i0 + tid;
    const bool active = i < nx;
    const int ic = active ? i : nx - 1;  // idle lanes load a valid column
    const int width = min(BX, nx - i0);
    const int j0 = blockIdx.y * A.rows_per_block;
    const int j1 = min(ny, j0 + A.rows_per_block);
    const long long pitch = nx;

    // x-stencil of this column: interior, or the clamped SBP closure row
    const bool xl = A.x_bounded && i == 0;
    const bool xr = A.x_bounded && i == nx - 1;
    const double cx = (xl || xr) ? A.c1x : A.cpx;
    const int sl = xl ? tid + 1 : tid;      // smem column of aL
    const int sr = xr ? tid + 1 : tid + 2;  // smem column of aR
    // halo columns of the tile: thread 0 -> left (smem col 0), thread 32 -> right
    const int halo_side = (tid == 0) ? 0 : ((tid == 32) ? 1 : -1);
    const bool halo_live = halo_side == 0 ? (i0 > 0 || !A.x_bounded)
                                          : (halo_side == 1 ? (i0 + width < nx || !A.x_bounded) : false);
    const int halo_i = halo_side == 0 ? (i0 > 0 ? i0 - 1 : nx - 1) : (i0 + width < nx ? i0 + width : 0);
    const int halo_scol = halo_side == 0 ? 0 : width + 1;
    const bool clamp_lo = A.y_lo == YE_CLAMP, clamp_hi = A.y_hi == YE_CLAMP;

    unsigned long long bad = 0;
    unsigned long long my_min = ~0ull;
    double my_err = 0.0;

    auto halo_fetch = [&](int jr, int hs) {  // async copy of the halo node's raw inputs
        if (halo_live) {
            const long long off = (long long)map_row(A, jr) * pitch + halo_i;
            double* d = halo_raw[hs][halo_side];
#pragma unroll
            for (int f = 0; f < 5; ++f) cp_async8(d + f, A.y + f * A.fs + off);
            if (MODE == MODE_S1 || MODE == MODE_S2) {
#pragma unroll
                for (int f = 0; f < 5; ++f) cp_async8(d + 5 + f, A.k + f * A.fs + off);
            }
            cp_async8(d + 10, A.b + off);
        }
        cp_async_commit();
    };
    auto halo_products = [&](int hs, double* S) {
        if (halo_live) {
            const double* d = halo_raw[hs][halo_side];
            Raw hr;
#pragma unroll
            for (int f = 0; f < 5; ++f) {
                hr.y[f] = d[f];
                hr.k[f] = d[5 + f];
            }
            hr.b = d[10];
            double q[5];
            stage_input<MODE>(A, hr, q);
            YQ unused;
            products(q, hr.b, S, halo_scol, true, false, unused);
        }
    };
    // S2: the part of ynew (and of the adaptive error partial) that does not
    // depend on k3 is formed when the node's raw data is in registers.
    auto centre_extras = [&](const Raw& r, double* S) {
        if (MODE == MODE_S2 && active) {
#pragma unroll
            for (int f = 0; f < 5; ++f)
                S[(CYP0 + f) * SW + tid + 1] = dadd(dadd(r.y[f], dmul(A.c1, r.kc[f])), dmul(A.c2, r.k[f]));
        }
    };

    // ---- prologue: rows j0-1 (prev, y-quantities only) and j0 (cur) ----------
    YQ yp, yc, yn;
    Raw raw;
    if (halo_side >= 0) halo_fetch(j0, 0);
    if (!(j0 == 0 && clamp_lo)) {
        load_raw<MODE>(A, (long long)map_row(A, j0 - 1) * pitch + ic, raw);
        double q[5];
        stage_input<MODE>(A, raw, q);
        products(q, raw.b, RING(2), tid + 1, false, false, yp);
    }
    load_raw<MODE>(A, (long long)j0 * pitch + ic, raw);
    {
        double q[5];
        stage_input<MODE>(A, raw, q);
        const bool ok = products(q, raw.b, RING(0), tid + 1, active, true, yc);
        if (active && !ok) ++bad;
        centre_extras(raw, RING(0));
    }
    if (j0 == 0 && clamp_lo) yp = yc;
    if (!(j0 + 1 == ny && clamp_hi)) load_raw<MODE>(A, (long long)map_row(A, j0 + 1) * pitch + ic, raw);
    if (halo_side >= 0) {
        cp_async_wait_all();
        halo_products(0, RING(0));
        if (j0 + 1 < j1) halo_fetch(j0 + 1, 1);
    }
    int slot_cur = 0;

    // ---- march down the strip --------------------------------------------
    for (int j = j0; j < j1; ++j) {
        const int jn = j + 1;
        const int slot_next = slot_cur == 2 ? 0 : slot_cur + 1;
        double* Sn = RING(slot_next);
        const bool finish_next = jn < j1;  // will row jn be finished by this CTA?
        if (jn == ny && clamp_hi) {
            yn = yc;
        } else {
            double q[5];
            stage_input<MODE>(A, raw, q);
            const bool ok = products(q, raw.b, Sn, tid + 1, active, finish_next, yn);
            if (active && finish_next && !ok) ++bad;
            if (finish_next) centre_extras(raw, Sn);
        }
        // software pipelining: raw inputs of row jn+1 are in flight during the finish
        if (finish_next && !(jn + 1 == ny && clamp_hi))
            load_raw<MODE>(A, (long long)map_row(A, jn + 1) * pitch + ic, raw);
        if (halo_side >= 0 && finish_next) {
            cp_async_wait_all();
            halo_products((jn - j0) & 1, Sn);
            if (jn + 1 < j1) halo_fetch(jn + 1, (jn + 1 - j0) & 1);
        }
        // One barrier per row: makes row j's products (written one iteration
        // ago, halo included) visible, and orders this iteration's writes to
        // slot_next after the last reads of that slot (two rows ago).
        __syncthreads();

        // ---- finish row j -------------------------------------------------
        const double* S = RING(slot_cur);
        if (active) {
            const double cy = ((j == 0 && clamp_lo) || (j == ny - 1 && clamp_hi)) ? A.c1y : A.cpy;
            const double h = yc.h, u = yc.u, v = yc.v, w = yc.w, b = yc.b;
            const double hv = yc.hv, v2 = yc.v2;
            const int cc = tid + 1;
            const double hu = S[XHU * SW + cc], u2 = S[XU2 * SW + cc];
            const double r = S[CR * SW + cc], rh = S[CRH * SW + cc];
#define DXQ(slot) sbp_d<POW2>(cx, S[(slot) * SW + sl], S[(slot) * SW + sr])
#define DYQ(fld) sbp_d<POW2>(cy, yp.fld, yn.fld)
            const double dh_x = DXQ(XH), du_x = DXQ(XU), dv_x = DXQ(XV);
            const double dh_y = DYQ(h), du_y = DYQ(u), dv_y = DYQ(v);
            const double de_x = DXQ(XE), de_y = DYQ(e);
            const double db_x = DXQ(XB), db_y = DYQ(b);
            const double g = A.g;
            double o[5];
            {  // continuity (rhs.hpp:156-157) + wall SAT (sbp.hpp:272-284)
                const double s =
                    dadd(dadd(dadd(dmul(u, dh_x), dmul(h, du_x)), dmul(v, dh_y)), dmul(h, dv_y));
                double ht = -s;
                if (A.walls) {
                    double sat = 0.0;
                    if (xl) sat = dsub(sat, dmul(A.tdx, hu));
                    if (xr) sat = dadd(sat, dmul(A.tdx, hu));
                    if (j == 0 && A.sat_y_lo) sat = dsub(sat, dmul(A.tdy, hv));
                    if (j == ny - 1 && A.sat_y_hi) sat = dadd(sat, dmul(A.tdy, hv));
                    ht = dadd(ht, sat);
                }
                o[0] = ht;
            }
            const double ghb = dmul(g, dadd(h, b));
            const double ls_rr = dmul(A.lam_sixth, dmul(r, r));
            const double lt_r = dmul(A.lam_third, r);
            const double omr = dsub(1.0, r);
            const double lh_omr = dmul(A.lam_half, omr);
            const double uv = dmul(u, v);
            {  // x-momentum (rhs.hpp:167-175), 0.5 factored out of the two split groups
                const double du2_x = DXQ(XU2), dhu_x = DXQ(XHU), dhuv_y = DYQ(huv);
                const double dhhb_x = DXQ(XHHB), de2h_x = DXQ(XE2H);
                double s = dsub(dmul(g, dhhb_x), dmul(ghb, dh_x));
                s = dadd(s, dmul(0.5, dsub(dadd(dsub(dmul(h, du2_x), dmul(u2, dh_x)), dmul(u, dhu_x)),
                                           dmul(hu, du_x))));
                s = dadd(s, dmul(0.5, dsub(dadd(dsub(dhuv_y, dmul(uv, dh_y)), dmul(hv, du_y)),
                                           dmul(hu, dv_y))));
                s = dadd(s, dadd(dsub(dsub(dadd(dmul(ls_rr, dh_x), dmul(A.lam_third, de_x)),
                                           dmul(lt_r, de_x)),
                                      dmul(A.lam_sixth, de2h_x)),
                                 dmul(lh_omr, db_x)));
                o[1] = div_by(-s, h, rh);
            }
            {  // y-momentum (rhs.hpp:180-188)
                const double dv2_y = DYQ(v2), dhv_y = DYQ(hv), dhuv_x = DXQ(XHUV);
                const double dhhb_y = DYQ(hhb), de2h_y = DYQ(e2h);
                double s = dsub(dmul(g, dhhb_y), dmul(ghb, dh_y));
                s = dadd(s, dmul(0.5, dsub(dadd(dsub(dmul(h, dv2_y), dmul(v2, dh_y)), dmul(v, dhv_y)),
                                           dmul(hv, dv_y))));
                s = dadd(s, dmul(0.5, dsub(dadd(dsub(dhuv_x, dmul(uv, dh_x)), dmul(hu, dv_x)),
                                           dmul(hv, du_x))));
                s = dadd(s, dadd(dsub(dsub(dadd(dmul(ls_rr, dh_y), dmul(A.lam_third, de_y)),
                                           dmul(lt_r, de_y)),
                                      dmul(A.lam_sixth, de2h_y)),
                                 dmul(lh_omr, db_y)));
                o[2] = div_by(-s, h, rh);
            }
            {  // vertical velocity (rhs.hpp:196-200)
                const double dw_x = DXQ(XW), dhuw_x = DXQ(XHUW);
                const double dw_y = DYQ(w), dhvw_y = DYQ(hvw);
                const double hw = dmul(h, w);
                double s = dmul(0.5, dsub(dsub(dadd(dhuw_x, dmul(hu, dw_x)), dmul(dmul(u, w), dh_x)),
                                          dmul(hw, du_x)));
                s = dadd(s, dmul(0.5, dsub(dsub(dadd(dhvw_y, dmul(hv, dw_y)), dmul(dmul(v, w), dh_y)),
                                           dmul(hw, dv_y))));
                o[3] = div_by(dsub(dmul(A.lambda, omr), s), h, rh);
            }
            {  // auxiliary depth (rhs.hpp:206-208)
                const double s = dadd(dadd(dadd(dmul(u, de_x), dmul(v, de_y)), dmul(dmul(1.5, u), db_x)),
                                      dmul(dmul(1.5, v), db_y));
                o[4] = dsub(w, s);
            }
#undef DXQ
#undef DYQ
            if (A.shallow) {  // rhs_shallow_water zeroes the decoupled tendencies
                o[3] = 0.0;
                o[4] = 0.0;
            }
            if (A.source) {  // add_manufactured_sources: after assembly (rhs.hpp:212-213)
                const double xg = dadd(A.x_min, dmul((double)i, A.dx));
                const double yg = dadd(A.y_min, dmul((double)(A.j_global0 + j), A.dy));
                double s5[5];
                mms_source(A.t, xg, yg, A.g, s5);
#pragma unroll
                for (int f = 0; f < 5; ++f) o[f] = dadd(o[f], s5[f]);
            }
            // ---- epilogue
            const long long off = (long long)j * pitch + i;
            if (MODE == MODE_S2) {
#pragma unroll
                for (int f = 0; f < 5; ++f) {  // state_add3: ((y + c1 k1) + c2 k2) + c3 k3
                    const double yn_f = dadd(S[(CYP0 + f) * SW + cc], dmul(A.c3, o[f]));
                    A.out[f * A.fs + off] = yn_f;
                    if (f == 0) {
                        const unsigned long long bits = (unsigned long long)__double_as_longlong(yn_f);
                        my_min = bits < my_min ? bits : my_min;
                    }
                }
                if (A.adaptive) {  // ((d1 k1 + d2 k2) + d3 k3) for the error estimate
#pragma unroll
                    for (int f = 0; f < 5; ++f) {
                        const double k1v = __ldg(A.kc + f * A.fs + off);
                        const double k2v = __ldg(A.k + f * A.fs + off);
                        A.part[f * A.fs + off] =
                            dadd(dadd(dmul(A.d1, k1v), dmul(A.d2, k2v)), dmul(A.d3, o[f]));
                    }
                }
            } else {
#pragma unroll
                for (int f = 0; f < 5; ++f) A.out[f * A.fs + off] = o[f];
                if (MODE == MODE_S3 && A.adaptive) {
                    // error_norm_and_min_h (time_integration.hpp:127-136)
#pragma unroll
                    for (int f = 0; f < 5; ++f) {
                        const double e = dmul(A.dt, dadd(A.part[f * A.fs + off], dmul(A.d4, o[f])));
                        const double ay = fabs(__ldg(A.yold + f * A.fs + off));
                        const double an = fabs(__ldg(A.y + f * A.fs + off));
                        const double scale = dadd(A.atol, dmul(A.rtol, ay < an ? an : ay));
                        const double rq = e / scale;
                        my_err = dadd(my_err, dmul(rq, rq));
                    }
                }
            }
        }
        yp = yc;
        yc = yn;
        slot_cur = slot_next;
    }
    if (halo_side >= 0) cp_async_wait_all();

    // ---- block reductions (fixed order inside the block)
    if (bad) atomicAdd(A.bad, bad);
    const int warp = tid >> 5, lane = tid & 31;
    if (MODE == MODE_S2 && A.minh) {
        const unsigned long long m = warp_min_u64(my_min);
        if (lane == 0) s_min[warp] = m;
        __syncthreads();
        if (tid == 0) {
            unsigned long long mm = s_min[0];
            for (int k = 1; k < BX / 32; ++k) mm = s_min[k] < mm ? s_min[k] : mm;
            if (mm != ~0ull) atomicMin(A.minh, mm);
        }
    }
    if (MODE == MODE_S3 && A.adaptive) {
        const double s = warp_sum(my_err);
        if (lane == 0) s_err[warp] = s;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int k = 0; k < BX / 32; ++k) t = dadd(t, s_err[k]);
            A.err_part[blockIdx.y * gridDim.x + blockIdx.x] = t;
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

constexpr size_t RING_BYTES = sizeof(double) * 3 * NSMEM * SW;

template <int MODE, bool POW2>
static cudaError_t launch_mode(const StageArgs& A, cudaStream_t st) {
    static bool configured = false;  // one-time opt-in above the 48 KB static limit
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(sgn_stage_kernel<MODE, POW2>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RING_BYTES);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    dim3 grid((A.nx + BX - 1) / BX, (A.ny + A.rows_per_block - 1) / A.rows_per_block);
    sgn_stage_kernel<MODE, POW2><<<grid, BX, RING_BYTES, st>>>(A);
    return cudaGetLastError();
}

cudaError_t launch_stage(int mode, const StageArgs& A, cudaStream_t st) {
    if (A.pow2) {
        switch (mode) {
            case MODE_RHS: return launch_mode<MODE_RHS, true>(A, st);
            case MODE_S1: return launch_mode<MODE_S1, true>(A, st);
            case MODE_S2: return launch_mode<MODE_S2, true>(A, st);
            default: return launch_mode<MODE_S3, true>(A, st);
        }
    }
    switch (mode) {
        case MODE_RHS: return launch_mode<MODE_RHS, false>(A, st);
        case MODE_S1: return launch_mode<MODE_S1, false>(A, st);
        case MODE_S2: return launch_mode<MODE_S2, false>(A, st);
        default: return launch_mode<MODE_S3, false>(A, st);
    }
}

int stage_grid_blocks(const StageArgs& A) {
    return ((A.nx + BX - 1) / BX) * ((A.ny + A.rows_per_block - 1) / A.rows_per_block);
}

cudaError_t launch_sum_partials(const double* part, int n, double* out, cudaStream_t st) {
    sum_partials_kernel<<<1, 256, 0, st>>>(part, n, out);
    return cudaGetLastError();
}

}  // namespace hsgn_dev
