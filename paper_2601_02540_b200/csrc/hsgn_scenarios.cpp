// hsgn_scenarios.cpp -- the scenario registry of the reference CLI front end
// (reference scenarios.hpp:18-707), host C++.
//
// A scenario is a domain, physics constants, closed-form initial data
// (bathymetry b, depth h, velocities u, v), optional exact solution and
// manufactured forcing, and default gauges / snapshot times.  make() resolves
// parameters exactly like make_scenario (scenarios.hpp:598-698: same names,
// defaults and error messages); sample() evaluates the initial data at the
// nodes x_min + i dx, y_min + j dy (grid.hpp:24-41).  w and eta are left to
// the device init_auxiliary (model.hpp:93-105), as prepare_run does
// (scenarios.hpp:55-78).
//
// Parity: every closed form below is evaluated with the same IEEE operations
// in the same association as the reference expression it cites, through the
// same libm (glibc) calls, and this file is compiled without FP contraction
// (-ffp-contract=off), so the sampled b, h, u, v are bit-identical to the
// reference's prepare_run (tests/test_scenarios.py).  The one exception is the
// manufactured EXACT solution at t > 0 used by the convergence driver: its w
// is the hand-derived closed form -h (u_x + v_y) + 1.5 (u b_x + v b_y) of
// DESIGN.md section 5, not the generated expression (agreement ~1e-15).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hsgn_b200.h"

namespace {

enum Kind { SOLITON = 0, MANUFACTURED, DINGEMANS, HEAD_ON, WALL_REFLECTION, GAUSSIAN, RIEMANN, FAVRE, STILL, LAKE, NKIND };

const char* const kNames[NKIND] = {"soliton",         "manufactured",      "dingemans", "head_on_collision",
                                   "wall_reflection", "gaussian_obstacle", "riemann",   "favre",
                                   "still_water",     "lake_at_rest"};

// Parameter names and defaults per scenario (scenarios.hpp:616-697).  The
// resolved values are stored in hsgn_scenario.p[] in this order.
struct Param {
    const char* key;
    double def;
};
const std::vector<Param> kParams[NKIND] = {
    {{"h_inf", 1.0}, {"amplitude", 0.2}, {"g", 9.81}, {"center", 0.0}, {"direction", 1.0}, {"axis", 0.0},
     {"half_length", 30.0}, {"lambda", 30000.0}},
    {{"g", 9.81}, {"lambda", 500.0}, {"bounded", 0.0}},
    {{"amplitude", 0.02}, {"wave_period", 2.02}, {"x_offset", 0.0}, {"n_waves", 20.0}, {"g", 9.81},
     {"lambda", 500.0}},
    {{"amplitude_right", 0.01077}, {"amplitude_left", 0.01195}, {"center_right", 0.4}, {"center_left", 1.195},
     {"h_inf", 0.05}, {"g", 9.81}, {"lambda", 500.0}},
    {{"amplitude", 0.075}, {"h_inf", 1.0}, {"g", 9.81}, {"center", -50.0}, {"lambda", 500.0}},
    {{"amplitude", 0.0365}, {"h_inf", 0.2}, {"g", 9.81}, {"bounded", 0.0}, {"lambda", 500.0}},
    {{"h_left", 1.8}, {"h_right", 1.0}, {"g", 9.81}, {"lambda", 500.0}},
    {{"eps", 0.1}, {"h0", 1.0}, {"x0", 0.0}, {"alpha", 1.0}, {"g", 9.81}, {"lambda", 500.0}},
    {{"depth", 1.0}, {"g", 9.81}, {"lambda", 500.0}},
    {{"depth", 1.0}, {"bump_amplitude", 0.1}, {"bump_width", 1.0}, {"g", 9.81}, {"bounded", 0.0},
     {"lambda", 500.0}},
};

// Derived constants kept after the parameters (index NP0 on).
constexpr int NP0 = 10;

// Solitary-wave shape (scenarios.hpp:88-114): kappa and speed from h_inf, A, g.
struct Shape {
    double h_inf, amp, kappa, speed;
};
bool make_shape(double h_inf, double amp, double g, Shape* s) {
    if (!(h_inf > 0.0) || !(amp > 0.0)) return false;
    const double eps = amp / h_inf;
    s->h_inf = h_inf;
    s->amp = amp;
    s->kappa = std::sqrt(3.0 * eps / (4.0 * h_inf * h_inf * (1.0 + eps)));
    s->speed = std::sqrt(g * h_inf * (1.0 + eps));
    return true;
}
double depth_of(const Shape& s, double xi) {
    const double c = 1.0 / std::cosh(s.kappa * xi);
    return s.h_inf + s.amp * c * c;
}
double velocity_of(const Shape& s, double xi) { return s.speed * (1.0 - s.h_inf / depth_of(s, xi)); }

// Newton solve of omega^2 = g k tanh(k d) (scenarios.hpp:223-238).
double wavenumber(double omega, double d, double g) {
    double k = omega / std::sqrt(g * d);
    for (int it = 0; it < 100; ++it) {
        const double th = std::tanh(k * d);
        const double f = g * k * th - omega * omega;
        const double df = g * th + g * k * d * (1.0 - th * th);
        const double step = f / df;
        k -= step;
        if (std::abs(step) <= 1e-15 * k) break;
    }
    return k;
}

// Manufactured bathymetry and initial state (manufactured_generated.hpp:11-38 at t = 0).
double mms_b(double x, double y) {
    const double f4 = 4 * M_PI, f2 = 2 * M_PI;
    return (1.0 / 25.0) * cos(x * f4) * cos(f4 * y) + (2.0 / 25.0) * cos(x * f2) * cos(f2 * y);
}

void set_name(hsgn_scenario* s, const char* n) {
    std::snprintf(s->name, sizeof s->name, "%s", n);
}

Shape shape_at(const hsgn_scenario* s, int k0) {  // stored as h_inf, amp, kappa, speed
    Shape sh;
    sh.h_inf = s->p[k0];
    sh.amp = s->p[k0 + 1];
    sh.kappa = s->p[k0 + 2];
    sh.speed = s->p[k0 + 3];
    return sh;
}
void store_shape(hsgn_scenario* s, int k0, const Shape& sh) {
    s->p[k0] = sh.h_inf;
    s->p[k0 + 1] = sh.amp;
    s->p[k0 + 2] = sh.kappa;
    s->p[k0 + 3] = sh.speed;
}

// Initial data of one node (b, h, u, v) -- the spec lambdas of scenarios.hpp.
void initial(const hsgn_scenario* s, double x, double y, double* b, double* h, double* u, double* v) {
    const double* p = s->p;
    *b = 0.0;
    *u = 0.0;
    *v = 0.0;
    switch (s->kind) {
        case SOLITON: {  // scenarios.hpp:140-152
            const Shape sh = shape_at(s, NP0);
            const double center = p[3], dir = p[NP0 + 4];
            if ((int)p[5] == 0) {
                *h = depth_of(sh, x - center);
                *u = dir * velocity_of(sh, x - center);
            } else {
                *h = depth_of(sh, y - center);
                *v = dir * velocity_of(sh, y - center);
            }
            break;
        }
        case MANUFACTURED: {  // scenarios.hpp:195-199 with exact_state(0, x, y)
            *b = mms_b(x, y);
            const double w2 = 2 * M_PI, w4 = 4 * M_PI;
            const double a1 = x * w2, cx2 = cos(a1), a3 = w2 * y, cy2 = cos(a3);
            const double cx4 = cos(x * w4), cy4 = cos(w4 * y);
            const double sx2 = sin(a1), sy2 = sin(a3);
            const double t0w = 0.0 * w2;
            const double prod = sx2 * sy2 * cos(t0w);
            *h = (1.0 / 2.0) * prod - 2.0 / 25.0 * cx2 * cy2 - 1.0 / 25.0 * cx4 * cy4 + 2;
            const double amp_t = (3.0 / 10.0) * sin(t0w);
            *u = sx2 * amp_t;
            *v = sy2 * amp_t;
            break;
        }
        case DINGEMANS: {  // scenarios.hpp:261-285
            const double amp = p[0], x_off = p[2];
            const double k = p[NP0], c = p[NP0 + 1], wl = p[NP0 + 2], lo = p[NP0 + 3], hi = p[NP0 + 4];
            const double depth = 0.8;
            double bb = 0.0;
            if (x >= 11.01 && x < 23.04)
                bb = 0.6 * (x - 11.01) / 12.03;
            else if (x >= 23.04 && x < 27.04)
                bb = 0.6;
            else if (x >= 27.04 && x < 33.07)
                bb = 0.6 * (33.07 - x) / 6.03;
            double el = 0.0;
            if (!(x <= lo || x >= hi)) {
                double env = 1.0;
                if (x < lo + wl)
                    env = 0.5 * (1.0 - std::cos(M_PI * (x - lo) / wl));
                else if (x > hi - wl)
                    env = 0.5 * (1.0 - std::cos(M_PI * (hi - x) / wl));
                el = amp * env * std::sin(k * (x - x_off));
            }
            *b = bb;
            *h = depth + el - bb;
            *u = c * el / depth;
            break;
        }
        case HEAD_ON: {  // scenarios.hpp:311-319
            const Shape s1 = shape_at(s, NP0), s2 = shape_at(s, NP0 + 4);
            const double ar = p[0], al = p[1], cr = p[2], cl = p[3], h_inf = p[4];
            *h = h_inf + ar * std::pow(1.0 / std::cosh(s1.kappa * (x - cr)), 2) +
                 al * std::pow(1.0 / std::cosh(s2.kappa * (x - cl)), 2);
            const double h1 = depth_of(s1, x - cr), h2 = depth_of(s2, x - cl);
            *u = s1.speed * (1.0 - h_inf / h1) - s2.speed * (1.0 - h_inf / h2);
            break;
        }
        case WALL_REFLECTION: {  // scenarios.hpp:340-341
            const Shape sh = shape_at(s, NP0);
            *h = depth_of(sh, x - p[3]);
            *u = velocity_of(sh, x - p[3]);
            break;
        }
        case GAUSSIAN: {  // scenarios.hpp:373-380
            const Shape sh = shape_at(s, NP0);
            const double bb = 0.1 * std::exp(-0.5 * (x * x + y * y));
            const double c = 1.0 / std::cosh(sh.kappa * (x + 3.0));
            *b = bb;
            *h = p[1] + p[0] * c * c - bb;
            *u = velocity_of(sh, x + 3.0);
            break;
        }
        case RIEMANN:  // scenarios.hpp:402-404
            *h = p[1] + 0.5 * (p[0] - p[1]) * (1.0 - std::tanh(0.5 * x));
            break;
        case FAVRE: {  // scenarios.hpp:455-460
            const double dh = p[NP0], du = p[NP0 + 1], h0 = p[1], x0 = p[2], alpha = p[3];
            *h = h0 + 0.5 * dh * (1.0 - std::tanh((x - x0) / alpha));
            *u = 0.5 * du * (1.0 - std::tanh((x - x0) / alpha));
            break;
        }
        case STILL:  // scenarios.hpp:476
            *h = p[0];
            break;
        case LAKE: {  // scenarios.hpp:494-498
            const double iw2 = p[NP0];
            const double bb = p[1] * std::exp(-0.5 * (x * x + y * y) * iw2);
            *b = bb;
            *h = p[0] - bb;
            break;
        }
    }
}

double node_x(const hsgn_scenario* s, int nx, int i) {
    const hsgn_grid& d = s->domain;
    const double dx = d.kind_x == HSGN_PERIODIC ? (d.x_max - d.x_min) / nx : (d.x_max - d.x_min) / (nx - 1);
    return d.x_min + i * dx;
}
double node_y(const hsgn_scenario* s, int ny, int j) {
    const hsgn_grid& d = s->domain;
    const double dy = d.kind_y == HSGN_PERIODIC ? (d.y_max - d.y_min) / ny : (d.y_max - d.y_min) / (ny - 1);
    return d.y_min + j * dy;
}

void err_msg(char* err, int len, const std::string& m) {
    if (err && len > 0) std::snprintf(err, (size_t)len, "%s", m.c_str());
}

}  // namespace

extern "C" {

int32_t hsgn_scenario_count(void) { return NKIND; }

const char* hsgn_scenario_name(int32_t k) { return (k >= 0 && k < NKIND) ? kNames[k] : nullptr; }

hsgn_status hsgn_scenario_make(const char* name, const char* const* keys, const double* vals, int32_t n,
                               hsgn_scenario* out, char* err, int32_t err_len) {
    if (!name || !out || (n > 0 && (!keys || !vals))) return HSGN_EINVAL;
    int kind = -1;
    for (int k = 0; k < NKIND; ++k)
        if (std::strcmp(name, kNames[k]) == 0) kind = k;
    if (kind < 0) {
        err_msg(err, err_len, std::string("unknown scenario '") + name + "'");
        return HSGN_EINVAL;
    }
    const std::vector<Param>& P = kParams[kind];
    hsgn_scenario s;
    std::memset(&s, 0, sizeof s);
    s.kind = kind;
    for (size_t k = 0; k < P.size(); ++k) s.p[k] = P[k].def;
    for (int a = 0; a < n; ++a) {  // check_keys (scenarios.hpp:604-615); the last value of a key wins
        size_t k = 0;
        while (k < P.size() && std::strcmp(keys[a], P[k].key) != 0) ++k;
        if (k == P.size()) {
            err_msg(err, err_len, std::string("scenario '") + name + "': unknown parameter '" + keys[a] + "'");
            return HSGN_EINVAL;
        }
        s.p[k] = vals[a];
    }
    // ScenarioSpec defaults (scenarios.hpp:21-46)
    s.domain.x_min = 0.0;
    s.domain.x_max = 1.0;
    s.domain.y_min = 0.0;
    s.domain.y_max = 1.0;
    s.domain.nx = 64;
    s.domain.ny = 64;
    s.domain.kind_x = HSGN_PERIODIC;
    s.domain.kind_y = HSGN_PERIODIC;
    s.g = 9.81;
    s.lambda = 500.0;
    s.t0 = 0.0;
    s.t_final = 1.0;
    auto square = [&](double lo, double hi) {
        s.domain.x_min = lo;
        s.domain.x_max = hi;
        s.domain.y_min = lo;
        s.domain.y_max = hi;
    };
    auto shape_or_fail = [&](double h_inf, double amp, double g, Shape* sh) {
        if (make_shape(h_inf, amp, g, sh)) return true;
        err_msg(err, err_len, "soliton_shape: need h_inf > 0 and amplitude > 0");
        return false;
    };
    const double* p = s.p;
    switch (kind) {
        case SOLITON: {  // scenarios.hpp:123-172, 616-626
            Shape sh;
            if (!shape_or_fail(p[0], p[1], p[2], &sh)) return HSGN_EINVAL;
            store_shape(&s, NP0, sh);
            const int direction = (int)p[4], axis = (int)p[5];
            s.p[4] = direction;
            s.p[5] = axis;
            s.p[NP0 + 4] = direction >= 0 ? 1.0 : -1.0;
            square(-p[6], p[6]);
            s.g = p[2];
            s.lambda = p[7];
            s.t_final = 2.0 * p[6] / sh.speed;
            s.domain.nx = axis == 0 ? 200 : 4;
            s.domain.ny = axis == 0 ? 4 : 200;
            s.has_exact = 1;
            s.n_exact_vars = 2;
            s.exact_vars[0] = 0;
            s.exact_vars[1] = axis == 0 ? 1 : 2;
            break;
        }
        case MANUFACTURED: {  // scenarios.hpp:179-217, 627-632
            square(-1.0, 1.0);
            const int kb = p[2] != 0.0 ? HSGN_BOUNDED : HSGN_PERIODIC;
            s.domain.kind_x = kb;
            s.domain.kind_y = kb;
            s.g = p[0];
            s.lambda = p[1];
            s.has_source = 1;
            s.has_exact = 1;
            s.n_exact_vars = 5;
            for (int f = 0; f < 5; ++f) s.exact_vars[f] = f;
            break;
        }
        case DINGEMANS: {  // scenarios.hpp:240-287
            const double omega = 2.0 * M_PI / p[1];
            const double k = wavenumber(omega, 0.8, p[4]);
            const double wl = 2.0 * M_PI / k;
            s.p[NP0] = k;
            s.p[NP0 + 1] = omega / k;
            s.p[NP0 + 2] = wl;
            s.p[NP0 + 3] = p[2] - p[3] * wl;
            s.p[NP0 + 4] = p[2];
            s.domain.x_min = -138.0;
            s.domain.x_max = 46.0;
            s.domain.y_min = -138.0;
            s.domain.y_max = 46.0;
            s.domain.nx = 3680;
            s.domain.ny = 4;
            s.g = p[4];
            s.lambda = p[5];
            s.t_final = 60.0;
            const double gx[6] = {3.04, 9.44, 20.04, 26.04, 30.44, 37.04};
            s.n_gauges = 6;
            for (int q = 0; q < 6; ++q) {
                s.gauges[q][0] = gx[q];
                s.gauges[q][1] = -46.0;
            }
            break;
        }
        case HEAD_ON: {  // scenarios.hpp:293-321
            Shape s1, s2;
            if (!shape_or_fail(p[4], p[0], p[5], &s1) || !shape_or_fail(p[4], p[1], p[5], &s2)) return HSGN_EINVAL;
            store_shape(&s, NP0, s1);
            store_shape(&s, NP0 + 4, s2);
            square(-10.0, 10.0);
            s.domain.nx = 400;
            s.domain.ny = 4;
            s.g = p[5];
            s.lambda = p[6];
            s.t0 = 18.5;
            s.t_final = 21.5;
            break;
        }
        case WALL_REFLECTION: {  // scenarios.hpp:325-352
            Shape sh;
            if (!shape_or_fail(p[1], p[0], p[2], &sh)) return HSGN_EINVAL;
            store_shape(&s, NP0, sh);
            s.domain.x_min = -100.0;
            s.domain.x_max = 0.0;
            s.domain.y_min = -50.0;
            s.domain.y_max = 50.0;
            s.domain.nx = 501;
            s.domain.ny = 4;
            s.domain.kind_x = HSGN_BOUNDED;
            s.g = p[2];
            s.lambda = p[4];
            s.t_final = 110.0 / sh.speed;
            const double scale = std::sqrt(p[1] / p[2]);
            static const double ts_a[5] = {24.0, 45.0, 48.0, 53.0, 90.0};
            static const double ts_b[5] = {0.0, 28.0, 38.0, 42.0, 70.0};
            const double* ts = std::abs(p[0] - 0.075) < 1e-12 ? ts_a : std::abs(p[0] - 0.65) < 1e-12 ? ts_b : nullptr;
            if (ts) {
                s.n_snapshots = 5;
                for (int q = 0; q < 5; ++q) s.snapshot_times[q] = ts[q] * scale;
            }
            s.n_gauges = 1;  // {0, 0}
            break;
        }
        case GAUSSIAN: {  // scenarios.hpp:356-383
            Shape sh;
            if (!shape_or_fail(p[1], p[0], p[2], &sh)) return HSGN_EINVAL;
            store_shape(&s, NP0, sh);
            const bool bounded = p[3] != 0.0;
            s.domain.x_min = -5.0;
            s.domain.x_max = 35.0;
            s.domain.y_min = -10.0;
            s.domain.y_max = 10.0;
            s.domain.nx = bounded ? 201 : 200;
            s.domain.ny = bounded ? 101 : 100;
            s.domain.kind_x = bounded ? HSGN_BOUNDED : HSGN_PERIODIC;
            s.domain.kind_y = s.domain.kind_x;
            s.g = p[2];
            s.lambda = p[4];
            s.t_final = 12.0;
            s.n_snapshots = 1;
            s.snapshot_times[0] = 12.0;
            break;
        }
        case RIEMANN:  // scenarios.hpp:389-408
            square(-600.0, 600.0);
            s.domain.nx = 2001;
            s.domain.ny = 4;
            s.domain.kind_x = HSGN_BOUNDED;
            s.g = p[2];
            s.lambda = p[3];
            s.t_final = 47.434;
            s.n_snapshots = 1;
            s.snapshot_times[0] = 47.434;
            break;
        case FAVRE: {  // scenarios.hpp:438-462
            const double dh = p[0] * p[1];
            const double h1 = p[1] + dh;
            s.p[NP0] = dh;
            s.p[NP0 + 1] = std::sqrt(p[4] * (h1 + p[1]) / (2.0 * p[1] * h1)) * dh;
            square(-150.0, 150.0);
            s.domain.nx = 1000;
            s.domain.ny = 4;
            s.g = p[4];
            s.lambda = p[5];
            s.t_final = 30.0;
            break;
        }
        case STILL:  // scenarios.hpp:465-477
            square(-5.0, 5.0);
            s.g = p[1];
            s.lambda = p[2];
            s.t_final = 10.0;
            break;
        case LAKE: {  // scenarios.hpp:480-500
            square(-5.0, 5.0);
            const bool bounded = p[4] != 0.0;
            s.domain.kind_x = bounded ? HSGN_BOUNDED : HSGN_PERIODIC;
            s.domain.kind_y = s.domain.kind_x;
            s.g = p[3];
            s.lambda = p[5];
            s.t_final = 10.0;
            s.p[NP0] = 1.0 / (p[2] * p[2]);
            break;
        }
    }
    set_name(&s, kNames[kind]);
    *out = s;
    return HSGN_OK;
}

hsgn_status hsgn_scenario_sample(const hsgn_scenario* s, int32_t nx, int32_t ny, double* b, double* q) {
    return hsgn_scenario_sample_rows(s, nx, ny, 0, ny, b, q);
}

hsgn_status hsgn_scenario_sample_rows(const hsgn_scenario* s, int32_t nx, int32_t ny, int32_t j0, int32_t j1,
                                      double* b, double* q) {
    if (!s || !b || !q || s->kind < 0 || s->kind >= NKIND || nx < 4 || ny < 4 || j0 < 0 || j1 > ny || j1 <= j0)
        return HSGN_EINVAL;
    const size_t n = (size_t)nx * (size_t)(j1 - j0);
    std::vector<double> xs(nx);
    for (int i = 0; i < nx; ++i) xs[i] = node_x(s, nx, i);
    for (int j = j0; j < j1; ++j) {
        const double y = node_y(s, ny, j);
        for (int i = 0; i < nx; ++i) {
            const size_t k = (size_t)(j - j0) * nx + i;
            initial(s, xs[i], y, &b[k], &q[k], &q[n + k], &q[2 * n + k]);
            q[3 * n + k] = 0.0;  // w, eta: init_auxiliary (model.hpp:93-105)
            q[4 * n + k] = 0.0;
        }
    }
    return HSGN_OK;
}

hsgn_status hsgn_scenario_eval(const hsgn_scenario* s, double x, double y, double* bhuv) {
    if (!s || !bhuv || s->kind < 0 || s->kind >= NKIND) return HSGN_EINVAL;
    initial(s, x, y, &bhuv[0], &bhuv[1], &bhuv[2], &bhuv[3]);  // the spec's b, h0, u0, v0 at (x, y)
    return HSGN_OK;
}

hsgn_status hsgn_scenario_exact(const hsgn_scenario* s, int32_t nx, int32_t ny, double t, double* q) {
    if (!s || !q || !s->has_exact || nx < 4 || ny < 4) return HSGN_EINVAL;
    const size_t n = (size_t)nx * (size_t)ny;
    for (int j = 0; j < ny; ++j) {
        const double y = node_y(s, ny, j);
        for (int i = 0; i < nx; ++i) {
            const double x = node_x(s, nx, i);
            const size_t k = (size_t)j * nx + i;
            double h, u = 0.0, v = 0.0, w = 0.0;
            if (s->kind == SOLITON) {  // scenarios.hpp:155-170
                const Shape sh = shape_at(s, NP0);
                const double L = 2.0 * s->p[6], dir = s->p[NP0 + 4];
                const int axis = (int)s->p[5];
                const double pos = axis == 0 ? x : y;
                double xi = pos - s->p[3] - dir * sh.speed * t;
                xi = xi - L * std::round(xi / L);
                h = depth_of(sh, xi);
                const double vel = dir * sh.speed * (1.0 - sh.h_inf / h);
                (axis == 0 ? u : v) = vel;
            } else {  // manufactured exact state (hand-derived closed form)
                const double tp = 2.0 * M_PI, fp = 4.0 * M_PI;
                const double s1x = std::sin(tp * x), c1x = std::cos(tp * x), s2x = std::sin(fp * x),
                             c2x = std::cos(fp * x);
                const double s1y = std::sin(tp * y), c1y = std::cos(tp * y), s2y = std::sin(fp * y),
                             c2y = std::cos(fp * y);
                const double st = std::sin(tp * t), ct = std::cos(tp * t);
                const double bb = (2.0 / 25.0) * c1x * c1y + (1.0 / 25.0) * c2x * c2y;
                const double bx = -(2.0 / 25.0) * tp * s1x * c1y - (1.0 / 25.0) * fp * s2x * c2y;
                const double by = -(2.0 / 25.0) * tp * c1x * s1y - (1.0 / 25.0) * fp * c2x * s2y;
                h = 2.0 + 0.5 * s1x * s1y * ct - bb;
                u = 0.3 * s1x * st;
                v = 0.3 * s1y * st;
                const double ux = 0.3 * tp * c1x * st, vy = 0.3 * tp * c1y * st;
                w = -h * (ux + vy) + 1.5 * (u * bx + v * by);
            }
            q[k] = h;
            q[n + k] = u;
            q[2 * n + k] = v;
            q[3 * n + k] = w;
            q[4 * n + k] = h;
        }
    }
    return HSGN_OK;
}

}  // extern "C"
