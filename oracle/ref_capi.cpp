// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY (the "oracle/_ref" checker).
//
// A thin extern "C" adapter that compiles the UNMODIFIED reference headers
// in place (-I /root/reference/proj/include, see oracle/Makefile) so tests
// and the CPU baseline can call the reference's own hot path on identical
// inputs.  No reference source is copied into this repository; every call
// below forwards to the reference symbol cited next to it.
//
// Built only when /root/reference exists (this container); the resulting
// oracle/_ref/libhsgn_ref.so is git-ignored and travels to the GPU box as a
// prebuilt file.  Never linked by the product library.

#include <random>
#include <hsgn/analysis.hpp>
#include <hsgn/config.hpp>
#include <hsgn/io.hpp>
#include <hsgn/manufactured_generated.hpp>
#include <hsgn/model.hpp>
#include <hsgn/rhs.hpp>
#include <hsgn/sbp.hpp>
#include <hsgn/scenarios.hpp>
#include <hsgn/threading.hpp>
#include <hsgn/time_integration.hpp>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <sstream>
#include <string>

#include "oracle_abi.h"

using namespace hsgn;

namespace {

BoundaryKind kind_of(int k) { return k ? BoundaryKind::bounded : BoundaryKind::periodic; }

Grid2D grid_of(const orc_grid* g) {
    return make_grid(g->x_min, g->x_max, g->y_min, g->y_max, g->nx, g->ny,
                     kind_of(g->kind_x), kind_of(g->kind_y));  // grid.hpp:47-68
}

void to_state(const double* q, StateField& s) {
    auto f = s.fields();
    const std::size_t n = f[0]->size();
    for (int k = 0; k < StateField::n_fields; ++k)
        std::memcpy(f[k]->data(), q + k * n, n * sizeof(double));
}

void from_state(const StateField& s, double* q) {
    auto f = s.fields();
    const std::size_t n = f[0]->size();
    for (int k = 0; k < StateField::n_fields; ++k)
        std::memcpy(q + k * n, f[k]->data(), n * sizeof(double));
}

Field2D field_of(const Grid2D& g, const double* p) {
    Field2D f(g.nx, g.ny);
    std::memcpy(f.data(), p, f.size() * sizeof(double));
    return f;
}

RhsContext context_of(const Grid2D& grid, const orc_phys* phys, const double* b, int source_kind) {
    PhysSetup ps;
    ps.g = phys->g;
    ps.lambda = phys->lambda;
    ps.h_floor = phys->h_floor;
    ps.b = field_of(grid, b);
    RhsContext ctx = make_rhs_context(grid, ps);  // rhs.hpp:40-54
    if (source_kind == 1) {
        const double gg = phys->g;
        ctx.source = [grid, gg](double t, StateField& tend) {
            add_manufactured_sources(tend, t, grid, [gg](double tt, double x, double y) {
                return manufactured::source_terms(tt, x, y, gg);  // manufactured_generated.hpp:69
            });
        };
    }
    return ctx;
}

IntegratorConfig cfg_of(const orc_cfg* c) {
    IntegratorConfig cfg;
    cfg.abs_tol = c->abs_tol;
    cfg.rel_tol = c->rel_tol;
    cfg.dt_initial = c->dt_initial;
    cfg.dt_max = c->dt_max;
    cfg.safety = c->safety;
    cfg.growth_cap = c->growth_cap;
    cfg.shrink_floor = c->shrink_floor;
    cfg.max_steps = c->max_steps;
    cfg.fixed_dt = c->fixed_dt;
    cfg.h_floor = c->h_floor;
    return cfg;
}

}  // namespace

extern "C" {

void ref_set_threads(int n) { set_thread_count(n); }  // threading.hpp:12

// The 300 random states of acceptance gate c2 (acceptance_main.cpp:88-127),
// drawn exactly as the gate draws them: one std::mt19937(20260822) stream,
// pos = U(0.5, 1.5), sym = U(-1, 1), per setup and trial the fields h (pos),
// u, v, w (sym), eta (pos) of a 32 x 32 grid in storage order (libstdc++
// streams, so the device tests get the reference's own inputs).
// out: n_setups * trials * 5 * 1024 doubles.
void ref_c2_states(int n_setups, int trials, double* out) {
    std::mt19937 rng(20260822u);
    std::uniform_real_distribution<double> pos(0.5, 1.5), sym(-1.0, 1.0);
    const int n = 32 * 32;
    for (int s = 0; s < n_setups; ++s)
        for (int t = 0; t < trials; ++t)
            for (int f = 0; f < 5; ++f) {
                const bool positive = f == 0 || f == 4;
                for (int k = 0; k < n; ++k) *out++ = positive ? pos(rng) : sym(rng);
            }
}
int ref_max_threads(void) { return max_thread_count(); }

void ref_default_cfg(orc_cfg* c) {
    IntegratorConfig d;  // time_integration.hpp:18-29 defaults
    c->abs_tol = d.abs_tol;
    c->rel_tol = d.rel_tol;
    c->dt_initial = d.dt_initial;
    c->dt_max = d.dt_max;
    c->safety = d.safety;
    c->growth_cap = d.growth_cap;
    c->shrink_floor = d.shrink_floor;
    c->max_steps = d.max_steps;
    c->fixed_dt = d.fixed_dt;
    c->h_floor = d.h_floor;
}

// rhs.hpp:236 (variant 0) / rhs.hpp:243 rhs_shallow_water (variant 1).
// Returns 0, or 1 when depth_error is thrown (out untouched).
int ref_rhs(const orc_grid* g, const orc_phys* phys, const double* b, int source_kind,
            int variant, double t, const double* q, double* out, int64_t* n_evals) {
    Grid2D grid = grid_of(g);
    RhsContext ctx = context_of(grid, phys, b, source_kind);
    StateField qs(grid), os(grid);
    to_state(q, qs);
    to_state(out, os);
    try {
        if (variant == 1)
            rhs_shallow_water(ctx, t, qs, os);
        else
            rhs(ctx, t, qs, os);
    } catch (const depth_error&) {
        return 1;
    }
    from_state(os, out);
    if (n_evals)
        *n_evals = ctx.n_evals;
    return 0;
}

// Repeats rhs() `reps` times on one context (cli.hpp:252-260 bench loop);
// used by the CPU baseline timing.  Returns depth status of the last call.
int ref_rhs_repeat(const orc_grid* g, const orc_phys* phys, const double* b, double t,
                   const double* q, double* out, int reps) {
    Grid2D grid = grid_of(g);
    RhsContext ctx = context_of(grid, phys, b, 0);
    StateField qs(grid), os(grid);
    to_state(q, qs);
    try {
        for (int r = 0; r < reps; ++r)
            rhs(ctx, t, qs, os);
    } catch (const depth_error&) {
        return 1;
    }
    from_state(os, out);
    return 0;
}

// adaptive_solve (time_integration.hpp:209-350) with the RHS of rhs.hpp:236.
// history (nullable): per AcceptObserver call (time_integration.hpp:255,335)
// writes (t, total_mass, total_energy, energy_rate) while n < hist_cap.
int ref_solve(const orc_grid* g, const orc_phys* phys, const double* b, int source_kind,
              const double* q0, double t0, double t_final, const orc_cfg* c, double* q_out,
              orc_record* rec_out, double* history, int64_t hist_cap, int64_t* hist_n) {
    Grid2D grid = grid_of(g);
    RhsContext ctx = context_of(grid, phys, b, source_kind);
    StateField qs(grid);
    to_state(q0, qs);
    IntegratorConfig cfg = cfg_of(c);
    int64_t nh = 0;
    AcceptObserver obs;
    if (history) {
        obs = [&](double t, const StateField& q, const StateField& qt) {
            if (nh < hist_cap) {
                double* row = history + 4 * nh;
                row[0] = t;
                row[1] = total_mass(ctx.op_x.mass, ctx.op_y.mass, q);
                row[2] = total_energy(ctx.op_x.mass, ctx.op_y.mass, q, ctx.phys);
                row[3] = energy_rate(ctx.op_x.mass, ctx.op_y.mass, q, qt, ctx.phys);
            }
            ++nh;
        };
    }
    SolutionRecord rec = adaptive_solve(
        [&ctx](double t, const StateField& q, StateField& out) { rhs(ctx, t, q, out); }, qs,
        t0, t_final, cfg, obs);
    from_state(rec.q, q_out);
    rec_out->t = rec.t;
    rec_out->accepted = rec.accepted;
    rec_out->rejected = rec.rejected;
    rec_out->rhs_evals = rec.rhs_evals;
    rec_out->rhs_evals_setup = rec.rhs_evals_setup;
    rec_out->aborted = rec.aborted ? 1 : 0;
    std::snprintf(rec_out->reason, sizeof rec_out->reason, "%s", rec.abort_reason.c_str());
    if (hist_n)
        *hist_n = nh;
    return rec.aborted ? 1 : 0;
}

// cmd_run's recorder wiring (cli.hpp:100-116): adaptive_solve with
// RunRecorder::on_accept as the observer, then flush() -- the reference
// writes gauges.csv, conservation.csv and snapshot_t*.csv into out_dir.
int ref_run_recorded(const orc_grid* g, const orc_phys* phys, const double* b, int source_kind,
                     const double* q0, double t0, double t_final, const orc_cfg* c, double* q_out,
                     orc_record* rec_out, const char* out_dir, int n_gauges, const double* gauge_xy,
                     int n_targets, const double* targets, int64_t stride) {
    Grid2D grid = grid_of(g);
    RhsContext ctx = context_of(grid, phys, b, source_kind);
    StateField qs(grid);
    to_state(q0, qs);
    std::vector<std::array<double, 2>> gauges;
    for (int k = 0; k < n_gauges; ++k) gauges.push_back({gauge_xy[2 * k], gauge_xy[2 * k + 1]});
    std::vector<double> tg(targets, targets + n_targets);
    std::filesystem::create_directories(out_dir);  // as cmd_run does (cli.hpp:93)
    RunRecorder recorder(ctx, out_dir, gauges, tg, stride);  // io.hpp:109-118
    SolutionRecord rec = adaptive_solve(
        [&ctx](double t, const StateField& q, StateField& out) { rhs(ctx, t, q, out); }, qs, t0,
        t_final, cfg_of(c),
        [&recorder](double t, const StateField& q, const StateField& qt) { recorder.on_accept(t, q, qt); });
    recorder.flush();  // io.hpp:155-185
    from_state(rec.q, q_out);
    rec_out->t = rec.t;
    rec_out->accepted = rec.accepted;
    rec_out->rejected = rec.rejected;
    rec_out->rhs_evals = rec.rhs_evals;
    rec_out->rhs_evals_setup = rec.rhs_evals_setup;
    rec_out->aborted = rec.aborted ? 1 : 0;
    std::snprintf(rec_out->reason, sizeof rec_out->reason, "%s", rec.abort_reason.c_str());
    return rec.aborted ? 1 : 0;
}

void ref_init_auxiliary(const orc_grid* g, const double* b, double* q) {
    Grid2D grid = grid_of(g);
    StateField qs(grid);
    to_state(q, qs);
    SbpOperator1D ox = build_d1(grid.kind_x, grid.nx, grid.dx);
    SbpOperator1D oy = build_d1(grid.kind_y, grid.ny, grid.dy);
    init_auxiliary(qs, ox, oy, field_of(grid, b));  // model.hpp:93-105
    from_state(qs, q);
}

double ref_total_mass(const orc_grid* g, const double* q) {
    Grid2D grid = grid_of(g);
    StateField qs(grid);
    to_state(q, qs);
    SbpOperator1D ox = build_d1(grid.kind_x, grid.nx, grid.dx);
    SbpOperator1D oy = build_d1(grid.kind_y, grid.ny, grid.dy);
    return total_mass(ox.mass, oy.mass, qs);  // model.hpp:77-80
}

double ref_total_energy(const orc_grid* g, const orc_phys* phys, const double* b,
                        const double* q) {
    Grid2D grid = grid_of(g);
    StateField qs(grid);
    to_state(q, qs);
    SbpOperator1D ox = build_d1(grid.kind_x, grid.nx, grid.dx);
    SbpOperator1D oy = build_d1(grid.kind_y, grid.ny, grid.dy);
    PhysSetup ps;
    ps.g = phys->g;
    ps.lambda = phys->lambda;
    ps.b = field_of(grid, b);
    return total_energy(ox.mass, oy.mass, qs, ps);  // model.hpp:82-87
}

double ref_energy_rate(const orc_grid* g, const orc_phys* phys, const double* b,
                       const double* q, const double* qt) {
    Grid2D grid = grid_of(g);
    StateField qs(grid), ts(grid);
    to_state(q, qs);
    to_state(qt, ts);
    SbpOperator1D ox = build_d1(grid.kind_x, grid.nx, grid.dx);
    SbpOperator1D oy = build_d1(grid.kind_y, grid.ny, grid.dy);
    PhysSetup ps;
    ps.g = phys->g;
    ps.lambda = phys->lambda;
    ps.b = field_of(grid, b);
    return energy_rate(ox.mass, oy.mass, qs, ts, ps);  // analysis.hpp:47-67
}

double ref_mass_weighted_sum(const orc_grid* g, const double* f) {
    Grid2D grid = grid_of(g);
    SbpOperator1D ox = build_d1(grid.kind_x, grid.nx, grid.dx);
    SbpOperator1D oy = build_d1(grid.kind_y, grid.ny, grid.dy);
    return mass_weighted_sum(ox.mass, oy.mass, field_of(grid, f));  // sbp.hpp:219-239
}

double ref_discrete_l2_error(const orc_grid* g, const double* a, const double* bb) {
    Grid2D grid = grid_of(g);
    SbpOperator1D ox = build_d1(grid.kind_x, grid.nx, grid.dx);
    SbpOperator1D oy = build_d1(grid.kind_y, grid.ny, grid.dy);
    return discrete_l2_error(ox.mass, oy.mass, field_of(grid, a), field_of(grid, bb));
}

// apply_dx / apply_dy (sbp.hpp:195-215); dir 0 = x, 1 = y.
void ref_apply_d(const orc_grid* g, int dir, const double* u, double* out) {
    Grid2D grid = grid_of(g);
    Field2D fu = field_of(grid, u), fo(grid.nx, grid.ny);
    if (dir == 0)
        apply_dx(build_d1(grid.kind_x, grid.nx, grid.dx), fu, fo);
    else
        apply_dy(build_d1(grid.kind_y, grid.ny, grid.dy), fu, fo);
    std::memcpy(out, fo.data(), fo.size() * sizeof(double));
}

// sat_mass_term (sbp.hpp:267-285)
void ref_sat(const orc_grid* g, const double* hu, const double* hv, double* out) {
    Grid2D grid = grid_of(g);
    Field2D fo(grid.nx, grid.ny);
    sat_mass_term(make_boundary_ops(grid), field_of(grid, hu), field_of(grid, hv), fo);
    std::memcpy(out, fo.data(), fo.size() * sizeof(double));
}

// error_norm_and_min_h (time_integration.hpp:103-142); ks = k1|k2|k3|k4, each 5n.
double ref_error_norm(double dt, const orc_grid* g, const double* k1, const double* k2,
                      const double* k3, const double* k4, const double* y,
                      const double* ynew, double atol, double rtol, double* min_h) {
    Grid2D grid = grid_of(g);
    StateField a(grid), bq(grid), cq(grid), dq(grid), ys(grid), yn(grid);
    to_state(k1, a);
    to_state(k2, bq);
    to_state(k3, cq);
    to_state(k4, dq);
    to_state(y, ys);
    to_state(ynew, yn);
    auto r = detail::error_norm_and_min_h(dt, a, bq, cq, dq, ys, yn, atol, rtol);
    if (min_h)
        *min_h = r.second;
    return r.first;
}

// check_sbp_property (sbp.hpp:309-333)
int ref_check_sbp(int kind, int n, double dx, double* max_residual) {
    SbpCheckResult r = check_sbp_property(build_d1(kind_of(kind), n, dx));
    if (max_residual)
        *max_residual = r.max_residual;
    return r.ok ? 1 : 0;
}

// manufactured_generated.hpp:11-115
double ref_mms_bathymetry(double x, double y) { return manufactured::bathymetry1(x, y)[0]; }
void ref_mms_state(double t, double x, double y, double* out5) {
    auto s = manufactured::exact_state(t, x, y);
    for (int k = 0; k < 5; ++k) out5[k] = s[k];
}
void ref_mms_state_dt(double t, double x, double y, double* out5) {
    auto s = manufactured::exact_state_dt(t, x, y);
    for (int k = 0; k < 5; ++k) out5[k] = s[k];
}
void ref_mms_source(double t, double x, double y, double g, double* out5) {
    auto s = manufactured::source_terms(t, x, y, g);
    for (int k = 0; k < 5; ++k) out5[k] = s[k];
}

// make_scenario + prepare_run (scenarios.hpp:598-698, 55-78).  Two-phase: call
// with b_out == NULL to learn the grid, then again with buffers (nx*ny and
// 5*nx*ny doubles).  nx/ny <= 0 select the scenario defaults.  Returns 0 or -1
// (unknown name / parameter; message in err).
int ref_prepare(const char* name, const char* const* keys, const double* vals, int nparams,
                int nx, int ny, orc_grid* g_out, orc_phys* p_out, double* b_out,
                double* q0_out, int* source_kind, double* t0, double* t_final, char* err,
                int err_len) {
    try {
        std::map<std::string, double> params;
        for (int k = 0; k < nparams; ++k)
            params[keys[k]] = vals[k];
        ScenarioSpec spec = make_scenario(name, params);
        if (nx <= 0) nx = spec.nx_default;
        if (ny <= 0) ny = spec.ny_default;
        g_out->nx = nx;
        g_out->ny = ny;
        g_out->kind_x = spec.kind_x == BoundaryKind::bounded;
        g_out->kind_y = spec.kind_y == BoundaryKind::bounded;
        g_out->x_min = spec.x_min;
        g_out->x_max = spec.x_max;
        g_out->y_min = spec.y_min;
        g_out->y_max = spec.y_max;
        p_out->g = spec.g;
        p_out->lambda = spec.lambda;
        p_out->h_floor = PhysSetup{}.h_floor;
        *source_kind = spec.source ? 1 : 0;
        *t0 = spec.t0;
        *t_final = spec.t_final;
        if (!b_out)
            return 0;
        PreparedRun run = prepare_run(spec, nx, ny);
        std::memcpy(b_out, run.ctx.phys.b.data(), run.ctx.phys.b.size() * sizeof(double));
        from_state(run.q0, q0_out);
        return 0;
    } catch (const std::exception& e) {
        if (err && err_len > 0)
            std::snprintf(err, err_len, "%s", e.what());
        return -1;
    }
}

// Samples the manufactured exact state at time t on grid g (scenarios.hpp:200-214).
void ref_mms_exact_field(const orc_grid* g, double t, double* q) {
    Grid2D grid = grid_of(g);
    const std::size_t n = grid.n_total();
    for (int j = 0; j < grid.ny; ++j)
        for (int i = 0; i < grid.nx; ++i) {
            auto s = manufactured::exact_state(t, grid.x(i), grid.y(j));
            for (int k = 0; k < 5; ++k)
                q[k * n + static_cast<std::size_t>(j) * grid.nx + i] = s[k];
        }
}

// parse_config_text (config.hpp:139-247) with a canonical dump of every
// RunConfig field (%.17g numbers, one "key=value" per line) for the
// differential tests of paper_2601_02540_b200/config.py.  Returns 0, or -1
// with the exception message in out.
int ref_parse_config(const char* text, char* out, int out_len) {
    std::ostringstream o;
    auto num = [&](const char* k, double v) {
        char b[64];
        std::snprintf(b, sizeof b, "%.17g", v);
        o << k << '=' << b << '\n';
    };
    try {
        RunConfig c = parse_config_text(text);
        o << "scenario=" << c.scenario << '\n';
        for (const auto& [k, v] : c.scenario_params) num(("param." + k).c_str(), v);
        num("nx", c.nx);
        num("ny", c.ny);
        num("t0", c.t0);
        num("t_final", c.t_final);
        num("threads", c.threads);
        num("abs_tol", c.integrator.abs_tol);
        num("rel_tol", c.integrator.rel_tol);
        num("dt_initial", c.integrator.dt_initial);
        num("dt_max", c.integrator.dt_max);
        num("fixed_dt", c.integrator.fixed_dt);
        num("max_steps", (double)c.integrator.max_steps);
        num("safety", c.integrator.safety);
        num("growth_cap", c.integrator.growth_cap);
        num("shrink_floor", c.integrator.shrink_floor);
        num("tolerances_set", c.tolerances_set);
        o << "output_dir=" << c.output_dir << '\n';
        num("gauges_set", c.gauges_set);
        for (const auto& g : c.gauges) {
            num("gauge.x", g[0]);
            num("gauge.y", g[1]);
        }
        num("snapshots_set", c.snapshots_set);
        for (double t : c.snapshot_times) num("snapshot", t);
        num("conservation_stride", (double)c.conservation_stride);
        num("cross_section_set", c.cross_section_set);
        num("cross_section_y", c.cross_section_y);
        for (int r : c.resolutions) num("resolution", r);
        num("converge_ny", c.converge_ny);
        for (int r : c.bench_resolutions) num("bench_resolution", r);
        num("bench_repetitions", c.bench_repetitions);
        num("bench_warmups", c.bench_warmups);
    } catch (const std::exception& e) {
        std::snprintf(out, (size_t)out_len, "%s", e.what());
        return -1;
    }
    std::snprintf(out, (size_t)out_len, "%s", o.str().c_str());
    return 0;
}

}  // extern "C"
