// dropin_test.cpp -- the reference's own RHS / integrator test cases
// (proj/tests/test_rhs.cpp, test_time_integration.cpp), rewritten against the
// C++ drop-in header: only the include and the namespace differ from a
// reference caller.  Built and run by tests/test_cpp_dropin.py on a B200.
#include <hsgn_b200.hpp>

#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <random>
#include <sstream>

using namespace hsgn_b200;

static int failures = 0;
#define CHECK(cond)                                                   \
    do {                                                              \
        if (!(cond)) {                                                \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                               \
        }                                                             \
    } while (0)

static RhsContext context_on(const Grid2D& g, double lambda, const std::function<double(double, double)>& bathy) {
    PhysSetup phys;
    phys.lambda = lambda;
    phys.b = g.sample(bathy);
    return RhsContext(g, phys);
}

static void randomize(StateField& q, unsigned seed) {  // test_rhs.cpp:22-33
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> depth(0.5, 1.5), vel(-1.0, 1.0);
    for (std::size_t k = 0; k < q.h.size(); ++k) {
        q.h[k] = depth(rng);
        q.u[k] = vel(rng);
        q.v[k] = vel(rng);
        q.w[k] = vel(rng);
        q.eta[k] = depth(rng);
    }
}

static std::string slurp(const std::string& p) {
    std::ifstream in(p);
    std::stringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

static std::vector<std::vector<double>> csv_rows(const std::string& p) {  // skips '#' lines and the header
    std::vector<std::vector<double>> rows;
    std::ifstream in(p);
    std::string line;
    bool header = true;
    while (std::getline(in, line)) {
        if (line.empty() || line[0] == '#') continue;
        if (header) {
            header = false;
            continue;
        }
        std::vector<double> r;
        std::stringstream ss(line);
        std::string cell;
        while (std::getline(ss, cell, ',')) r.push_back(std::stod(cell));
        rows.push_back(r);
    }
    return rows;
}

// lake_at_rest (scenarios.hpp:480-500) recorded as cmd_run does (cli.hpp:88-116)
static SolutionRecord run_lake(const std::string& dir, int n, double t_final, std::vector<std::array<double, 2>> gauges,
                               std::vector<double> snaps, int64_t stride, std::vector<SnapshotRecord>* taken) {
    std::filesystem::remove_all(dir);
    std::filesystem::create_directories(dir);
    Grid2D g = make_grid(-5.0, 5.0, -5.0, 5.0, n, n);
    RhsContext ctx = context_on(g, 500.0, [](double x, double y) { return 0.1 * std::exp(-0.5 * (x * x + y * y)); });
    StateField q0(g);
    for (std::size_t k = 0; k < q0.h.size(); ++k) q0.h[k] = 1.0 - ctx.phys.b[k];
    q0.eta = q0.h;
    init_auxiliary(ctx, q0);
    RunRecorder rec(ctx, dir, gauges, snaps, stride);
    SolutionRecord sol = adaptive_solve(ctx, q0, 0.0, t_final, IntegratorConfig(), rec);
    rec.flush();
    if (taken) *taken = rec.snapshots();
    return sol;
}

static double mass_sum(const Grid2D& g, const Field2D& f) {  // sbp.hpp:219-239 weights, plain sum
    double s = 0.0;
    for (int j = 0; j < g.ny; ++j)
        for (int i = 0; i < g.nx; ++i) {
            double wx = g.dx, wy = g.dy;
            if (g.kind_x == BoundaryKind::bounded && (i == 0 || i == g.nx - 1)) wx *= 0.5;
            if (g.kind_y == BoundaryKind::bounded && (j == 0 || j == g.ny - 1)) wy *= 0.5;
            s += wx * wy * f(i, j);
        }
    return s;
}

int main() {
    auto flat = [](double, double) { return 0.0; };
    {  // uniform columns are steady (test_rhs.cpp:39-65)
        Grid2D g = make_grid(-1.0, 1.0, -1.0, 1.0, 12, 10);
        RhsContext ctx = context_on(g, 500.0, flat);
        StateField q(g), out(g);
        q.h.fill(1.0);
        q.u.fill(0.3);
        q.v.fill(-0.7);
        q.eta.fill(1.0);
        rhs_periodic(ctx, 0.0, q, out);
        for (Field2D* f : out.fields())
            for (std::size_t k = 0; k < f->size(); ++k) CHECK((*f)[k] == 0.0);
        Grid2D gb = make_grid(-1.0, 1.0, -1.0, 1.0, 12, 10, BoundaryKind::bounded, BoundaryKind::bounded);
        RhsContext cb = context_on(gb, 500.0, flat);
        StateField qb(gb), ob(gb);
        qb.h.fill(2.0);
        qb.eta.fill(2.0);
        rhs_reflecting(cb, 0.0, qb, ob);
        for (Field2D* f : ob.fields())
            for (std::size_t k = 0; k < f->size(); ++k) CHECK((*f)[k] == 0.0);
    }
    {  // lake at rest over a bump (test_rhs.cpp:67-82)
        auto bump = [](double x, double y) { return 0.1 * std::exp(-(x * x + y * y)); };
        for (BoundaryKind kind : {BoundaryKind::periodic, BoundaryKind::bounded}) {
            Grid2D g = make_grid(-5.0, 5.0, -5.0, 5.0, 33, 33, kind, kind);
            RhsContext ctx = context_on(g, 500.0, bump);
            StateField q(g), out(g);
            for (std::size_t k = 0; k < q.h.size(); ++k) q.h[k] = 1.0 - ctx.phys.b[k];
            init_auxiliary(ctx, q);
            rhs(ctx, 0.0, q, out);
            for (Field2D* f : out.fields())
                for (std::size_t k = 0; k < f->size(); ++k) CHECK(std::abs((*f)[k]) <= 1e-12 * 9.81);
        }
    }
    {  // mass invariance (test_rhs.cpp:84-106) and energy rate (108-127)
        Grid2D g = make_grid(-1.0, 1.0, -1.0, 1.0, 24, 20, BoundaryKind::bounded, BoundaryKind::bounded);
        RhsContext ctx = context_on(g, 500.0, [](double x, double y) { return 0.05 * std::cos(x - y); });
        StateField q(g), out(g);
        randomize(q, 12);
        rhs_reflecting(ctx, 0.0, q, out);
        CHECK(std::abs(mass_sum(g, out.h)) <= 1e-12);
        const double e = total_energy(ctx, q);
        CHECK(std::abs(energy_rate(ctx, q, out)) <= 1e-11 * std::abs(e));
    }
    {  // determinism (test_rhs.cpp:159-174)
        Grid2D g = make_grid(-1.0, 1.0, -1.0, 1.0, 20, 20, BoundaryKind::bounded, BoundaryKind::periodic);
        RhsContext ctx = context_on(g, 500.0, [](double x, double y) { return 0.03 * std::sin(x * y); });
        StateField q(g), a(g), b(g);
        randomize(q, 41);
        rhs(ctx, 0.5, q, a);
        rhs(ctx, 0.5, q, b);
        auto fa = a.fields();
        auto fb = b.fields();
        for (int f = 0; f < 5; ++f)
            for (std::size_t k = 0; k < fa[f]->size(); ++k) CHECK((*fa[f])[k] == (*fb[f])[k]);
        CHECK(ctx.n_evals() == 2);
    }
    {  // non-positive depth raises (test_rhs.cpp:176-186)
        Grid2D g = make_grid(-1.0, 1.0, -1.0, 1.0, 8, 8);
        RhsContext ctx = context_on(g, 500.0, flat);
        StateField q(g), out(g);
        q.h.fill(1.0);
        q.eta.fill(1.0);
        q.h(3, 4) = -0.25;
        bool threw = false;
        try {
            rhs(ctx, 0.0, q, out);
        } catch (const depth_error&) {
            threw = true;
        }
        CHECK(threw);
    }
    {  // invalid grids throw like grid.hpp:51-55
        bool threw = false;
        try {
            make_grid(0.0, 1.0, 0.0, 1.0, 3, 8);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    }
    {  // integrator: ledger, observer, mass through full steps (test_time_integration.cpp:127-150, 290-307)
        Grid2D g = make_grid(-5.0, 5.0, -5.0, 5.0, 32, 32);
        RhsContext ctx = context_on(g, 500.0, flat);
        StateField q0(g);
        q0.h = g.sample([](double x, double y) { return 1.0 + 0.1 * std::exp(-(x * x + y * y)); });
        init_auxiliary(ctx, q0);
        const double m0 = total_mass(ctx, q0);
        std::vector<double> times;
        IntegratorConfig cfg;
        SolutionRecord rec =
            adaptive_solve(ctx, q0, 0.0, 0.1, cfg, [&](double t, const StateField&, const StateField&) { times.push_back(t); });
        CHECK(!rec.aborted);
        CHECK(rec.t == 0.1);
        CHECK(times.size() == static_cast<std::size_t>(rec.accepted) + 1);
        CHECK(rec.rhs_evals == 3 * (rec.accepted + rec.rejected) + 1 + rec.rhs_evals_setup);
        CHECK(std::abs(total_mass(ctx, rec.q) - m0) <= 1e-12 * std::abs(m0));
        SolutionRecord back = adaptive_solve(ctx, q0, 2.0, 1.0, cfg);
        CHECK(back.aborted && back.abort_reason.find("precedes") != std::string::npos);
        IntegratorConfig one;
        one.max_steps = 1;
        one.dt_initial = 1e-3;
        SolutionRecord budget = adaptive_solve(ctx, q0, 0.0, 100.0, one);
        CHECK(budget.aborted && budget.abort_reason.find("step budget exhausted") != std::string::npos);
        CHECK(budget.accepted == 1);
    }
    {  // run recorder: test_cli.cpp:61-131 ("run command produces the full output set")
        const std::string dir = "/tmp/hsgn_dropin_run_lake";
        std::vector<SnapshotRecord> snaps;
        SolutionRecord sol = run_lake(dir, 20, 1.0, {{0.0, 0.0}}, {0.0, 0.5}, 1, &snaps);
        CHECK(!sol.aborted && sol.t == 1.0);
        CHECK(std::filesystem::exists(dir + "/snapshot_t0.csv"));
        CHECK(std::filesystem::exists(dir + "/snapshot_t0.5.csv"));
        auto cons = csv_rows(dir + "/conservation.csv");
        CHECK(cons.size() == static_cast<std::size_t>(sol.accepted) + 1);
        CHECK(slurp(dir + "/conservation.csv").rfind("t,total_mass,total_energy,semidiscrete_energy_rate\n", 0) == 0);
        for (const auto& r : cons) {
            CHECK(std::abs(r[1] - cons[0][1]) <= 1e-12 * std::abs(cons[0][1]));
            CHECK(std::abs(r[2] - cons[0][2]) <= 1e-12 * std::abs(cons[0][2]));
            CHECK(std::abs(r[3]) <= 1e-11 * std::abs(cons[0][2]));
        }
        auto gauges = csv_rows(dir + "/gauges.csv");
        CHECK(gauges.size() == cons.size());
        for (const auto& r : gauges) CHECK(std::abs(r[1] - 1.0) <= 1e-12);
        CHECK(snaps.size() == 2 && snaps[0].target == 0.0 && snaps[0].actual == 0.0);
        CHECK(csv_rows(dir + "/snapshot_t0.csv").size() == 20 * 20);
    }
    {  // reruns are byte-identical (test_cli.cpp:134-156)
        const std::string a = "/tmp/hsgn_dropin_rerun_a", b = "/tmp/hsgn_dropin_rerun_b";
        run_lake(a, 16, 0.5, {{1.0, -1.0}}, {0.25}, 1, nullptr);
        run_lake(b, 16, 0.5, {{1.0, -1.0}}, {0.25}, 1, nullptr);
        CHECK(slurp(a + "/conservation.csv") == slurp(b + "/conservation.csv"));
        CHECK(slurp(a + "/gauges.csv") == slurp(b + "/gauges.csv"));
        CHECK(!slurp(a + "/snapshot_t0.25.csv").empty());
        CHECK(slurp(a + "/snapshot_t0.25.csv") == slurp(b + "/snapshot_t0.25.csv"));
    }
    {  // scenario registry (scenarios.hpp:598-705): names, errors, prepare_run, exact state
        CHECK(scenario_names().size() == 10 && scenario_names()[0] == "soliton");
        bool threw = false;
        try {
            make_scenario("maelstrom");
        } catch (const std::invalid_argument& e) {
            threw = std::string(e.what()) == "unknown scenario 'maelstrom'";
        }
        CHECK(threw);
        threw = false;
        try {
            make_scenario("soliton", {{"amplitud", 0.1}});
        } catch (const std::invalid_argument& e) {
            threw = std::string(e.what()) == "scenario 'soliton': unknown parameter 'amplitud'";
        }
        CHECK(threw);
        ScenarioSpec spec = make_scenario("soliton", {{"amplitude", 0.2}});
        CHECK(spec.lambda == 30000.0 && spec.nx_default == 200 && spec.exact_vars.size() == 2);
        PreparedRun run = prepare_run(spec, 256, 4);
        CHECK(run.grid.nx == 256 && run.grid.x_min == -30.0);
        for (std::size_t k = 0; k < run.q0.h.size(); ++k) CHECK(run.q0.eta[k] == run.q0.h[k]);  // init_auxiliary
        StateField ex(run.grid);
        exact_state(spec, 0.0, run.grid, ex);
        for (int i = 0; i < 256; ++i)
            if (std::abs(run.grid.x(i)) < 29.0) CHECK(ex.h(i, 0) == run.q0.h(i, 0) && ex.u(i, 0) == run.q0.u(i, 0));
        IntegratorConfig cfg;
        cfg.fixed_dt = 2e-3;
        const double m0 = total_mass(run.ctx, run.q0);
        SolutionRecord sol = adaptive_solve(run.ctx, run.q0, 0.0, 0.2, cfg);
        CHECK(!sol.aborted && sol.accepted == 100);
        CHECK(std::abs(total_mass(run.ctx, sol.q) - m0) <= 1e-12 * std::abs(m0));
        PreparedRun mms = prepare_run(make_scenario("manufactured"), 32, 32);  // forcing on the device
        CHECK(mms.ctx.n_evals() == 0);
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "PASSED", failures);
    return failures ? 1 : 0;
}
