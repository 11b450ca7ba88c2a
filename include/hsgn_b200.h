/*
 * hsgn_b200.h -- C ABI of the B200-native time-stepping hot path for the
 * energy-conserving split-form SBP discretisation of the hyperbolized
 * Serre-Green-Naghdi equations (arXiv 2601.02540).
 *
 * The reference (/root/reference/proj, "hsgn") is a header-only C++20
 * library with no FFI; its boundary for this path is the C++ operator API
 * listed next to each entry point below.  This header is that API flattened
 * to plain C (pointers + sizes, no C++ or torch types) so a C++ shim
 * (include/hsgn_b200.hpp), ctypes (paper_2601_02540_b200/_native.py) or any
 * other FFI can bind it.  See INTEGRATION.md for the bindings.
 *
 * Data layout on the host side of every copy: a state is 5 contiguous fp64
 * fields h, u, v, w, eta, each nx*ny, row-major with x fastest (index
 * j*nx + i) -- exactly the reference StateField / Field2D storage
 * (model.hpp:22-35, field.hpp:9-10).  Device-side layout is private (see
 * per-field slabs with ghost rows).
 *
 * Error behaviour mirrors the reference exceptions:
 *   HSGN_EINVAL  <- std::invalid_argument (grid.hpp:51-55, sbp.hpp:37-40, rhs.hpp:41-42)
 *   HSGN_EDEPTH  <- hsgn::depth_error     (rhs.hpp:111-113): output untouched
 *   HSGN_ECUDA / HSGN_ENCCL                device / communicator failures
 * hsgn_last_error() returns the message of the last failure on a context.
 * There is no CPU fallback: every compute entry point runs sm_100a kernels
 * and fails with HSGN_ECUDA when no B200 is present.
 */
#ifndef HSGN_B200_H
#define HSGN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HSGN_OK = 0,
    HSGN_EINVAL = 1,
    HSGN_EDEPTH = 2,
    HSGN_ECUDA = 3,
    HSGN_ENCCL = 4
} hsgn_status;

/* reference grid.hpp:11 BoundaryKind */
enum { HSGN_PERIODIC = 0, HSGN_BOUNDED = 1 };

/* reference grid.hpp:16-41 Grid2D (spacing derived as in make_grid :47-68) */
typedef struct {
    int32_t nx, ny;
    int32_t kind_x, kind_y;
    double x_min, x_max, y_min, y_max;
} hsgn_grid;

/* reference model.hpp:40-45 PhysSetup (bathymetry passed separately) */
typedef struct {
    double g, lambda, h_floor;
} hsgn_phys;

/* reference time_integration.hpp:18-29 IntegratorConfig */
typedef struct {
    double abs_tol, rel_tol, dt_initial, dt_max, safety, growth_cap, shrink_floor;
    int64_t max_steps;
    double fixed_dt, h_floor;
} hsgn_cfg;

/* reference time_integration.hpp:33-42 SolutionRecord (state returned separately) */
typedef struct {
    double t;
    int64_t accepted, rejected, rhs_evals, rhs_evals_setup;
    int32_t aborted;
    char reason[256];
} hsgn_record;

typedef struct hsgn_ctx hsgn_ctx;     /* RhsContext: grid, physics, operators, b, workspace */
typedef struct hsgn_state hsgn_state; /* device-resident StateField */

/* AcceptObserver (time_integration.hpp:49): called on the initial state and
 * after every accepted step with (t, y, FSAL tendency).  The states are
 * device resident and valid only during the call. */
typedef void (*hsgn_observer)(double t, const hsgn_state* q, const hsgn_state* q_t, void* user);

/* ------------------------------------------------------------ context */

/* make_rhs_context (rhs.hpp:40-54) on one device.  b_host: nx*ny doubles.
 * device < 0 selects the current device. */
hsgn_status hsgn_ctx_create(const hsgn_grid* grid, const hsgn_phys* phys, const double* b_host,
                            int device, hsgn_ctx** out);

/* Slab of a y-decomposed grid (multi-GPU): rows
 * [j_begin, j_end) of the global grid (at least 2) live on this rank; b_host
 * holds the slab's rows only.  Neighbour ranks are (rank-1, rank+1) mod
 * nranks. */
hsgn_status hsgn_ctx_create_slab(const hsgn_grid* grid, const hsgn_phys* phys, const double* b_host,
                                 int device, int32_t j_begin, int32_t j_end, int32_t rank,
                                 int32_t nranks, hsgn_ctx** out);

/* Attach an NCCL communicator for the slab halo exchange (nccl_id: the 128
 * bytes of an ncclUniqueId produced by hsgn_nccl_unique_id on rank 0 and
 * broadcast by the caller). */
hsgn_status hsgn_nccl_unique_id(unsigned char out_id[128]);
hsgn_status hsgn_ctx_attach_nccl(hsgn_ctx* ctx, const unsigned char nccl_id[128]);

hsgn_status hsgn_ctx_destroy(hsgn_ctx* ctx);
const char* hsgn_last_error(const hsgn_ctx* ctx);

/* ctx.source hook (rhs.hpp:24-26): 0 none, 1 manufactured solution
 * (scenarios.hpp:179-217 / manufactured_generated.hpp:69-115). */
hsgn_status hsgn_set_source(hsgn_ctx* ctx, int32_t kind);

/* Launch-shape tuning (rows marched per CTA); 0 restores the default. */
hsgn_status hsgn_set_rows_per_block(hsgn_ctx* ctx, int32_t rows);

/* Stencil arithmetic variant (all bit-identical):
 * 0 general, 1 power-of-two coefficients, 2 one common power-of-two factor
 * (fully periodic, dx == dy).  -1 = automatic (the most specialised valid
 * one); a request above what the grid allows is capped.  Used by the parity
 * tests to cover every variant on the same inputs. */
hsgn_status hsgn_set_stencil_kind(hsgn_ctx* ctx, int32_t kind);
int32_t hsgn_stencil_kind(const hsgn_ctx* ctx);

/* Kernel structure of the fixed steps and adaptive attempts (both
 * bit-identical): 0 = one kernel per stage,
 * 3 (default) = stages 1+2 fused (S12), then stage 3.  Other values:
 * HSGN_EINVAL. */
hsgn_status hsgn_set_fused_stages(hsgn_ctx* ctx, int32_t mode);
int32_t hsgn_fused_stages(const hsgn_ctx* ctx);

/* ctx.n_evals (rhs.hpp:28,84) */
int64_t hsgn_n_evals(const hsgn_ctx* ctx);

/* ------------------------------------------------------------ states */

hsgn_status hsgn_state_alloc(hsgn_ctx* ctx, hsgn_state** out);
hsgn_status hsgn_state_free(hsgn_ctx* ctx, hsgn_state* s);
/* host <-> device, host layout as documented above (slab rows only on slabs) */
hsgn_status hsgn_state_upload(hsgn_ctx* ctx, hsgn_state* s, const double* host);
hsgn_status hsgn_state_download(hsgn_ctx* ctx, const hsgn_state* s, double* host);
hsgn_status hsgn_state_copy(hsgn_ctx* ctx, const hsgn_state* src, hsgn_state* dst);
/* Device pointer of field f, row 0 (row pitch = nx doubles; rows -2, -1
 * and ny_local, ny_local + 1 are the ghost rows). */
hsgn_status hsgn_state_field_ptr(const hsgn_state* s, int32_t f, double** out);

/* ------------------------------------------------------------ operators */

/* rhs / rhs_periodic / rhs_reflecting (rhs.hpp:219-238): out = tendency(q, t).
 * HSGN_EDEPTH when some node has !(h > 0); *bad_nodes gets the count and
 * out is left untouched. */
hsgn_status hsgn_rhs(hsgn_ctx* ctx, double t, const hsgn_state* q, hsgn_state* out, int64_t* bad_nodes);
/* rhs_shallow_water (rhs.hpp:243-248) */
hsgn_status hsgn_rhs_shallow_water(hsgn_ctx* ctx, double t, const hsgn_state* q, hsgn_state* out,
                                   int64_t* bad_nodes);
/* init_auxiliary (model.hpp:93-105): eta = h, w from the SBP operators. */
hsgn_status hsgn_init_auxiliary(hsgn_ctx* ctx, hsgn_state* q);

/* ------------------------------------------------------------ integrator */

/* adaptive_solve (time_integration.hpp:209-350) with the fused stage
 * kernels; fixed-step mode (cfg->fixed_dt > 0) runs CUDA-graph chunks.
 * q_out receives the final (or last valid) state. */
hsgn_status hsgn_solve(hsgn_ctx* ctx, const hsgn_state* q0, double t0, double t_final,
                       const hsgn_cfg* cfg, hsgn_state* q_out, hsgn_record* rec, hsgn_observer obs,
                       void* user);

/* ------------------------------------------------------------ run recorder */

/* RunRecorder (io.hpp:107-219) on the device: gauge samples h + b at the
 * nearest nodes of gauge_xy (n_gauges (x, y) pairs, io.hpp:38-48) after
 * every accepted step, the conservation row (t, total mass, total energy,
 * semidiscrete energy rate) every conservation_stride accepted steps
 * (counting the initial state), and snapshots of the accepted state closest
 * to each target time.  Fixed-step runs keep their CUDA-graph chunks (the
 * gauge gather is captured in them).  Whole-grid contexts only. */
typedef struct hsgn_recorder hsgn_recorder;
hsgn_status hsgn_recorder_create(hsgn_ctx* ctx, int32_t n_gauges, const double* gauge_xy, int32_t n_targets,
                                 const double* targets, int64_t conservation_stride, hsgn_recorder** out);
hsgn_status hsgn_recorder_destroy(hsgn_recorder* r);
/* adaptive_solve with the recorder attached as its AcceptObserver
 * (cli.hpp:100-111); obs may be NULL. */
hsgn_status hsgn_solve_recorded(hsgn_ctx* ctx, const hsgn_state* q0, double t0, double t_final,
                                const hsgn_cfg* cfg, hsgn_state* q_out, hsgn_record* rec, hsgn_observer obs,
                                void* user, hsgn_recorder* r);
hsgn_status hsgn_recorder_counts(const hsgn_recorder* r, int64_t* gauge_rows, int64_t* cons_rows,
                                 int32_t* snapshots);
/* node (i, j) and coordinates of gauge k */
hsgn_status hsgn_recorder_gauge_node(const hsgn_recorder* r, int32_t k, int32_t* i, int32_t* j, double* x,
                                     double* y);
/* t[rows], values[rows * n_gauges] */
hsgn_status hsgn_recorder_gauges(const hsgn_recorder* r, double* t, double* values);
/* rows4[rows * 4] = (t, mass, energy, energy_rate) */
hsgn_status hsgn_recorder_conservation(const hsgn_recorder* r, double* rows4);
/* snapshot k: target time, time of the state used, and the state (host
 * layout, may be NULL) */
hsgn_status hsgn_recorder_snapshot(const hsgn_recorder* r, int32_t k, double* target, double* actual,
                                   double* host_state);

/* The bare fused fixed-step pipeline used by the benchmark: `steps` BS3 steps
 * of size dt on (y, k1) in place (k1 must hold f(y) on entry; it holds f(y)
 * of the new state on return, FSAL).  The caller's buffers are the
 * integrator's parity-0 pair (no copies for an even count).  Graph-captured
 * (slab contexts capture their NCCL halo exchanges too).  Returns
 * HSGN_EDEPTH if any stage input had !(h > 0); *steps_done gets the
 * completed count.  hsgn_last_timing() gives the device ms of the whole call. */
hsgn_status hsgn_bs3_fixed_steps(hsgn_ctx* ctx, hsgn_state* y, hsgn_state* k1, double t, double dt,
                                 int64_t steps, int64_t* steps_done);
/* Builds (captures and instantiates) the CUDA graphs that
 * hsgn_bs3_fixed_steps(ctx, y, k1, ..., dt, steps, ...) will launch, without
 * running a step: graph construction is one-time host work, kept out of a
 * timed run. */
hsgn_status hsgn_prepare_fixed_steps(hsgn_ctx* ctx, hsgn_state* y, hsgn_state* k1, double dt, int64_t steps);
/* Per-kernel timing of the fixed-step graphs (whole-grid S12 + S3 contexts):
 * with it on, the captured graphs carry CUDA event nodes around every
 * kernel, and hsgn_kernel_times() returns the mean S12 and S3 durations of
 * the last hsgn_bs3_fixed_steps call (measured inside that call). */
hsgn_status hsgn_set_kernel_timing(hsgn_ctx* ctx, int32_t on);
hsgn_status hsgn_kernel_times(const hsgn_ctx* ctx, double* s12_ms, double* s3_ms, int64_t* steps);

/* ------------------------------------------------------------ diagnostics */

/* total_mass, total_energy (model.hpp:77-87), energy_rate (analysis.hpp:47-67),
 * mass_weighted_sum of a single field f of q (sbp.hpp:219-239). */
hsgn_status hsgn_total_mass(hsgn_ctx* ctx, const hsgn_state* q, double* out);
hsgn_status hsgn_total_energy(hsgn_ctx* ctx, const hsgn_state* q, double* out);
hsgn_status hsgn_energy_rate(hsgn_ctx* ctx, const hsgn_state* q, const hsgn_state* q_t, double* out);
hsgn_status hsgn_mass_weighted_sum(hsgn_ctx* ctx, const hsgn_state* q, int32_t field, double* out);
/* discrete_l2_error (analysis.hpp:15-25) of field f between a and b */
hsgn_status hsgn_discrete_l2_error(hsgn_ctx* ctx, const hsgn_state* a, const hsgn_state* b, int32_t field,
                                   double* out);
/* Per-row weighted sums r_j = sum_i wx_i F_ij for slab rows (kind: 0 mass,
 * 1 energy density, 2 energy rate, 3 field f=aux squared difference);
 * the caller combines rows across slabs (deterministic outer sum). */
hsgn_status hsgn_row_sums(hsgn_ctx* ctx, int32_t kind, const hsgn_state* q, const hsgn_state* q_t,
                          int32_t field, double* rows_host);
/* Outer compensated sum over rows with the y mass weights (sbp.hpp:232-237). */
double hsgn_outer_sum(const hsgn_grid* grid, const double* rows, int32_t j_begin, int32_t j_end);

/* Mean device ms of each of the three fused stage kernels over `reps` steps
 * (CUDA events on the context stream; inputs copied, caller state intact). */
hsgn_status hsgn_profile_stages(hsgn_ctx* ctx, const hsgn_state* y, const hsgn_state* k1, double dt,
                                int32_t reps, double* ms3);

/* Mean device ms of the fused S12 kernel over `reps` launches (inputs
 * copied, caller state intact). */
hsgn_status hsgn_profile_fused(hsgn_ctx* ctx, const hsgn_state* y, const hsgn_state* k1, double dt, int32_t reps,
                               double* ms);

/* ------------------------------------------------------------ in-process slab group */

/* The y-slab decomposition driven from ONE process:
 * n slab contexts on devices[r] (NULL: current device; several slabs may
 * share a GPU), halo rows pulled from the neighbours' boundary rows through
 * (peer) device pointers after every stage, ordered by CUDA events.  Same
 * arithmetic and exchange schedule as the NCCL path; host arrays are the
 * FULL grid. */
typedef struct hsgn_group hsgn_group;
typedef struct hsgn_gstate hsgn_gstate;
hsgn_status hsgn_group_create(const hsgn_grid* grid, const hsgn_phys* phys, const double* b_full,
                              const int* devices, int32_t n, hsgn_group** out);
hsgn_status hsgn_group_destroy(hsgn_group* g);
const char* hsgn_group_last_error(const hsgn_group* g);
hsgn_status hsgn_group_state_alloc(hsgn_group* g, hsgn_gstate** out);
hsgn_status hsgn_group_state_free(hsgn_group* g, hsgn_gstate* s);
hsgn_status hsgn_group_state_upload(hsgn_group* g, hsgn_gstate* s, const double* host_full);
hsgn_status hsgn_group_state_download(hsgn_group* g, const hsgn_gstate* s, double* host_full);
hsgn_status hsgn_group_rhs(hsgn_group* g, double t, const hsgn_gstate* q, hsgn_gstate* out, int64_t* bad_nodes);
hsgn_status hsgn_group_bs3_fixed_steps(hsgn_group* g, hsgn_gstate* y, hsgn_gstate* k1, double t, double dt,
                                       int64_t steps, int64_t* steps_done);
/* kind: 0 total mass, 1 total energy, 2 energy rate (q_t required) */
hsgn_status hsgn_group_reduce(hsgn_group* g, int32_t kind, const hsgn_gstate* q, const hsgn_gstate* q_t,
                              double* out);

/* ------------------------------------------------------------ scenarios (CLI front end) */

/* The reference scenario registry (scenarios.hpp:18-707): make_scenario
 * resolves a scenario by name with numeric parameter overrides (same names,
 * defaults and messages, :598-698); sample() evaluates its initial b, h, u, v
 * at the nodes of an nx x ny grid over `domain` (w and eta are left zero for
 * hsgn_init_auxiliary, as prepare_run does, :55-78); exact() fills the exact
 * state at time t (soliton, manufactured).  Host-side, no device needed. */
typedef struct {
    char name[32];
    hsgn_grid domain; /* extents and kinds; nx, ny = the scenario's default resolution */
    double g, lambda, t0, t_final;
    int32_t has_source; /* manufactured forcing: hsgn_set_source(ctx, 1) */
    int32_t has_exact;
    int32_t n_exact_vars, exact_vars[5]; /* field indices compared by the convergence study */
    int32_t n_gauges, n_snapshots;
    double gauges[8][2];
    double snapshot_times[8];
    int32_t kind, reserved;
    double p[24]; /* resolved parameters and derived constants (private) */
} hsgn_scenario;
int32_t hsgn_scenario_count(void);
const char* hsgn_scenario_name(int32_t k); /* scenario_names(), scenarios.hpp:700-705 */
hsgn_status hsgn_scenario_make(const char* name, const char* const* keys, const double* vals, int32_t n,
                               hsgn_scenario* out, char* err, int32_t err_len);
hsgn_status hsgn_scenario_sample(const hsgn_scenario* s, int32_t nx, int32_t ny, double* b, double* q5);
/* The same for global rows [j0, j1) of the nx x ny grid only (a slab's
 * rows; b and q5 hold (j1 - j0) * nx nodes per field). */
hsgn_status hsgn_scenario_sample_rows(const hsgn_scenario* s, int32_t nx, int32_t ny, int32_t j0, int32_t j1,
                                      double* b, double* q5);
hsgn_status hsgn_scenario_exact(const hsgn_scenario* s, int32_t nx, int32_t ny, double t, double* q5);
/* The spec's closed forms at one point: bhuv = {b, h0, u0, v0}(x, y). */
hsgn_status hsgn_scenario_eval(const hsgn_scenario* s, double x, double y, double bhuv[4]);

/* ------------------------------------------------------------ misc */
hsgn_status hsgn_synchronize(hsgn_ctx* ctx);
/* Elapsed ms of the last hsgn_bs3_fixed_steps call measured with CUDA events
 * on the context stream, and the number of kernels it launched. */
hsgn_status hsgn_last_timing(const hsgn_ctx* ctx, double* ms, int64_t* kernels);
const char* hsgn_build_info(void);

#ifdef __cplusplus
}
#endif
#endif
