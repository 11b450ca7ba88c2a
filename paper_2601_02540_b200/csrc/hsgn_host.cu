// hsgn_host.cu -- host runtime of the B200 hot path and its C ABI
// (include/hsgn_b200.h).
//
// Owns: the device context (RhsContext analogue, rhs.hpp:17-54), device
// states with the slab layout, the fused BS3 driver (adaptive_solve,
// time_integration.hpp:209-350) with CUDA-graph-captured fixed-step chunks,
// the SBP-norm diagnostics, and the multi-GPU slab halo exchange over NCCL.
// No CPU compute path exists: every operator launches sm_100a kernels.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/hsgn_b200.h"
#include "sgn_device.cuh"

namespace hsgn_dev {
// sgn_stage.cu
cudaError_t launch_stage(int mode, const StageArgs& A, cudaStream_t st);
int stage_launches(int mode, const StageArgs& A);
cudaError_t launch_src_factors(double x0, double dx, int n, double* out, cudaStream_t st);
int stage_grid_blocks(const StageArgs& A);
cudaError_t launch_sum_partials(const double* part, int n, double* out, cudaStream_t st);
// sgn_aux.cu
cudaError_t launch_cons_rows(const AuxArgs& A, const double* q, const double* qt, double* rows, cudaStream_t st);
cudaError_t launch_gauges(const double* h, const double* b, const long long* idx, int n, double* out,
                          cudaStream_t st);
cudaError_t launch_row_sums(const AuxArgs& A, int kind, const double* q, const double* qt, int field,
                            double* rows, cudaStream_t st);
cudaError_t launch_depth_check(const double* h, long long n, unsigned long long* bad, cudaStream_t st);
cudaError_t launch_axpy5(const double* a, double c, const double* x, double* out, long long n, long long fs,
                         cudaStream_t st);
int wrms_blocks();
cudaError_t launch_wrms(const double* x, const double* ref, double atol, double rtol, long long n, long long fs,
                        double* part, cudaStream_t st);
cudaError_t launch_init_aux(const AuxArgs& A, double* q, cudaStream_t st);
}  // namespace hsgn_dev

using namespace hsgn_dev;

// ------------------------------------------------------------------ NCCL (dlopen)
// The slab exchange and the cross-rank agreement need a few NCCL entry points; they are resolved at run
// time from the libnccl.so.2 already mapped by torch (or the system one), so
// single-GPU use carries no NCCL dependency.
namespace {
typedef struct {
    char internal[128];
} nccl_uid;
typedef void* nccl_comm;
typedef int (*p_get_uid)(nccl_uid*);
typedef int (*p_init_rank)(nccl_comm*, int, nccl_uid, int);
typedef int (*p_send)(const void*, size_t, int, int, nccl_comm, cudaStream_t);
typedef int (*p_recv)(void*, size_t, int, int, nccl_comm, cudaStream_t);
typedef int (*p_allreduce)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t);
typedef int (*p_group)(void);
typedef int (*p_destroy)(nccl_comm);
typedef const char* (*p_errstr)(int);
struct NcclApi {
    bool ok = false;
    p_get_uid get_uid;
    p_init_rank init_rank;
    p_send send;
    p_recv recv;
    p_allreduce allreduce;
    p_group group_start, group_end;
    p_destroy destroy;
    p_errstr errstr;
};
const NcclApi& nccl() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return api;
    api.get_uid = (p_get_uid)dlsym(h, "ncclGetUniqueId");
    api.init_rank = (p_init_rank)dlsym(h, "ncclCommInitRank");
    api.send = (p_send)dlsym(h, "ncclSend");
    api.recv = (p_recv)dlsym(h, "ncclRecv");
    api.allreduce = (p_allreduce)dlsym(h, "ncclAllReduce");
    api.group_start = (p_group)dlsym(h, "ncclGroupStart");
    api.group_end = (p_group)dlsym(h, "ncclGroupEnd");
    api.destroy = (p_destroy)dlsym(h, "ncclCommDestroy");
    api.errstr = (p_errstr)dlsym(h, "ncclGetErrorString");
    api.ok = api.get_uid && api.init_rank && api.send && api.recv && api.allreduce && api.group_start &&
             api.group_end && api.destroy;
    return api;
}
constexpr int NCCL_UINT64 = 5;   // ncclUint64
constexpr int NCCL_FLOAT64 = 8;  // ncclDouble
constexpr int NCCL_SUM = 0, NCCL_MAX = 2, NCCL_MIN = 3;
}  // namespace

// ------------------------------------------------------------------ types

struct hsgn_state {
    double* base = nullptr;  // 5 fields, each (ny_local + 2) rows of nx
    long long fs = 0;        // field stride (elements)
    double* f(int k) const { return base + k * fs; }
};

namespace {

struct FixedGraph {
    cudaGraphExec_t exec = nullptr;
    int steps = 0;
    int64_t kernels = 0;  // kernel nodes of this library in the graph
};

}  // namespace

struct hsgn_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t cstream = nullptr;  // high-priority comm stream of an NCCL slab (halos, agreement)
    cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_c = nullptr, ev_d = nullptr, ev_e = nullptr;  // slab schedule
    // global grid + slab
    hsgn_grid grid{};
    hsgn_phys phys{};
    int j_begin = 0, j_end = 0, ny_loc = 0, rank = 0, nranks = 1;
    double dx = 0, dy = 0;
    long long fs = 0;  // elements per field incl. ghost rows
    double* b = nullptr;  // bathymetry row 0 pointer (ghost rows allocated)
    double* b_alloc = nullptr;
    StageArgs base{};
    AuxArgs aux{};
    int source = 0;
    int rows_per_block = 0;
    int forced_kind = -1;  // stencil kind override (tests); -1 = automatic
    int in_group = 0;      // member of an in-process slab group (halo pulls by the group)
    int ring1 = 0;         // 1-slab ring: NCCL attached to a 1-rank periodic-y context (halos to itself)
    int b_lit = 0;         // some b value (of any slab) outside the magnitude guard (sgn_device.cuh)
    int* d_hint = nullptr; // literal-pass tile hints (StageArgs::hint_s12 / hint_stage)
    double* d_srcx = nullptr;  // manufactured-source factor tables (StageArgs::srcx / srcy)
    double* d_srcy = nullptr;
    long long hint_cap = 0;
    int fused = 3;         // fixed-step structure: 0 one kernel per stage, 3 S12 + S3
    int64_t n_evals = 0;
    int64_t launches = 0;  // kernels of this library launched (or captured) on the context stream
    std::string err;
    // workspace for the integrator
    hsgn_state ws[8];  // y0,y1,k1a,k1b,k2,part,scratchA,scratchB
    bool ws_ready = false;
    StepRec* d_rec = nullptr;  // per-step records (capacity rec_cap)
    int rec_cap = 0;
    int* d_halt = nullptr;
    double* d_err_part = nullptr;
    int err_part_cap = 0;
    double* d_scalar = nullptr;  // [0] err sum, [1..] misc
    double* d_rows = nullptr;
    double* h_rows = nullptr;
    StepRec* h_rec = nullptr;
    // fixed-step graphs by (steps, parity, recorder id, dt, rows per block, floor, y, k1, kernel timing)
    std::map<std::tuple<int, int, uint64_t, uint64_t, uint64_t, uint64_t, const void*, const void*, int>, FixedGraph>
        graphs;
    // per-kernel timing of the fixed-step chunks (whole grid, S12 + S3): event
    // nodes around every kernel of the captured graphs; the host accumulates
    // the S12 and S3 durations after each chunk
    int ktiming = 0;
    std::vector<cudaEvent_t> kev;  // 3 per step + 1
    double kt_ms[2] = {0.0, 0.0};  // summed S12, S3 ms
    int64_t kt_n = 0;              // steps timed
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    double last_ms = 0.0;
    int64_t last_kernels = 0;
    // NCCL
    nccl_comm comm = nullptr;
};

// On-device run recorder (io.hpp:107-219 RunRecorder): gauge samples are
// gathered by a kernel into a staging block (captured per step in the
// fixed-step graphs), conservation rows are one fused row-sum pass at the
// stride, snapshots are stream-ordered D2H copies into pinned memory.
struct hsgn_recorder {
    hsgn_ctx* c = nullptr;
    uint64_t id = 0;  // unique per recorder: keys the gauge-sampling graphs (never a reused address)
    std::vector<int32_t> gi, gj;
    std::vector<double> gx, gy;
    long long* d_idx = nullptr;  // j*nx + i per gauge
    double* d_gauge = nullptr;   // staging: gauge_cap rows x n_gauges
    double* h_gauge = nullptr;   // pinned mirror
    int gauge_cap = 0;
    double* d_cons = nullptr;  // 3 x ny row sums (mass, energy, energy rate)
    double* h_cons = nullptr;
    std::vector<double> targets;  // sorted
    size_t next_target = 0;
    int64_t stride = 1;
    bool first = true;
    double prev_t = 0.0;
    int64_t accept_count = 0;
    // results
    std::vector<double> gauge_t, gauge_vals, cons;  // cons: (t, mass, energy, rate) rows
    struct Snap {
        double target, actual;
        double* host;  // pinned, 5 * nx * ny
    };
    std::vector<Snap> snaps;
};

namespace {

hsgn_status fail(hsgn_ctx* c, hsgn_status s, const char* fmt, ...) {
    if (c) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        c->err = buf;
    }
    return s;
}

#define CK(call)                                                                               \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) return fail(c, HSGN_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

// Every entry point runs on its context's device and leaves the caller's
// current device as it found it (torch and other libraries rely on it).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int d) {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur == d) return;  // nothing to switch or restore
        prev = cur;
        cudaSetDevice(d);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};
struct DeviceRestore {  // the group functions switch devices per member
    int prev = -1;
    DeviceRestore() {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    }
    ~DeviceRestore() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

bool is_pow2_ge1(double v) {
    if (!(v >= 1.0) || !std::isfinite(v)) return false;
    int e;
    return std::frexp(v, &e) == 0.5;
}

double spacing(double lo, double hi, int n, int bounded) {  // grid.hpp:43-45
    return bounded ? (hi - lo) / (n - 1) : (hi - lo) / n;
}

// A single-domain context (wrap/clamp y edges, graph-captured fixed steps)
// rather than a slab of a P-rank decomposition (ghost-row edges, halos).
inline bool whole(const hsgn_ctx* c) { return c->nranks == 1 && !c->ring1; }

// Global y edge modes of a slab.
void slab_edges(const hsgn_ctx* c, int* lo, int* hi) {
    const bool yb = c->grid.kind_y == HSGN_BOUNDED;
    if (c->nranks == 1 && !c->ring1) {
        *lo = yb ? YE_CLAMP : YE_WRAP;
        *hi = yb ? YE_CLAMP : YE_WRAP;
        return;
    }
    *lo = (c->j_begin == 0 && yb) ? YE_CLAMP : YE_GHOST;
    *hi = (c->j_end == c->grid.ny && yb) ? YE_CLAMP : YE_GHOST;
}

hsgn_status alloc_state(hsgn_ctx* c, hsgn_state* s) {
    s->fs = c->fs;
    CK(cudaMalloc(&s->base, sizeof(double) * 5 * c->fs));
    CK(cudaMemsetAsync(s->base, 0, sizeof(double) * 5 * c->fs, c->stream));
    s->base += GHOST * c->grid.nx;  // row 0 of field 0 (rows -GHOST..-1 are ghost rows)
    return HSGN_OK;
}

}  // namespace

// Freed pointer must be the allocation base (row -1 of field 0).
static void free_state_c(hsgn_ctx* c, hsgn_state* s) {
    if (s->base) cudaFree(s->base - GHOST * c->grid.nx);
    s->base = nullptr;
}

static hsgn_status setup_ctx(hsgn_ctx* c) {
    const hsgn_grid& g = c->grid;
    c->dx = spacing(g.x_min, g.x_max, g.nx, g.kind_x);
    c->dy = spacing(g.y_min, g.y_max, g.ny, g.kind_y);
    c->ny_loc = c->j_end - c->j_begin;
    c->fs = (long long)(c->ny_loc + 2 * GHOST) * g.nx;
    StageArgs& A = c->base;
    std::memset(&A, 0, sizeof A);
    A.nx = g.nx;
    A.ny = c->ny_loc;
    A.fs = c->fs;
    slab_edges(c, &A.y_lo, &A.y_hi);
    A.x_bounded = g.kind_x == HSGN_BOUNDED;
    A.walls = (g.kind_x == HSGN_BOUNDED) || (g.kind_y == HSGN_BOUNDED);
    A.sat_y_lo = g.kind_y == HSGN_BOUNDED && c->j_begin == 0;
    A.sat_y_hi = g.kind_y == HSGN_BOUNDED && c->j_end == g.ny;
    // sbp.hpp:46,63 (interior), :66 (closure), :254 (SAT); rhs.hpp:143-145
    A.cpx = 1.0 / (2.0 * c->dx);
    A.cpy = 1.0 / (2.0 * c->dy);
    A.c1x = 1.0 / c->dx;
    A.c1y = 1.0 / c->dy;
    A.tdx = 2.0 / c->dx;
    A.tdy = 2.0 / c->dy;
    // stencil kind (sgn_device.cuh sbp_d): 1 = power-of-two coefficients,
    // 2 = additionally one common factor (fully periodic, dx == dy)
    const bool p2 = is_pow2_ge1(A.cpx) && is_pow2_ge1(A.cpy) && A.c1x == 2.0 * A.cpx && A.c1y == 2.0 * A.cpy;
    const bool cf = p2 && A.cpx == A.cpy && !A.x_bounded && A.y_lo != YE_CLAMP && A.y_hi != YE_CLAMP && !A.walls;
    A.pow2 = cf ? 2 : (p2 ? 1 : 0);
    if (c->forced_kind >= 0 && c->forced_kind < A.pow2) A.pow2 = c->forced_kind;
    // magnitude guard of the fast association (sgn_device.cuh lit_node): the
    // constants must be zero or in [2^-60, 2^60], else every row is literal
    auto guard_ok = [](double x) { return x == 0.0 || (std::fabs(x) >= 0x1p-60 && std::fabs(x) <= 0x1p60); };
    // (b, g and lambda matter only under the common factor, stencil kind 2)
    A.lit_all = !(guard_ok(A.cpx) && guard_ok(A.cpy) && guard_ok(A.c1x) && guard_ok(A.c1y)) ||
                (A.pow2 == 2 && (c->b_lit || !guard_ok(c->phys.g) || !guard_ok(c->phys.lambda)));
#ifdef HSGN_FORCE_LIT
    A.lit_all = 1;  // experiments: literal association everywhere
#endif
    A.g = c->phys.g;
    A.lambda = c->phys.lambda;
    A.lam_half = c->phys.lambda / 2.0;
    A.lam_third = c->phys.lambda / 3.0;
    A.lam_sixth = c->phys.lambda / 6.0;
    A.x_min = g.x_min;
    A.y_min = g.y_min;
    A.dx = c->dx;
    A.dy = c->dy;
    A.j_global0 = c->j_begin;
    A.ny_global = g.ny;
    A.y_bounded = g.kind_y == HSGN_BOUNDED;
    A.srcx = c->d_srcx;
    A.srcy = c->d_srcy;
    A.b = c->b;
    A.h_floor = c->phys.h_floor;
    // default launch shape: rows per CTA so that the grid is >= ~6 waves
    A.rows_per_block = c->rows_per_block > 0 ? c->rows_per_block : 0;
    if (A.rows_per_block <= 0) {
        const int tiles_x = (g.nx + 127) / 128;
        int rpb = 128;
        while (rpb > 16 && (long long)tiles_x * ((c->ny_loc + rpb - 1) / rpb) < 148LL * 3 * 6) rpb /= 2;
        A.rows_per_block = rpb;
    }
    {  // literal-pass tile hints: one int per CTA of a whole-slab S12 / per-stage launch
        const long long nb = (c->ny_loc + A.rows_per_block - 1) / A.rows_per_block;
        const long long n12 = (g.nx + 123) / 124 * nb, nst = (g.nx + 125) / 126 * nb;
        if (n12 + nst > c->hint_cap) {
            if (c->d_hint) cudaFree(c->d_hint);
            c->d_hint = nullptr;
            c->hint_cap = 0;
            if (cudaMalloc(&c->d_hint, sizeof(int) * (n12 + nst)) == cudaSuccess) c->hint_cap = n12 + nst;
        }
        if (c->d_hint) cudaMemset(c->d_hint, 0, sizeof(int) * c->hint_cap);
        A.hint_s12 = c->d_hint;
        A.hint_stage = c->d_hint ? c->d_hint + n12 : nullptr;
    }
    AuxArgs& X = c->aux;
    X.nx = g.nx;
    X.ny = c->ny_loc;
    X.fs = c->fs;
    X.y_lo = A.y_lo;
    X.y_hi = A.y_hi;
    X.x_bounded = A.x_bounded;
    X.y_bounded_lo = A.y_lo == YE_CLAMP;
    X.y_bounded_hi = A.y_hi == YE_CLAMP;
    X.pow2 = A.pow2 >= 1;
    X.dx = c->dx;
    X.cpx = A.cpx;
    X.cpy = A.cpy;
    X.c1x = A.c1x;
    X.c1y = A.c1y;
    X.g = c->phys.g;
    X.lambda = c->phys.lambda;
    X.b = c->b;
    return HSGN_OK;
}

// ------------------------------------------------------------------ halo exchange

// After a kernel wrote `s` (rows 0..ny_loc-1), fill the neighbours' ghost
// rows: send rows 0..GHOST-1 to rank-1 (its upper ghost rows) and the last
// GHOST rows to rank+1; receive into our rows -GHOST..-1 / ny_loc..ny_loc+
// GHOST-1.  One grouped NCCL call per exchange, on the context stream
// (graph-capturable).
static hsgn_status exchange_on(hsgn_ctx* c, const hsgn_state* s, int nfields, cudaStream_t stream) {
    if ((c->nranks == 1 && !c->ring1) || c->in_group) return HSGN_OK;  // in a group the driver pulls halos
    if (!c->comm) return fail(c, HSGN_ENCCL, "slab context has no NCCL communicator attached");
    const NcclApi& N = nccl();
    const int nx = c->grid.nx;
    const bool yb = c->grid.kind_y == HSGN_BOUNDED;
    const int up = c->rank + 1 < c->nranks ? c->rank + 1 : (yb ? -1 : 0);
    const int dn = c->rank > 0 ? c->rank - 1 : (yb ? -1 : c->nranks - 1);
    const size_t span = (size_t)GHOST * nx;  // GHOST contiguous rows per field and direction
    // NCCL matches the k-th send to a peer with that peer's k-th receive from
    // us.  With two ranks on a periodic ring (and a 1-rank ring) `up` and `dn`
    // are the same peer, so every rank posts the upward leg (our top rows ->
    // up's lower ghost rows) before the downward leg: the pairs then match
    // for every P, including dn == up.
    int r = N.group_start();
    for (int f = 0; f < nfields && r == 0; ++f) {
        double* fld = s->f(f);
        if (up >= 0) r |= N.send(fld + (long long)(c->ny_loc - GHOST) * nx, span, NCCL_FLOAT64, up, c->comm, stream);
        if (dn >= 0) r |= N.recv(fld - span, span, NCCL_FLOAT64, dn, c->comm, stream);
        if (dn >= 0) r |= N.send(fld, span, NCCL_FLOAT64, dn, c->comm, stream);
        if (up >= 0) r |= N.recv(fld + (long long)c->ny_loc * nx, span, NCCL_FLOAT64, up, c->comm, stream);
    }
    r |= N.group_end();
    if (r) return fail(c, HSGN_ENCCL, "ncclSend/Recv halo exchange failed (%d)", r);
    return HSGN_OK;
}

static hsgn_status exchange(hsgn_ctx* c, const hsgn_state* s, int nfields) {
    return exchange_on(c, s, nfields, c->stream);
}

// Cross-rank agreement of a P-rank decomposition.  Every decision the
// reference takes on a global quantity (depth failures, min depth, the
// adaptive error norm, the start-step norms) must be identical on all ranks,
// or their step sequences -- and the halo exchanges pairing them -- diverge.
// The rank-local device values are summed / min-reduced in place on the
// context stream before the host reads them (graph-capturable, no host sync).
static bool multi_rank(const hsgn_ctx* c) { return c->nranks > 1 && !c->in_group; }

static hsgn_status agree(hsgn_ctx* c, void* d, size_t count, int dtype, int op, cudaStream_t stream = nullptr) {
    if (!multi_rank(c)) return HSGN_OK;
    if (!c->comm) return fail(c, HSGN_ENCCL, "slab context has no NCCL communicator attached");
    const int r = nccl().allreduce(d, d, count, dtype, op, c->comm, stream ? stream : c->stream);
    if (r) return fail(c, HSGN_ENCCL, "ncclAllReduce failed (%d)", r);
    return HSGN_OK;
}

// A step record: depth-failure counts summed, min(ynew.h) bit pattern
// min-reduced (positive doubles order as their bit patterns), one NCCL group.
static hsgn_status agree_rec(hsgn_ctx* c, StepRec* rec, cudaStream_t stream = nullptr) {
    if (!multi_rank(c) || !rec) return HSGN_OK;
    const NcclApi& N = nccl();
    int r = N.group_start();
    hsgn_status s = agree(c, rec->bad, 3, NCCL_UINT64, NCCL_SUM, stream);
    if (!s) s = agree(c, &rec->minh, 1, NCCL_UINT64, NCCL_MIN, stream);
    r |= N.group_end();
    if (s) return s;
    if (r) return fail(c, HSGN_ENCCL, "ncclGroupEnd failed (%d)", r);
    return HSGN_OK;
}

// ------------------------------------------------------------------ stage launch helpers

static StageArgs stage_args(hsgn_ctx* c, int mode, double t) {
    StageArgs A = c->base;  // (mode: for symmetry with launch(); all modes share the base args)
    (void)mode;
    A.source = c->source;
    A.t = t;
    return A;
}

static hsgn_status launch(hsgn_ctx* c, int mode, const StageArgs& A) {
    CK(launch_stage(mode, A, c->stream));
    c->launches += stage_launches(mode, A);
    return HSGN_OK;
}

static hsgn_status gauges_launch(hsgn_ctx* c, const hsgn_state* q, const hsgn_recorder* R, int row) {
    CK(launch_gauges(q->base, c->b, R->d_idx, (int)R->gi.size(), R->d_gauge + (size_t)row * R->gi.size(), c->stream));
    ++c->launches;
    return HSGN_OK;
}

static hsgn_status ensure_recs(hsgn_ctx* c, int rec_cap);

static hsgn_status ensure_ws(hsgn_ctx* c, int rec_cap) {
    if (!c->ws_ready) {
        for (int k = 0; k < 8; ++k) {
            hsgn_status s = alloc_state(c, &c->ws[k]);
            if (s) return s;
        }
        c->ws_ready = true;
    }
    return ensure_recs(c, rec_cap);
}

static hsgn_status ensure_recs(hsgn_ctx* c, int rec_cap) {
    if (!c->d_halt) {
        StageArgs A = c->base;
        c->err_part_cap = stage_grid_blocks(A) + 1;
        c->err_part_cap = std::max(c->err_part_cap, wrms_blocks());
        CK(cudaMalloc(&c->d_err_part, sizeof(double) * c->err_part_cap));
        CK(cudaMalloc(&c->d_scalar, sizeof(double) * 8));
        CK(cudaMalloc(&c->d_halt, sizeof(int) * 4));
    }
    if (rec_cap > c->rec_cap) {
        if (c->d_rec) cudaFree(c->d_rec);
        if (c->h_rec) cudaFreeHost(c->h_rec);
        CK(cudaMalloc(&c->d_rec, sizeof(StepRec) * rec_cap));
        CK(cudaMallocHost(&c->h_rec, sizeof(StepRec) * rec_cap));
        c->rec_cap = rec_cap;
    }
    return HSGN_OK;
}

static void reset_recs(hsgn_ctx* c, int n) {
    // bad counters -> 0, minh -> all-ones ("none"), halt -> 0
    cudaMemsetAsync(c->d_rec, 0xFF, sizeof(StepRec) * n, c->stream);
    for (int s = 0; s < n; ++s) cudaMemsetAsync(&c->d_rec[s].bad[0], 0, sizeof(unsigned long long) * 3, c->stream);
    cudaMemsetAsync(c->d_halt, 0, sizeof(int), c->stream);
}

// Enqueue one fused BS3 step (S1, S2, S3 + halo exchanges) on the stream.
//   y, k1 : step inputs;  ynew, k4 : outputs;  k2 : scratch;  rec : this step's record
//   prev  : previous step's record (halt check) or null
// One stage kernel of a fused BS3 step (stage = 1, 2, 3), without the halo
// exchange of its output (k2, ynew, k4 respectively).
static hsgn_status enqueue_stage(hsgn_ctx* c, int stage, const hsgn_state* y, const hsgn_state* k1, hsgn_state* k2,
                                 hsgn_state* ynew, hsgn_state* k4, hsgn_state* part, StepRec* rec,
                                 const StepRec* prev, double t, double dt, bool adaptive, double atol,
                                 double rtol) {
    StageArgs A;
    if (stage == 1) {  // k2 = f(t + dt/2, y + (dt/2) k1)
        A = stage_args(c, MODE_S1, t + 0.5 * dt);
        A.a = 0.5 * dt;
        A.y = y->base;
        A.k = k1->base;
        A.out = k2->base;
        A.bad = &rec->bad[0];
        A.halt = c->d_halt;
        if (prev)  // the previous step's (agreed) record: any stage failure or the floor
            for (int k = 0; k < 3; ++k) A.chk_bad[k] = &prev->bad[k];
        A.chk_minh = prev ? &prev->minh : nullptr;
        return launch(c, MODE_S1, A);
    }
    if (stage == 3) {  // k4 = f(t + dt, ynew) (FSAL)
        A = stage_args(c, MODE_S3, t + dt);
        A.y = ynew->base;
        A.out = k4->base;
        A.adaptive = adaptive;
        A.d4 = -1.0 / 8.0;
        A.dt = dt;
        A.atol = atol;
        A.rtol = rtol;
        A.part = part ? part->base : nullptr;
        A.yold = y->base;
        A.err_part = c->d_err_part;
        A.bad = &rec->bad[2];
        A.halt = c->d_halt;
        A.chk_bad[0] = &rec->bad[0];
        A.chk_bad[1] = &rec->bad[1];
        return launch(c, MODE_S3, A);
    }
    // stage 2: k3 = f(t + 3dt/4, y + (3dt/4) k2); ynew = y + (2/9 dt) k1 + (1/3 dt) k2 + (4/9 dt) k3
    A = stage_args(c, MODE_S2, t + 0.75 * dt);
    A.a = 0.75 * dt;
    A.c1 = dt * (2.0 / 9.0);
    A.c2 = dt * (1.0 / 3.0);
    A.c3 = dt * (4.0 / 9.0);
    A.y = y->base;
    A.k = k2->base;
    A.kc = k1->base;
    A.out = ynew->base;
    A.adaptive = adaptive;
    A.d1 = -5.0 / 72.0;
    A.d2 = 1.0 / 12.0;
    A.d3 = 1.0 / 9.0;
    A.d4 = -1.0 / 8.0;
    A.part = part ? part->base : nullptr;
    A.bad = &rec->bad[1];
    A.minh = &rec->minh;
    A.halt = c->d_halt;
    A.chk_bad[0] = &rec->bad[0];
    return launch(c, MODE_S2, A);
}

// One fixed step as S12 (stages 1+2: y, k1 -> ynew) then S3 (k4 = f(ynew)).
// Rows [band0, band1) of the slab only (band1 == 0: all rows).
static hsgn_status enqueue_s12(hsgn_ctx* c, const hsgn_state* y, const hsgn_state* k1, hsgn_state* ynew,
                               StepRec* rec, const StepRec* prev, double dt, hsgn_state* part = nullptr,
                               int band0 = 0, int band1 = 0, double t = 0.0) {
    // stage times of the source term (time_integration.hpp:279,281)
    StageArgs A = stage_args(c, MODE_S12, t + 0.5 * dt);
    A.t2 = t + 0.75 * dt;
    A.band0 = band0;
    A.band1 = band1;
    A.a = 0.5 * dt;
    A.a2 = 0.75 * dt;
    A.c1 = dt * (2.0 / 9.0);
    A.c2 = dt * (1.0 / 3.0);
    A.c3 = dt * (4.0 / 9.0);
    A.y = y->base;
    A.k = k1->base;
    A.out = ynew->base;
    A.bad = &rec->bad[0];
    A.bad2 = &rec->bad[1];
    A.minh = &rec->minh;
    A.halt = c->d_halt;
    // halt on the previous step's record: with a P-rank decomposition it is
    // the agreed one, so every rank stops at the same step even when a
    // stage-1 / stage-2 failure was local to another rank
    if (prev)
        for (int k = 0; k < 3; ++k) A.chk_bad[k] = &prev->bad[k];
    A.chk_minh = prev ? &prev->minh : nullptr;
    if (part) {  // adaptive attempt: error partials for the adaptive S3
        A.adaptive = 1;
        A.d1 = -5.0 / 72.0;
        A.d2 = 1.0 / 12.0;
        A.d3 = 1.0 / 9.0;
        A.part = part->base;
    }
    return launch(c, MODE_S12, A);
}

static hsgn_status enqueue_s3_fixed(hsgn_ctx* c, const hsgn_state* ynew, hsgn_state* k4, StepRec* rec, double dt,
                                    int band0 = 0, int band1 = 0, double t = 0.0) {
    StageArgs A = stage_args(c, MODE_S3, t + dt);  // k4 = f(t + dt, ynew), FSAL
    A.band0 = band0;
    A.band1 = band1;
    A.y = ynew->base;
    A.out = k4->base;
    A.bad = &rec->bad[2];
    A.halt = c->d_halt;
    A.chk_bad[0] = &rec->bad[0];
    A.chk_bad[1] = &rec->bad[1];
    return launch(c, MODE_S3, A);
}

// The integrator's double-buffered fixed-step state: step s reads (Y[p],
// K[p]) and writes (Y[p^1], K[p^1]), p = (parity + s) & 1.
struct Bufs {
    hsgn_state* Y[2];
    hsgn_state* K[2];
};

static Bufs ws_bufs(hsgn_ctx* c) { return Bufs{{&c->ws[0], &c->ws[1]}, {&c->ws[2], &c->ws[3]}}; }

#define CKE(call)                                                                              \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) return fail(c, HSGN_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

// Overlapped slab step: the rows that feed or need
// ghost rows run as separate edge-band launches, the halo exchanges and the
// step agreement run on the high-priority comm stream while the interior
// band computes.  Stream C (context stream):
//   S12[0,G) S12[ny-G,ny) -evA-  S12[G,ny-G)  (wait evB) S3[0,G) S3[ny-G,ny) -evC-  S3[G,ny-G) -evE-
// stream M:  (wait evA) exchange ynew -evB-  (wait evC) exchange k4  (wait evE) agree(rec) -evD-
// and the next step's first kernel waits evD (its ghost rows and the agreed
// record).  G = GHOST: the exchanged boundary rows of ynew are written by
// the S12 edge bands and those of k4 by the S3 edge bands, so the interior
// launches never touch a row in flight.
static hsgn_status enqueue_slab_step(hsgn_ctx* c, const Bufs& B, int p, StepRec* rec, const StepRec* prev,
                                     double dt, double t) {
    const int ny = c->ny_loc, G = GHOST;
    hsgn_state *y = B.Y[p], *k1 = B.K[p], *yn = B.Y[p ^ 1], *k4 = B.K[p ^ 1];
    hsgn_status st;
    if (prev) CKE(cudaStreamWaitEvent(c->stream, c->ev_d, 0));
    if ((st = enqueue_s12(c, y, k1, yn, rec, prev, dt, nullptr, 0, G, t))) return st;
    if ((st = enqueue_s12(c, y, k1, yn, rec, prev, dt, nullptr, ny - G, ny, t))) return st;
    CKE(cudaEventRecord(c->ev_a, c->stream));
    CKE(cudaStreamWaitEvent(c->cstream, c->ev_a, 0));
    if ((st = exchange_on(c, yn, 5, c->cstream))) return st;
    CKE(cudaEventRecord(c->ev_b, c->cstream));
    if ((st = enqueue_s12(c, y, k1, yn, rec, prev, dt, nullptr, G, ny - G, t))) return st;
    CKE(cudaStreamWaitEvent(c->stream, c->ev_b, 0));
    if ((st = enqueue_s3_fixed(c, yn, k4, rec, dt, 0, G, t))) return st;
    if ((st = enqueue_s3_fixed(c, yn, k4, rec, dt, ny - G, ny, t))) return st;
    CKE(cudaEventRecord(c->ev_c, c->stream));
    CKE(cudaStreamWaitEvent(c->cstream, c->ev_c, 0));
    if ((st = exchange_on(c, k4, 5, c->cstream))) return st;
    if ((st = enqueue_s3_fixed(c, yn, k4, rec, dt, G, ny - G, t))) return st;
    CKE(cudaEventRecord(c->ev_e, c->stream));
    CKE(cudaStreamWaitEvent(c->cstream, c->ev_e, 0));
    if ((st = agree_rec(c, rec, c->cstream))) return st;  // all stage counters of this step are final
    CKE(cudaEventRecord(c->ev_d, c->cstream));
    return HSGN_OK;
}

static bool slab_overlap(const hsgn_ctx* c) { return !whole(c) && !c->in_group && c->ny_loc >= 3 * GHOST; }

// A chunk of `steps` fixed steps as S12 + S3 per step (+1 gauge gather per
// step with a recorder).  Whole grid: two launches per step.  NCCL slab:
// the overlapped schedule above, or (thin slabs) the exchanges serialised
// after each kernel.  t: time of the first step (source terms only: a chunk
// with a source is launched directly, not captured).
static hsgn_status enqueue_chunk_s12(hsgn_ctx* c, const Bufs& B, int parity, int steps, double dt,
                                     const hsgn_recorder* R, double t = 0.0) {
    const bool gauges = R && !R->gi.empty();
    const bool overlap = slab_overlap(c);
    hsgn_status st;
    for (int s = 0; s < steps; ++s) {
        const int p = (parity + s) & 1;
        StepRec* rec = &c->d_rec[s];
        const StepRec* prev = s ? &c->d_rec[s - 1] : nullptr;
        const double ts = t;
        t = t + dt;  // time_integration.hpp:321
        if (overlap) {
            if ((st = enqueue_slab_step(c, B, p, rec, prev, dt, ts))) return st;
            continue;
        }
        const bool kt = c->ktiming && whole(c);
        // (event record NODES of the captured graph: cudaEventRecordExternal)
        if (kt) CKE(cudaEventRecordWithFlags(c->kev[3 * s], c->stream, cudaEventRecordExternal));
        if ((st = enqueue_s12(c, B.Y[p], B.K[p], B.Y[p ^ 1], rec, prev, dt, nullptr, 0, 0, ts))) return st;
        if (kt) CKE(cudaEventRecordWithFlags(c->kev[3 * s + 1], c->stream, cudaEventRecordExternal));
        if ((st = exchange(c, B.Y[p ^ 1], 5))) return st;
        if (gauges && (st = gauges_launch(c, B.Y[p ^ 1], R, s))) return st;
        if (kt) CKE(cudaEventRecordWithFlags(c->kev[3 * s + 2], c->stream, cudaEventRecordExternal));
        if ((st = enqueue_s3_fixed(c, B.Y[p ^ 1], B.K[p ^ 1], rec, dt, 0, 0, ts))) return st;
        if (kt && s + 1 == steps) CKE(cudaEventRecordWithFlags(c->kev[3 * steps], c->stream, cudaEventRecordExternal));
        if ((st = exchange(c, B.K[p ^ 1], 5))) return st;
        if ((st = agree_rec(c, rec))) return st;  // the next S12 halts on the global record
    }
    if (overlap && steps > 0) CKE(cudaStreamWaitEvent(c->stream, c->ev_d, 0));  // join the comm stream
    return HSGN_OK;
}

// One BS3 step as one kernel per stage (S1, S2, S3) with the slab halo
// exchange after each stage (k2, ynew, k4): DESIGN.md section 6.
static hsgn_status enqueue_step(hsgn_ctx* c, const hsgn_state* y, const hsgn_state* k1, hsgn_state* k2,
                                hsgn_state* ynew, hsgn_state* k4, hsgn_state* part, StepRec* rec,
                                const StepRec* prev, double t, double dt, bool adaptive, double atol,
                                double rtol) {
    hsgn_state* produced[3] = {k2, ynew, k4};
    for (int stage = 1; stage <= 3; ++stage) {
        hsgn_status s = enqueue_stage(c, stage, y, k1, k2, ynew, k4, part, rec, prev, t, dt, adaptive, atol, rtol);
        if (s) return s;
        if ((s = exchange(c, produced[stage - 1], 5))) return s;
    }
    return agree_rec(c, rec);
}

// A chunk of `steps` fixed steps, one kernel per stage (+ gauges); t is the
// time of the first step (the source term needs it; graphs are built only
// without a source).
static hsgn_status enqueue_chunk_stages(hsgn_ctx* c, const Bufs& B, int parity, int steps, double t, double dt,
                                        const hsgn_recorder* R) {
    const bool gauges = R && !R->gi.empty();
    hsgn_status st;
    double ts = t;
    for (int s = 0; s < steps; ++s) {
        const int p = (parity + s) & 1;
        if ((st = enqueue_step(c, B.Y[p], B.K[p], &c->ws[4], B.Y[p ^ 1], B.K[p ^ 1], nullptr, &c->d_rec[s],
                               s ? &c->d_rec[s - 1] : nullptr, ts, dt, false, 0, 0)))
            return st;
        if (gauges && (st = gauges_launch(c, B.Y[p ^ 1], R, s))) return st;
        ts = ts + dt;
    }
    return HSGN_OK;
}

// RHS evaluation into out (no depth pre-check): used by the integrator.
static hsgn_status rhs_raw(hsgn_ctx* c, double t, const hsgn_state* q, hsgn_state* out, bool shallow,
                           unsigned long long* d_bad) {
    StageArgs A = stage_args(c, MODE_RHS, t);
    if (shallow) {
        A.lambda = 0.0;
        A.lam_half = 0.0;
        A.lam_third = 0.0;
        A.lam_sixth = 0.0;
        A.shallow = 1;
    }
    A.y = q->base;
    A.out = out->base;
    A.bad = d_bad;
    ++c->n_evals;
    hsgn_status s = launch(c, MODE_RHS, A);
    if (s) return s;
    return exchange(c, out, 5);
}

static hsgn_status rhs_checked(hsgn_ctx* c, double t, const hsgn_state* q, hsgn_state* out, bool shallow,
                               int64_t* bad_nodes) {
    hsgn_status s = ensure_recs(c, 1);
    if (s) return s;
    unsigned long long* d_bad = &c->d_rec[0].bad[0];
    CK(cudaMemsetAsync(d_bad, 0, sizeof(unsigned long long), c->stream));
    CK(launch_depth_check(q->base, (long long)c->ny_loc * c->grid.nx, d_bad, c->stream));
    ++c->launches;
    if ((s = agree(c, d_bad, 1, NCCL_UINT64, NCCL_SUM))) return s;
    unsigned long long hb = 0;
    CK(cudaMemcpyAsync(&hb, d_bad, sizeof hb, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (bad_nodes) *bad_nodes = (int64_t)hb;
    if (hb) {
        ++c->n_evals;  // rhs.hpp:84 counts the evaluation before throwing
        return fail(c, HSGN_EDEPTH, "tendency evaluation at t = %f: %llu nodes with non-positive depth", t, hb);
    }
    s = rhs_raw(c, t, q, out, shallow, &c->d_rec[0].bad[1]);
    if (s) return s;
    CK(cudaStreamSynchronize(c->stream));
    return HSGN_OK;
}

// ------------------------------------------------------------------ reductions

static hsgn_status row_sums_dev(hsgn_ctx* c, int kind, const hsgn_state* q, const hsgn_state* qt, int field) {
    if (!c->d_rows) {
        CK(cudaMalloc(&c->d_rows, sizeof(double) * c->ny_loc));
        CK(cudaMallocHost(&c->h_rows, sizeof(double) * c->ny_loc));
    }
    CK(launch_row_sums(c->aux, kind, q->base, qt ? qt->base : nullptr, field, c->d_rows, c->stream));
    CK(cudaMemcpyAsync(c->h_rows, c->d_rows, sizeof(double) * c->ny_loc, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return HSGN_OK;
}

static double outer_sum(const hsgn_grid* g, const double* rows, int j_begin, int j_end) {
    // sbp.hpp:232-237: Kahan over wy_j * row_j in row order
    const double dy = spacing(g->y_min, g->y_max, g->ny, g->kind_y);
    double sum = 0.0, comp = 0.0;
    for (int j = j_begin; j < j_end; ++j) {
        double wy = dy;
        if (g->kind_y == HSGN_BOUNDED && (j == 0 || j == g->ny - 1)) wy = 0.5 * dy;
        const double term = wy * rows[j - j_begin] - comp;
        const double t = sum + term;
        comp = (t - sum) - term;
        sum = t;
    }
    return sum;
}

static hsgn_status reduce_full(hsgn_ctx* c, int kind, const hsgn_state* q, const hsgn_state* qt, int field,
                               double* out) {
    DeviceGuard dg_(c->device);
    if (c->nranks != 1)
        return fail(c, HSGN_EINVAL, "slab contexts reduce via hsgn_row_sums + hsgn_outer_sum");
    hsgn_status s = row_sums_dev(c, kind, q, qt, field);
    if (s) return s;
    *out = outer_sum(&c->grid, c->h_rows, 0, c->grid.ny);
    return HSGN_OK;
}

// ------------------------------------------------------------------ C ABI

extern "C" {

const char* hsgn_build_info(void) {
    return "hsgn_b200: fused fp64 SGN split-form stage kernels, sm_100a, --fmad=false";
}

static hsgn_status create_common(const hsgn_grid* grid, const hsgn_phys* phys, const double* b_host, int device,
                                 int j_begin, int j_end, int rank, int nranks, hsgn_ctx** out) {
    DeviceRestore dr_;
    if (!grid || !phys || !b_host || !out) return HSGN_EINVAL;
    *out = nullptr;
    hsgn_ctx* c = new hsgn_ctx();
    c->grid = *grid;
    c->phys = *phys;
    auto bad_arg = [&](const char* msg) {
        // make_grid / make_rhs_context errors (grid.hpp:51-55)
        fprintf(stderr, "hsgn_ctx_create: %s\n", msg);
        delete c;
        return HSGN_EINVAL;
    };
    if (!(grid->x_max > grid->x_min) || !(grid->y_max > grid->y_min))
        return bad_arg("make_grid: domain extents must be increasing");
    if (grid->nx < 4 || grid->ny < 4) return bad_arg("make_grid: need at least 4 nodes per direction");
    if (nranks < 1 || rank < 0 || rank >= nranks || j_begin < 0 || j_end > grid->ny || j_end - j_begin < GHOST)
        return bad_arg("invalid slab");
    if (nranks == 1 && (j_begin != 0 || j_end != grid->ny))  // one rank holds the whole grid
        return bad_arg("invalid slab: a 1-rank decomposition must own rows [0, ny)");
    c->j_begin = j_begin;
    c->j_end = j_end;
    c->rank = rank;
    c->nranks = nranks;
    if (device < 0) cudaGetDevice(&device);
    c->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        fprintf(stderr, "hsgn_ctx_create: %s\n", cudaGetErrorString(e));
        delete c;
        return HSGN_ECUDA;
    }
    const int ny_loc = j_end - j_begin;
    const long long fsz = (long long)(ny_loc + 2 * GHOST) * grid->nx;
    c->b_lit = b_needs_literal(b_host, (long long)ny_loc * grid->nx);
    e = cudaMalloc(&c->b_alloc, sizeof(double) * fsz);
    if (e == cudaSuccess) {
        c->b = c->b_alloc + GHOST * grid->nx;
        e = cudaMemcpyAsync(c->b, b_host, sizeof(double) * ny_loc * grid->nx, cudaMemcpyHostToDevice, c->stream);
    }
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev1);
    if (e != cudaSuccess) {
        fprintf(stderr, "hsgn_ctx_create: %s\n", cudaGetErrorString(e));
        hsgn_ctx_destroy(c);
        return HSGN_ECUDA;
    }
    setup_ctx(c);
    if (nranks == 1) {
        // single slab: fill b's ghost rows for completeness (unused: wrap/clamp)
        cudaStreamSynchronize(c->stream);
    }
    *out = c;
    return HSGN_OK;
}

hsgn_status hsgn_ctx_create(const hsgn_grid* grid, const hsgn_phys* phys, const double* b_host, int device,
                            hsgn_ctx** out) {
    if (!grid) return HSGN_EINVAL;
    return create_common(grid, phys, b_host, device, 0, grid->ny, 0, 1, out);
}

hsgn_status hsgn_ctx_create_slab(const hsgn_grid* grid, const hsgn_phys* phys, const double* b_host, int device,
                                 int32_t j_begin, int32_t j_end, int32_t rank, int32_t nranks, hsgn_ctx** out) {
    return create_common(grid, phys, b_host, device, j_begin, j_end, rank, nranks, out);
}

hsgn_status hsgn_nccl_unique_id(unsigned char out_id[128]) {
    const NcclApi& N = nccl();
    if (!N.ok) return HSGN_ENCCL;
    nccl_uid id;
    if (N.get_uid(&id)) return HSGN_ENCCL;
    std::memcpy(out_id, id.internal, 128);
    return HSGN_OK;
}

hsgn_status hsgn_ctx_attach_nccl(hsgn_ctx* c, const unsigned char nccl_id[128]) {
    if (!c) return HSGN_EINVAL;
    const NcclApi& N = nccl();
    if (!N.ok) return fail(c, HSGN_ENCCL, "libnccl.so.2 not loadable");
    nccl_uid id;
    std::memcpy(id.internal, nccl_id, 128);
    DeviceGuard dg_(c->device);
    int r = N.init_rank(&c->comm, c->nranks, id, c->rank);
    if (r) return fail(c, HSGN_ENCCL, "ncclCommInitRank failed (%d)", r);
    if (!c->cstream) {  // the slab schedule's comm stream: highest priority, so its
                        // NCCL kernels take the next free SM slots of a running interior launch
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithPriority(&c->cstream, cudaStreamNonBlocking, hi));
        for (cudaEvent_t* e : {&c->ev_a, &c->ev_b, &c->ev_c, &c->ev_d, &c->ev_e})
            CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    if (c->nranks == 1 && c->grid.kind_y != HSGN_BOUNDED && !c->ring1) {
        // a 1-rank periodic communicator: the context becomes a 1-slab ring
        // (ghost-row edges, halos sent to itself), i.e. exactly the P-rank
        // code path at P = 1 (the slab schedule without a second GPU)
        if (c->ws_ready || !c->graphs.empty())
            return fail(c, HSGN_EINVAL, "attach the communicator before the first integration");
        c->ring1 = 1;
        setup_ctx(c);  // re-derives the edge modes, stencil kind and launch shape
    }
    // exchange b's ghost rows once (static field)
    hsgn_state bs;
    bs.base = c->b;
    bs.fs = c->fs;
    hsgn_status s = exchange(c, &bs, 1);
    if (s) return s;
    if (multi_rank(c)) {  // the guard's b flag covers every slab (ghost rows come from the neighbours)
        if ((s = ensure_recs(c, 0))) return s;  // d_scalar
        double* d = c->d_scalar;
        const double f = c->b_lit;
        CK(cudaMemcpyAsync(d, &f, sizeof f, cudaMemcpyHostToDevice, c->stream));
        if ((s = agree(c, d, 1, NCCL_FLOAT64, NCCL_MAX))) return s;
        double g = 0.0;
        CK(cudaMemcpyAsync(&g, d, sizeof g, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (g != 0.0 && !c->b_lit) {
            c->b_lit = 1;
            setup_ctx(c);
        }
    }
    CK(cudaStreamSynchronize(c->stream));
    return HSGN_OK;
}

hsgn_status hsgn_ctx_destroy(hsgn_ctx* c) {
    if (!c) return HSGN_OK;
    DeviceGuard dg_(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (auto& kv : c->graphs)
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    if (c->ws_ready)
        for (int k = 0; k < 8; ++k) free_state_c(c, &c->ws[k]);
    if (c->b_alloc) cudaFree(c->b_alloc);
    if (c->d_rec) cudaFree(c->d_rec);
    if (c->h_rec) cudaFreeHost(c->h_rec);
    if (c->d_halt) cudaFree(c->d_halt);
    if (c->d_err_part) cudaFree(c->d_err_part);
    if (c->d_scalar) cudaFree(c->d_scalar);
    if (c->d_hint) cudaFree(c->d_hint);
    if (c->d_srcx) cudaFree(c->d_srcx);
    if (c->d_srcy) cudaFree(c->d_srcy);
    if (c->d_rows) cudaFree(c->d_rows);
    if (c->h_rows) cudaFreeHost(c->h_rows);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    for (cudaEvent_t e : c->kev) cudaEventDestroy(e);
    if (c->comm) nccl().destroy(c->comm);
    for (cudaEvent_t e : {c->ev_a, c->ev_b, c->ev_c, c->ev_d, c->ev_e})
        if (e) cudaEventDestroy(e);
    if (c->cstream) cudaStreamDestroy(c->cstream);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return HSGN_OK;
}

const char* hsgn_last_error(const hsgn_ctx* c) { return c ? c->err.c_str() : "null context"; }

hsgn_status hsgn_set_source(hsgn_ctx* c, int32_t kind) {
    if (!c || kind < 0 || kind > 1) return HSGN_EINVAL;
    if (kind == 1 && !c->d_srcx) {  // the per-column / per-row factors of the source term, once
        DeviceGuard dg_(c->device);
        const hsgn_grid& g = c->grid;
        CK(cudaMalloc(&c->d_srcx, sizeof(double) * 4 * g.nx));
        CK(cudaMalloc(&c->d_srcy, sizeof(double) * 4 * g.ny));
        CK(launch_src_factors(g.x_min, c->dx, g.nx, c->d_srcx, c->stream));
        CK(launch_src_factors(g.y_min, c->dy, g.ny, c->d_srcy, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        c->base.srcx = c->d_srcx;
        c->base.srcy = c->d_srcy;
    }
    c->source = kind;
    return HSGN_OK;
}

static hsgn_status reconfigure(hsgn_ctx* c) {
    DeviceGuard dg_(c->device);
    cudaStreamSynchronize(c->stream);
    setup_ctx(c);
    for (auto& kv : c->graphs)
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    c->graphs.clear();
    if (c->d_err_part) {  // err partial buffer sized by the grid shape
        const int need = std::max(stage_grid_blocks(c->base) + 1, wrms_blocks());
        if (need > c->err_part_cap) {
            cudaFree(c->d_err_part);
            CK(cudaMalloc(&c->d_err_part, sizeof(double) * need));
            c->err_part_cap = need;
        }
    }
    return HSGN_OK;
}

hsgn_status hsgn_set_rows_per_block(hsgn_ctx* c, int32_t rows) {
    if (!c || rows < 0) return HSGN_EINVAL;
    c->rows_per_block = rows;
    return reconfigure(c);
}

hsgn_status hsgn_set_stencil_kind(hsgn_ctx* c, int32_t kind) {
    if (!c || kind < -1 || kind > 2) return HSGN_EINVAL;
    c->forced_kind = kind;
    return reconfigure(c);
}

int32_t hsgn_stencil_kind(const hsgn_ctx* c) { return c ? c->base.pow2 : -1; }

hsgn_status hsgn_set_fused_stages(hsgn_ctx* c, int32_t mode) {
    if (!c || (mode != 0 && mode != 3)) return HSGN_EINVAL;
    c->fused = mode;
    return reconfigure(c);
}

int32_t hsgn_fused_stages(const hsgn_ctx* c) { return c ? c->fused : 0; }

int64_t hsgn_n_evals(const hsgn_ctx* c) { return c ? c->n_evals : 0; }

hsgn_status hsgn_state_alloc(hsgn_ctx* c, hsgn_state** out) {
    if (!c || !out) return HSGN_EINVAL;
    DeviceGuard dg_(c->device);
    hsgn_state* s = new hsgn_state();
    hsgn_status st = alloc_state(c, s);
    if (st) {
        delete s;
        return st;
    }
    CK(cudaStreamSynchronize(c->stream));
    *out = s;
    return HSGN_OK;
}

hsgn_status hsgn_state_free(hsgn_ctx* c, hsgn_state* s) {
    if (!c || !s) return HSGN_EINVAL;
    DeviceGuard dg_(c->device);
    cudaStreamSynchronize(c->stream);
    free_state_c(c, s);
    delete s;
    return HSGN_OK;
}

hsgn_status hsgn_state_upload(hsgn_ctx* c, hsgn_state* s, const double* host) {
    if (!c || !s || !host) return HSGN_EINVAL;
    DeviceGuard dg_(c->device);
    const long long n = (long long)c->ny_loc * c->grid.nx;
    for (int f = 0; f < 5; ++f)
        CK(cudaMemcpyAsync(s->f(f), host + f * n, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    hsgn_status st = exchange(c, s, 5);
    if (st) return st;
    CK(cudaStreamSynchronize(c->stream));
    return HSGN_OK;
}

hsgn_status hsgn_state_download(hsgn_ctx* c, const hsgn_state* s, double* host) {
    if (!c || !s || !host) return HSGN_EINVAL;
    DeviceGuard dg_(c->device);
    const long long n = (long long)c->ny_loc * c->grid.nx;
    for (int f = 0; f < 5; ++f)
        CK(cudaMemcpyAsync(host + f * n, s->f(f), sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return HSGN_OK;
}

hsgn_status hsgn_state_copy(hsgn_ctx* c, const hsgn_state* src, hsgn_state* dst) {
    if (!c || !src || !dst) return HSGN_EINVAL;
    DeviceGuard dg_(c->device);
    CK(cudaMemcpyAsync(dst->base - GHOST * c->grid.nx, src->base - GHOST * c->grid.nx, sizeof(double) * 5 * c->fs,
                       cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return HSGN_OK;
}

hsgn_status hsgn_state_field_ptr(const hsgn_state* s, int32_t f, double** out) {
    if (!s || !out || f < 0 || f > 4) return HSGN_EINVAL;
    *out = s->f(f);
    return HSGN_OK;
}

hsgn_status hsgn_rhs(hsgn_ctx* c, double t, const hsgn_state* q, hsgn_state* out, int64_t* bad_nodes) {
    if (!c || !q || !out) return HSGN_EINVAL;
    DeviceGuard dg_(c->device);
    return rhs_checked(c, t, q, out, false, bad_nodes);
}

hsgn_status hsgn_rhs_shallow_water(hsgn_ctx* c, double t, const hsgn_state* q, hsgn_state* out,
                                   int64_t* bad_nodes) {
    if (!c || !q || !out) return HSGN_EINVAL;
    DeviceGuard dg_(c->device);
    return rhs_checked(c, t, q, out, true, bad_nodes);
}

hsgn_status hsgn_init_auxiliary(hsgn_ctx* c, hsgn_state* q) {
    if (!c || !q) return HSGN_EINVAL;
    DeviceGuard dg_(c->device);
    // u, v ghost rows must be current for the slab y-derivative
    hsgn_status s = exchange(c, q, 3);
    if (s) return s;
    AuxArgs X = c->aux;
    CK(launch_init_aux(X, q->base, c->stream));
    s = exchange(c, q, 5);
    if (s) return s;
    CK(cudaStreamSynchronize(c->stream));
    return HSGN_OK;
}

hsgn_status hsgn_total_mass(hsgn_ctx* c, const hsgn_state* q, double* out) {
    if (!c || !q || !out) return HSGN_EINVAL;
    return reduce_full(c, 0, q, nullptr, 0, out);
}
hsgn_status hsgn_total_energy(hsgn_ctx* c, const hsgn_state* q, double* out) {
    if (!c || !q || !out) return HSGN_EINVAL;
    return reduce_full(c, 1, q, nullptr, 0, out);
}
hsgn_status hsgn_energy_rate(hsgn_ctx* c, const hsgn_state* q, const hsgn_state* qt, double* out) {
    if (!c || !q || !qt || !out) return HSGN_EINVAL;
    return reduce_full(c, 2, q, qt, 0, out);
}
hsgn_status hsgn_mass_weighted_sum(hsgn_ctx* c, const hsgn_state* q, int32_t field, double* out) {
    if (!c || !q || !out || field < 0 || field > 4) return HSGN_EINVAL;
    return reduce_full(c, 0, q, nullptr, field, out);
}
hsgn_status hsgn_discrete_l2_error(hsgn_ctx* c, const hsgn_state* a, const hsgn_state* b, int32_t field,
                                   double* out) {
    if (!c || !a || !b || !out || field < 0 || field > 4) return HSGN_EINVAL;
    double s2 = 0.0;
    hsgn_status st = reduce_full(c, 3, a, b, field, &s2);
    if (st) return st;
    *out = std::sqrt(s2);
    return HSGN_OK;
}
hsgn_status hsgn_row_sums(hsgn_ctx* c, int32_t kind, const hsgn_state* q, const hsgn_state* qt, int32_t field,
                          double* rows_host) {
    if (!c || !q || !rows_host || kind < 0 || kind > 3) return HSGN_EINVAL;
    DeviceGuard dg_(c->device);
    hsgn_status s = row_sums_dev(c, kind, q, qt, field);
    if (s) return s;
    std::memcpy(rows_host, c->h_rows, sizeof(double) * c->ny_loc);
    return HSGN_OK;
}
double hsgn_outer_sum(const hsgn_grid* g, const double* rows, int32_t j_begin, int32_t j_end) {
    return outer_sum(g, rows, j_begin, j_end);
}

hsgn_status hsgn_synchronize(hsgn_ctx* c) {
    if (!c) return HSGN_EINVAL;
    DeviceGuard dg_(c->device);
    CK(cudaStreamSynchronize(c->stream));
    return HSGN_OK;
}

hsgn_status hsgn_last_timing(const hsgn_ctx* c, double* ms, int64_t* kernels) {
    if (!c) return HSGN_EINVAL;
    if (ms) *ms = c->last_ms;
    if (kernels) *kernels = c->last_kernels;
    return HSGN_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ integrator

namespace {

uint64_t bits_of(double v) {
    uint64_t u;
    std::memcpy(&u, &v, 8);
    return u;
}

// Enqueue a chunk of `steps` fixed steps on buffers B from parity `parity`
// in the context's fixed-step structure (records reset first).
hsgn_status enqueue_chunk(hsgn_ctx* c, const Bufs& B, int parity, int steps, double t, double dt,
                          const hsgn_recorder* R) {
    reset_recs(c, steps);
    if (c->fused == 3) return enqueue_chunk_s12(c, B, parity, steps, dt, R, t);
    return enqueue_chunk_stages(c, B, parity, steps, t, dt, R);
}

// Capture (or fetch) a graph of `steps` fixed steps on buffers B from parity
// `parity`; with a recorder that has gauges, each step also samples them
// (row s of the staging block).  Slab contexts capture their NCCL halo
// exchanges, the step agreement and the comm-stream fork / join too.
hsgn_status get_fixed_graph(hsgn_ctx* c, const Bufs& B, int steps, int parity, double dt, const hsgn_recorder* R,
                            FixedGraph** out) {
    const bool gauges = R && !R->gi.empty();
    const int kt = c->ktiming && whole(c) && c->fused == 3;
    auto key = std::make_tuple(steps, parity, gauges ? R->id : 0ull, bits_of(dt), (uint64_t)c->base.rows_per_block,
                               bits_of(c->base.h_floor), (const void*)B.Y[0]->base, (const void*)B.K[0]->base, kt);
    auto it = c->graphs.find(key);
    if (it != c->graphs.end()) {
        *out = &it->second;
        return HSGN_OK;
    }
    cudaGraph_t g = nullptr;
    const int64_t l0 = c->launches;
    while (kt && (int)c->kev.size() < 3 * steps + 1) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        c->kev.push_back(e);
    }
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    hsgn_status st = enqueue_chunk(c, B, parity, steps, 0.0, dt, R);
    cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    if (st) {
        if (g) cudaGraphDestroy(g);
        return st;
    }
    CK(e);
    FixedGraph fg;
    fg.steps = steps;
    fg.kernels = c->launches - l0;
    c->launches = l0;  // captured, not launched: counted when the graph runs
    e = cudaGraphInstantiate(&fg.exec, g, 0);
    cudaGraphDestroy(g);
    CK(e);
    auto res = c->graphs.emplace(key, fg);
    *out = &res.first->second;
    return HSGN_OK;
}

}  // namespace

// Fixed-step chunk runner: runs `steps` steps from (B.Y[parity],
// B.K[parity]) without a source term (one CUDA graph) or with one (direct
// launches, t baked per step).  Returns the number of completed steps and
// the failure kind (0 none, 1 depth at stage k (fail_stage), 2 floor).
static hsgn_status run_fixed_chunk(hsgn_ctx* c, const Bufs& B, int parity, int steps, double t, double dt,
                                   int* done, int* fail_kind, int* fail_stage, const hsgn_recorder* R = nullptr) {
    hsgn_status st;
    if ((st = ensure_ws(c, steps))) return st;
    if (c->source == 0) {
        FixedGraph* fg = nullptr;
        if ((st = get_fixed_graph(c, B, steps, parity, dt, R, &fg))) return st;
        CK(cudaGraphLaunch(fg->exec, c->stream));
        c->launches += fg->kernels;
    } else if ((st = enqueue_chunk(c, B, parity, steps, t, dt, R))) {
        return st;
    }
    CK(cudaMemcpyAsync(c->h_rec, c->d_rec, sizeof(StepRec) * steps, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (c->ktiming && whole(c) && c->fused == 3 && c->source == 0) {  // the chunk's event nodes have fired
        for (int s = 0; s < steps; ++s) {
            float a = 0.f, b = 0.f;
            CK(cudaEventElapsedTime(&a, c->kev[3 * s], c->kev[3 * s + 1]));
            CK(cudaEventElapsedTime(&b, c->kev[3 * s + 2], c->kev[3 * s + 3]));
            c->kt_ms[0] += a;
            c->kt_ms[1] += b;
        }
        c->kt_n += steps;
    }
    *done = steps;
    *fail_kind = 0;
    for (int s = 0; s < steps; ++s) {
        const StepRec& r = c->h_rec[s];
        for (int k = 0; k < 3; ++k)
            if (r.bad[k]) {
                *done = s;
                *fail_kind = 1;
                *fail_stage = k;
                return HSGN_OK;
            }
        double mh;
        std::memcpy(&mh, &r.minh, 8);
        if (r.minh != ~0ull && mh <= c->base.h_floor) {  // the run's floor (IntegratorConfig::h_floor)
            *done = s;
            *fail_kind = 2;
            return HSGN_OK;
        }
    }
    return HSGN_OK;
}

static double smin(double a, double b) { return (b < a) ? b : a; }
static double smax(double a, double b) { return (a < b) ? b : a; }
static double sclamp(double v, double lo, double hi) { return (v < lo) ? lo : (hi < v) ? hi : v; }

// weighted_rms on device (time_integration.hpp:144-162)
static hsgn_status wrms(hsgn_ctx* c, const hsgn_state* x, const hsgn_state* ref, double atol, double rtol,
                        double* out) {
    const long long n = (long long)c->ny_loc * c->grid.nx;
    CK(launch_wrms(x->base, ref->base, atol, rtol, n, c->fs, c->d_err_part, c->stream));
    CK(launch_sum_partials(c->d_err_part, wrms_blocks(), c->d_scalar, c->stream));
    c->launches += 2;
    hsgn_status st = agree(c, c->d_scalar, 1, NCCL_FLOAT64, NCCL_SUM);
    if (st) return st;
    double s = 0;
    CK(cudaMemcpyAsync(&s, c->d_scalar, sizeof s, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    *out = std::sqrt(s / (5.0 * (double)c->grid.nx * (double)c->grid.ny));  // global node count
    return HSGN_OK;
}

// Depth-checked RHS into out: returns HSGN_EDEPTH (out garbage) on failure.
static hsgn_status rhs_eval(hsgn_ctx* c, double t, const hsgn_state* q, hsgn_state* out) {
    unsigned long long* d_bad = &c->d_rec[0].bad[0];
    CK(cudaMemsetAsync(d_bad, 0, sizeof(unsigned long long), c->stream));
    hsgn_status s = rhs_raw(c, t, q, out, false, d_bad);
    if (s) return s;
    if ((s = agree(c, d_bad, 1, NCCL_UINT64, NCCL_SUM))) return s;
    unsigned long long hb = 0;
    CK(cudaMemcpyAsync(&hb, d_bad, sizeof hb, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (hb) return fail(c, HSGN_EDEPTH, "tendency evaluation at t = %f: %llu nodes with non-positive depth", t, hb);
    return HSGN_OK;
}

// ------------------------------------------------------------------ recorder

// Append `rows` staged gauge rows (sample times ts[0..rows)) to the series.
static hsgn_status rec_collect_gauges(hsgn_recorder* R, const double* ts, int rows) {
    hsgn_ctx* c = R->c;
    const size_t ng = R->gi.size();
    if (!ng || rows <= 0) return HSGN_OK;
    CK(cudaMemcpyAsync(R->h_gauge, R->d_gauge, sizeof(double) * ng * rows, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int s = 0; s < rows; ++s) {
        R->gauge_t.push_back(ts[s]);
        R->gauge_vals.insert(R->gauge_vals.end(), R->h_gauge + s * ng, R->h_gauge + (s + 1) * ng);
    }
    return HSGN_OK;
}

// Sample the gauges of q at time t (one row, staged then collected).
static hsgn_status rec_gauges_now(hsgn_recorder* R, double t, const hsgn_state* q) {
    hsgn_ctx* c = R->c;
    if (R->gi.empty()) return HSGN_OK;
    CK(launch_gauges(q->base, c->b, R->d_idx, (int)R->gi.size(), R->d_gauge, c->stream));
    ++c->launches;
    return rec_collect_gauges(R, &t, 1);
}

// take_snapshot (io.hpp:197-204): stream-ordered copy into pinned memory; the
// host does not wait (the CSV is written by the caller from the copy).
static hsgn_status rec_snapshot(hsgn_recorder* R, double target, double actual, const hsgn_state* q) {
    hsgn_ctx* c = R->c;
    const size_t n = (size_t)c->grid.nx * c->ny_loc;
    hsgn_recorder::Snap sn{target, actual, nullptr};
    CK(cudaMallocHost(&sn.host, sizeof(double) * 5 * n));
    R->snaps.push_back(sn);
    for (int f = 0; f < 5; ++f)
        CK(cudaMemcpyAsync(sn.host + f * n, q->f(f), sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    return HSGN_OK;
}

// RunRecorder::on_accept (io.hpp:120-152) for the state q (tendency qt) at
// time t; prev is the previously accepted state (the other buffer of the
// integrator's pair).  The gauge row is sampled by the caller.
static hsgn_status rec_accept(hsgn_recorder* R, double t, const hsgn_state* q, const hsgn_state* qt,
                              const hsgn_state* prev) {
    hsgn_ctx* c = R->c;
    hsgn_status st;
    if (R->first) {
        R->first = false;
        R->prev_t = t;
        while (R->next_target < R->targets.size() && R->targets[R->next_target] <= t)
            if ((st = rec_snapshot(R, R->targets[R->next_target++], t, q))) return st;
    } else {
        while (R->next_target < R->targets.size() && R->targets[R->next_target] <= t) {
            const double target = R->targets[R->next_target++];
            const bool prev_closer = target - R->prev_t < t - target;
            if ((st = rec_snapshot(R, target, prev_closer ? R->prev_t : t, prev_closer ? prev : q))) return st;
        }
        R->prev_t = t;
    }
    if (R->accept_count % R->stride == 0) {
        const int ny = c->ny_loc;
        CK(launch_cons_rows(c->aux, q->base, qt->base, R->d_cons, c->stream));
        ++c->launches;
        CK(cudaMemcpyAsync(R->h_cons, R->d_cons, sizeof(double) * 3 * ny, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        R->cons.push_back(t);
        for (int k = 0; k < 3; ++k) R->cons.push_back(outer_sum(&c->grid, R->h_cons + (size_t)k * ny, 0, ny));
    }
    ++R->accept_count;
    return HSGN_OK;
}

extern "C" hsgn_status hsgn_solve(hsgn_ctx* c, const hsgn_state* q0, double t0, double t_final, const hsgn_cfg* cfg,
                                  hsgn_state* q_out, hsgn_record* rec, hsgn_observer obs, void* user) {
    return hsgn_solve_recorded(c, q0, t0, t_final, cfg, q_out, rec, obs, user, nullptr);
}

extern "C" hsgn_status hsgn_solve_recorded(hsgn_ctx* c, const hsgn_state* q0, double t0, double t_final,
                                           const hsgn_cfg* cfg, hsgn_state* q_out, hsgn_record* rec,
                                           hsgn_observer obs, void* user, hsgn_recorder* R) {
    if (!c || !q0 || !cfg || !q_out || !rec) return HSGN_EINVAL;
    if (R && R->c != c) return fail(c, HSGN_EINVAL, "recorder belongs to another context");
    DeviceGuard dg_(c->device);
    std::memset(rec, 0, sizeof *rec);
    rec->t = t0;
    hsgn_status st;
    const int CHUNK = 64;
    const int64_t l0 = c->launches;
    if ((st = ensure_ws(c, CHUNK))) return st;
    c->base.h_floor = cfg->h_floor;  // the stage kernels' halt test and the chunk scan use the run's floor
    auto copy_state = [&](const hsgn_state* src, hsgn_state* dst) -> hsgn_status {
        CK(cudaMemcpyAsync(dst->base - GHOST * c->grid.nx, src->base - GHOST * c->grid.nx, sizeof(double) * 5 * c->fs,
                           cudaMemcpyDeviceToDevice, c->stream));
        return HSGN_OK;
    };
    if (!(t_final > t0)) {
        if ((st = copy_state(q0, q_out))) return st;
        CK(cudaStreamSynchronize(c->stream));
        if (t_final == t0) return HSGN_OK;
        rec->aborted = 1;
        snprintf(rec->reason, sizeof rec->reason, "t_final precedes t0");
        return HSGN_OK;
    }
    // buffers: y = B.Y[p], k1 = B.K[p], k2 = ws[4], part = ws[5], scratch ws[6], ws[7].
    // The caller's output state is the integrator's parity-0 y buffer (one
    // copy of q0 in, none out after an even number of accepted steps).
    Bufs B = ws_bufs(c);
    if (q_out != q0) B.Y[0] = q_out;
    int p = 0;
    if ((st = copy_state(q0, B.Y[0]))) return st;
    double t = t0;
    auto abort_with = [&](const char* why) -> hsgn_status {
        if (B.Y[p] != q_out) {
            hsgn_status s2 = copy_state(B.Y[p], q_out);
            if (s2) return s2;
        }
        CK(cudaStreamSynchronize(c->stream));
        rec->t = t;
        rec->aborted = 1;
        snprintf(rec->reason, sizeof rec->reason, "%s", why);
        return HSGN_OK;
    };
    char why[256];
    st = rhs_eval(c, t, B.Y[0], B.K[0]);
    if (st == HSGN_EDEPTH) {
        snprintf(why, sizeof why, "initial tendency: %s", c->err.c_str());
        return abort_with(why);
    }
    if (st) return st;
    ++rec->rhs_evals;

    double dt;
    const bool fixed = cfg->fixed_dt > 0.0;
    if (fixed)
        dt = cfg->fixed_dt;
    else if (cfg->dt_initial > 0.0)
        dt = smin(cfg->dt_initial, smin(cfg->dt_max, t_final - t0));
    else {
        // estimate_initial_dt (time_integration.hpp:170-203)
        const double dt_cap = smin(cfg->dt_max, t_final - t0);
        double d0, d1;
        if ((st = wrms(c, B.Y[0], B.Y[0], cfg->abs_tol, cfg->rel_tol, &d0))) return st;
        if ((st = wrms(c, B.K[0], B.Y[0], cfg->abs_tol, cfg->rel_tol, &d1))) return st;
        if (d1 == 0.0) {
            dt = dt_cap;
        } else {
            double h0 = (d0 >= 1e-5 && d1 >= 1e-5) ? 0.01 * d0 / d1 : 1e-6;
            h0 = smin(h0, dt_cap);
            const long long n = (long long)c->ny_loc * c->grid.nx;
            CK(launch_axpy5(B.Y[0]->base, h0, B.K[0]->base, c->ws[6].base, n, c->fs, c->stream));
            ++c->launches;
            if ((st = exchange(c, &c->ws[6], 5))) return st;
            double d2 = 0.0;
            bool probed = false;
            st = rhs_eval(c, t0 + h0, &c->ws[6], &c->ws[7]);
            if (st == HSGN_OK) {
                ++rec->rhs_evals_setup;
                CK(launch_axpy5(c->ws[7].base, -1.0, B.K[0]->base, c->ws[6].base, n, c->fs, c->stream));
                ++c->launches;
                double r;
                if ((st = wrms(c, &c->ws[6], B.Y[0], cfg->abs_tol, cfg->rel_tol, &r))) return st;
                d2 = r / h0;
                probed = true;
            } else if (st != HSGN_EDEPTH) {
                return st;
            }
            double h1;
            const double dmax = smax(d1, d2);
            if (!probed || dmax <= 1e-15)
                h1 = smax(1e-6, h0 * 1e-3);
            else
                h1 = std::pow(0.01 / dmax, 1.0 / 3.0);
            double r = 100.0 * h0;
            if (h1 < r) r = h1;
            if (dt_cap < r) r = dt_cap;
            dt = r;
        }
        rec->rhs_evals += rec->rhs_evals_setup;
    }
    if (R) {
        if ((st = rec_gauges_now(R, t, B.Y[0]))) return st;
        if ((st = rec_accept(R, t, B.Y[0], B.K[0], nullptr))) return st;
    }
    if (obs) {
        CK(cudaStreamSynchronize(c->stream));
        obs(t, B.Y[0], B.K[0], user);
    }

    const double order_exp = 1.0 / 3.0;
    double err_prev = 1.0;
    const double tiny = 4.0 * std::numeric_limits<double>::epsilon();

    while (t < t_final - tiny * smax(1.0, std::fabs(t_final))) {
        if (rec->accepted + rec->rejected >= cfg->max_steps) {
            snprintf(why, sizeof why, "step budget exhausted at t = %f", t);
            return abort_with(why);
        }
        const bool clipped = dt >= t_final - t;
        if (clipped) dt = t_final - t;
        if (!(dt > tiny * smax(1.0, std::fabs(t)))) {
            snprintf(why, sizeof why, "step size underflow at t = %f", t);
            return abort_with(why);
        }
        if (fixed && !obs && !clipped) {
            // plan a chunk of unclipped steps: replicate the host t sequence exactly.
            // With a recorder the chunk ends at the next conservation record or
            // at the step that crosses the next snapshot target, so recorder
            // work inside a chunk is only the (graph-captured) gauge sample.
            int cap = CHUNK;
            if (R) {
                const int64_t k = R->accept_count, krec = (k + R->stride - 1) / R->stride * R->stride;
                cap = (int)std::min<int64_t>(cap, krec - k + 1);
            }
            int n = 0;
            double tt = t;
            double ts[CHUNK];
            while (n < cap && rec->accepted + rec->rejected + n < cfg->max_steps &&
                   tt < t_final - tiny * smax(1.0, std::fabs(t_final)) && !(dt >= t_final - tt) &&
                   (dt > tiny * smax(1.0, std::fabs(tt)))) {
                tt = tt + dt;
                ts[n++] = tt;
                if (R && R->next_target < R->targets.size() && R->targets[R->next_target] <= tt) break;
            }
            if (n >= 2) {
                if ((n & 1) && !R) --n;  // even chunks keep the buffer parity (fewer graphs)
                int done = 0, fk = 0, fs_ = 0;
                if ((st = run_fixed_chunk(c, B, p, n, t, dt, &done, &fk, &fs_, R))) return st;
                for (int s = 0; s < done; ++s) {
                    t = t + dt;
                    ++rec->accepted;
                    rec->rhs_evals += 3;
                    p ^= 1;
                }
                c->n_evals += 3 * (int64_t)done;
                if (R) {
                    if ((st = rec_collect_gauges(R, ts, done))) return st;
                    if (done == n) {  // steps 1..n-1 carry no record by construction
                        R->accept_count += n - 1;
                        R->prev_t = ts[n - 2];
                        if ((st = rec_accept(R, t, B.Y[p], B.K[p], B.Y[p ^ 1]))) return st;
                    } else {
                        R->accept_count += done;
                    }
                }
                if (fk) {
                    if (fk == 1) {
                        rec->rhs_evals += fs_;
                        c->n_evals += fs_ + 1;
                        snprintf(why, sizeof why, "non-positive depth in fixed-step mode at t = %f", t);
                    } else {
                        rec->rhs_evals += 3;
                        c->n_evals += 3;
                        snprintf(why, sizeof why, "depth reached the floor %f during the step to t = %f",
                                 cfg->h_floor, t + dt);
                    }
                    return abort_with(why);
                }
                continue;
            }
        }
        // ---- one attempt (adaptive, clipped or observed step)
        const int q = p ^ 1;
        reset_recs(c, 1);
        if (c->fused == 3) {  // S12 + S3 (with error partials when adaptive)
            st = enqueue_s12(c, B.Y[p], B.K[p], B.Y[q], &c->d_rec[0], nullptr, dt, fixed ? nullptr : &c->ws[5], 0, 0,
                             t);
            if (!st) st = exchange(c, B.Y[q], 5);
            if (!st)
                st = enqueue_stage(c, 3, B.Y[p], B.K[p], &c->ws[4], B.Y[q], B.K[q], &c->ws[5], &c->d_rec[0], nullptr, t,
                                   dt, !fixed, cfg->abs_tol, cfg->rel_tol);
            if (!st) st = exchange(c, B.K[q], 5);
            if (!st) st = agree_rec(c, &c->d_rec[0]);
        } else {
            st = enqueue_step(c, B.Y[p], B.K[p], &c->ws[4], B.Y[q], B.K[q], &c->ws[5], &c->d_rec[0], nullptr, t, dt,
                              !fixed, cfg->abs_tol, cfg->rel_tol);
        }
        if (st) return st;
        if (!fixed) {
            CK(launch_sum_partials(c->d_err_part, stage_grid_blocks(c->base), c->d_scalar, c->stream));
            ++c->launches;
            if ((st = agree(c, c->d_scalar, 1, NCCL_FLOAT64, NCCL_SUM))) return st;
        }
        StepRec r;
        double err_sum = 0.0;
        CK(cudaMemcpyAsync(&r, &c->d_rec[0], sizeof r, cudaMemcpyDeviceToHost, c->stream));
        if (!fixed) CK(cudaMemcpyAsync(&err_sum, c->d_scalar, sizeof err_sum, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        int fail_stage = -1;
        for (int k = 0; k < 3 && fail_stage < 0; ++k)
            if (r.bad[k]) fail_stage = k;
        c->n_evals += fail_stage < 0 ? 3 : fail_stage + 1;
        if (fail_stage >= 0) {
            rec->rhs_evals += fail_stage;
            if (fixed) {
                snprintf(why, sizeof why, "non-positive depth in fixed-step mode at t = %f", t);
                return abort_with(why);
            }
            ++rec->rejected;
            dt *= 0.25;
            continue;
        }
        rec->rhs_evals += 3;
        double err = 0.0, min_h = std::numeric_limits<double>::infinity();
        if (r.minh != ~0ull) std::memcpy(&min_h, &r.minh, 8);
        if (!fixed) {
            const double n5 = 5.0 * (double)c->grid.nx * (double)c->grid.ny;  // global node count
            err = std::sqrt(err_sum / n5);
        }
        const bool accept = fixed || err <= 1.0;
        if (accept) {
            if (min_h <= cfg->h_floor) {
                snprintf(why, sizeof why, "depth reached the floor %f during the step to t = %f", cfg->h_floor,
                         t + dt);
                return abort_with(why);
            }
            p = q;  // swap(y, ynew); swap(k1, k4)
            t = clipped ? t_final : t + dt;
            ++rec->accepted;
            if (!fixed) {
                double fac;
                if (err == 0.0)
                    fac = cfg->growth_cap;
                else
                    fac = cfg->safety * std::pow(err, -0.7 * order_exp) * std::pow(err_prev, 0.4 * order_exp);
                fac = sclamp(fac, cfg->shrink_floor, cfg->growth_cap);
                dt = smin(dt * fac, cfg->dt_max);
                err_prev = smax(err, 1e-10);
            }
            if (R) {
                if ((st = rec_gauges_now(R, t, B.Y[p]))) return st;
                if ((st = rec_accept(R, t, B.Y[p], B.K[p], B.Y[p ^ 1]))) return st;
            }
            if (obs) obs(t, B.Y[p], B.K[p], user);
        } else {
            ++rec->rejected;
            const double fac = std::isfinite(err) ? sclamp(cfg->safety * std::pow(err, -order_exp), 0.1, 0.9) : 0.1;
            dt *= fac;
        }
    }
    if (B.Y[p] != q_out && (st = copy_state(B.Y[p], q_out))) return st;
    CK(cudaStreamSynchronize(c->stream));
    rec->t = t;
    c->last_kernels = c->launches - l0;
    return HSGN_OK;
}

extern "C" hsgn_status hsgn_recorder_create(hsgn_ctx* c, int32_t n_gauges, const double* gauge_xy,
                                            int32_t n_targets, const double* targets, int64_t conservation_stride,
                                            hsgn_recorder** out) {
    if (!c || !out || n_gauges < 0 || n_targets < 0 || (n_gauges && !gauge_xy) || (n_targets && !targets))
        return HSGN_EINVAL;
    *out = nullptr;
    if (conservation_stride < 1)  // config.hpp:234-237
        return fail(c, HSGN_EINVAL, "conservation_stride must be >= 1");
    if (!whole(c)) return fail(c, HSGN_EINVAL, "the recorder needs a whole-grid context");
    DeviceGuard dg_(c->device);
    hsgn_recorder* R = new hsgn_recorder;
    static uint64_t next_id = 0;
    R->c = c;
    R->id = ++next_id;
    R->stride = conservation_stride;
    const hsgn_grid& g = c->grid;
    std::vector<long long> idx;
    for (int k = 0; k < n_gauges; ++k) {  // nearest_node (io.hpp:38-48)
        const double x = gauge_xy[2 * k], y = gauge_xy[2 * k + 1];
        const int i = std::clamp(static_cast<int>(std::lround((x - g.x_min) / c->dx)), 0, g.nx - 1);
        const int j = std::clamp(static_cast<int>(std::lround((y - g.y_min) / c->dy)), 0, g.ny - 1);
        R->gi.push_back(i);
        R->gj.push_back(j);
        R->gx.push_back(g.x_min + i * c->dx);  // Grid2D::x / y (grid.hpp:24-25)
        R->gy.push_back(g.y_min + j * c->dy);
        idx.push_back((long long)j * g.nx + i);
    }
    R->targets.assign(targets, targets + n_targets);
    std::sort(R->targets.begin(), R->targets.end());
    auto cleanup_fail = [&](cudaError_t e) {
        hsgn_recorder_destroy(R);
        return fail(c, HSGN_ECUDA, "recorder allocation: %s", cudaGetErrorString(e));
    };
    cudaError_t e;
    R->gauge_cap = 64;  // >= the fixed-step chunk
    if (n_gauges) {
        if ((e = cudaMalloc(&R->d_idx, sizeof(long long) * n_gauges))) return cleanup_fail(e);
        if ((e = cudaMemcpy(R->d_idx, idx.data(), sizeof(long long) * n_gauges, cudaMemcpyHostToDevice)))
            return cleanup_fail(e);
        if ((e = cudaMalloc(&R->d_gauge, sizeof(double) * n_gauges * R->gauge_cap))) return cleanup_fail(e);
        if ((e = cudaMallocHost(&R->h_gauge, sizeof(double) * n_gauges * R->gauge_cap))) return cleanup_fail(e);
    }
    if ((e = cudaMalloc(&R->d_cons, sizeof(double) * 3 * c->ny_loc))) return cleanup_fail(e);
    if ((e = cudaMallocHost(&R->h_cons, sizeof(double) * 3 * c->ny_loc))) return cleanup_fail(e);
    *out = R;
    return HSGN_OK;
}

extern "C" hsgn_status hsgn_recorder_destroy(hsgn_recorder* R) {
    if (!R) return HSGN_OK;
    DeviceRestore dr_;
    if (R->c) cudaSetDevice(R->c->device);
    if (R->c) {
        cudaStreamSynchronize(R->c->stream);  // pending snapshot copies
        // the gauge-sampling graphs captured this recorder's buffers
        for (auto it = R->c->graphs.begin(); it != R->c->graphs.end();) {
            if (std::get<2>(it->first) == R->id) {
                cudaGraphExecDestroy(it->second.exec);
                it = R->c->graphs.erase(it);
            } else {
                ++it;
            }
        }
    }
    cudaFree(R->d_idx);
    cudaFree(R->d_gauge);
    cudaFreeHost(R->h_gauge);
    cudaFree(R->d_cons);
    cudaFreeHost(R->h_cons);
    for (auto& s : R->snaps) cudaFreeHost(s.host);
    delete R;
    return HSGN_OK;
}

extern "C" hsgn_status hsgn_recorder_counts(const hsgn_recorder* R, int64_t* gauge_rows, int64_t* cons_rows,
                                            int32_t* snapshots) {
    if (!R) return HSGN_EINVAL;
    if (gauge_rows) *gauge_rows = (int64_t)R->gauge_t.size();
    if (cons_rows) *cons_rows = (int64_t)(R->cons.size() / 4);
    if (snapshots) *snapshots = (int32_t)R->snaps.size();
    return HSGN_OK;
}

extern "C" hsgn_status hsgn_recorder_gauge_node(const hsgn_recorder* R, int32_t k, int32_t* i, int32_t* j, double* x,
                                                double* y) {
    if (!R || k < 0 || k >= (int32_t)R->gi.size()) return HSGN_EINVAL;
    if (i) *i = R->gi[k];
    if (j) *j = R->gj[k];
    if (x) *x = R->gx[k];
    if (y) *y = R->gy[k];
    return HSGN_OK;
}

extern "C" hsgn_status hsgn_recorder_gauges(const hsgn_recorder* R, double* t, double* values) {
    if (!R) return HSGN_EINVAL;
    if (t) std::copy(R->gauge_t.begin(), R->gauge_t.end(), t);
    if (values) std::copy(R->gauge_vals.begin(), R->gauge_vals.end(), values);
    return HSGN_OK;
}

extern "C" hsgn_status hsgn_recorder_conservation(const hsgn_recorder* R, double* rows4) {
    if (!R || !rows4) return HSGN_EINVAL;
    std::copy(R->cons.begin(), R->cons.end(), rows4);
    return HSGN_OK;
}

extern "C" hsgn_status hsgn_recorder_snapshot(const hsgn_recorder* R, int32_t k, double* target, double* actual,
                                              double* host_state) {
    if (!R || k < 0 || k >= (int32_t)R->snaps.size()) return HSGN_EINVAL;
    const auto& s = R->snaps[k];
    if (target) *target = s.target;
    if (actual) *actual = s.actual;
    if (host_state) {
        hsgn_ctx* c = R->c;
        DeviceGuard dg_(c->device);
        CK(cudaStreamSynchronize(c->stream));  // the stream-ordered copy has landed
        std::memcpy(host_state, s.host, sizeof(double) * 5 * (size_t)c->grid.nx * c->ny_loc);
    }
    return HSGN_OK;
}

// The buffers of hsgn_bs3_fixed_steps: the caller's (y, k1) are parity 0,
// the workspace pair parity 1, so an even number of steps ends in place.
static Bufs caller_bufs(hsgn_ctx* c, hsgn_state* y, hsgn_state* k1) {
    return Bufs{{y, &c->ws[1]}, {k1, &c->ws[3]}};
}

static const int FIXED_CHUNK = 64;  // steps per captured graph of hsgn_bs3_fixed_steps

extern "C" hsgn_status hsgn_prepare_fixed_steps(hsgn_ctx* c, hsgn_state* y, hsgn_state* k1, double dt,
                                                int64_t steps) {
    if (!c || !y || !k1 || steps < 0) return HSGN_EINVAL;
    DeviceGuard dg_(c->device);
    hsgn_status st;
    if ((st = ensure_ws(c, FIXED_CHUNK))) return st;
    if (c->source) return HSGN_OK;  // direct launches: nothing to build
    c->base.h_floor = c->phys.h_floor;
    const Bufs B = caller_bufs(c, y, k1);
    int p = 0;
    for (int64_t left = steps; left > 0;) {  // the chunk sequence of hsgn_bs3_fixed_steps
        const int n = (int)std::min<int64_t>(FIXED_CHUNK, left);
        FixedGraph* fg = nullptr;
        if ((st = get_fixed_graph(c, B, n, p, dt, nullptr, &fg))) return st;
        left -= n;
        p ^= n & 1;
    }
    return HSGN_OK;
}

extern "C" hsgn_status hsgn_bs3_fixed_steps(hsgn_ctx* c, hsgn_state* y, hsgn_state* k1, double t, double dt,
                                            int64_t steps, int64_t* steps_done) {
    if (!c || !y || !k1 || steps < 0) return HSGN_EINVAL;
    DeviceGuard dg_(c->device);
    hsgn_status st;
    if ((st = ensure_ws(c, FIXED_CHUNK))) return st;
    c->base.h_floor = c->phys.h_floor;
    // in place on the caller's buffers (workspace pair for odd steps); the
    // event window covers everything the call does on the device
    const Bufs B = caller_bufs(c, y, k1);
    int p = 0;
    int64_t done_total = 0;
    const int64_t l0 = c->launches;
    c->kt_ms[0] = c->kt_ms[1] = 0.0;
    c->kt_n = 0;
    CK(cudaEventRecord(c->ev0, c->stream));
    hsgn_status result = HSGN_OK;
    while (done_total < steps) {
        const int n = (int)std::min<int64_t>(FIXED_CHUNK, steps - done_total);
        int done = 0, fk = 0, fs_ = 0;
        if ((st = run_fixed_chunk(c, B, p, n, t, dt, &done, &fk, &fs_))) return st;
        for (int s = 0; s < done; ++s) {
            t = t + dt;
            p ^= 1;
        }
        done_total += done;
        c->n_evals += 3 * (int64_t)done;
        if (fk == 1) {
            result = fail(c, HSGN_EDEPTH, "non-positive depth in fixed-step mode at t = %f", t);
            break;
        }
        if (fk == 2) {
            result = fail(c, HSGN_EDEPTH, "depth reached the floor %f during the step to t = %f", c->phys.h_floor,
                          t + dt);
            break;
        }
    }
    if (p) {  // odd number of completed steps: the last state is in the workspace pair
        CK(cudaMemcpyAsync(y->base - GHOST * c->grid.nx, B.Y[1]->base - GHOST * c->grid.nx,
                           sizeof(double) * 5 * c->fs, cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaMemcpyAsync(k1->base - GHOST * c->grid.nx, B.K[1]->base - GHOST * c->grid.nx,
                           sizeof(double) * 5 * c->fs, cudaMemcpyDeviceToDevice, c->stream));
    }
    CK(cudaEventRecord(c->ev1, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    c->last_ms = ms;
    c->last_kernels = c->launches - l0;
    if (steps_done) *steps_done = done_total;
    return result;
}

extern "C" hsgn_status hsgn_set_kernel_timing(hsgn_ctx* c, int32_t on) {
    if (!c) return HSGN_EINVAL;
    c->ktiming = on ? 1 : 0;
    return HSGN_OK;
}

extern "C" hsgn_status hsgn_kernel_times(const hsgn_ctx* c, double* s12_ms, double* s3_ms, int64_t* steps) {
    if (!c) return HSGN_EINVAL;
    const double n = c->kt_n ? (double)c->kt_n : 1.0;
    if (s12_ms) *s12_ms = c->kt_ms[0] / n;
    if (s3_ms) *s3_ms = c->kt_ms[1] / n;
    if (steps) *steps = c->kt_n;
    return HSGN_OK;
}

// Per-stage device time of the fused step (CUDA events around each stage
// kernel on the context stream, averaged over `reps` steps on workspace
// copies of (y, k1)).  ms3[k] = mean ms of stage k+1.  Used by bench.py for
// the roofline of the dominant kernel.
extern "C" hsgn_status hsgn_profile_stages(hsgn_ctx* c, const hsgn_state* y, const hsgn_state* k1, double dt,
                                           int32_t reps, double* ms3) {
    if (!c || !y || !k1 || !ms3 || reps < 1) return HSGN_EINVAL;
    DeviceGuard dg_(c->device);
    hsgn_status st;
    if ((st = ensure_ws(c, 1))) return st;
    CK(cudaMemcpyAsync(c->ws[0].base - GHOST * c->grid.nx, y->base - GHOST * c->grid.nx, sizeof(double) * 5 * c->fs,
                       cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(c->ws[2].base - GHOST * c->grid.nx, k1->base - GHOST * c->grid.nx, sizeof(double) * 5 * c->fs,
                       cudaMemcpyDeviceToDevice, c->stream));
    cudaEvent_t ev[4];
    for (int k = 0; k < 4; ++k) CK(cudaEventCreate(&ev[k]));
    double acc[3] = {0, 0, 0};
    for (int r = 0; r < reps; ++r) {
        reset_recs(c, 1);
        const hsgn_state *Y = &c->ws[0], *K1 = &c->ws[2];
        hsgn_state *K2 = &c->ws[4], *YN = &c->ws[1], *K4 = &c->ws[3];
        StepRec* rec = &c->d_rec[0];
        StageArgs A = stage_args(c, MODE_S1, 0.5 * dt);
        A.a = 0.5 * dt;
        A.y = Y->base;
        A.k = K1->base;
        A.out = K2->base;
        A.bad = &rec->bad[0];
        CK(cudaEventRecord(ev[0], c->stream));
        if ((st = launch(c, MODE_S1, A))) return st;
        CK(cudaEventRecord(ev[1], c->stream));
        A = stage_args(c, MODE_S2, 0.75 * dt);
        A.a = 0.75 * dt;
        A.c1 = dt * (2.0 / 9.0);
        A.c2 = dt * (1.0 / 3.0);
        A.c3 = dt * (4.0 / 9.0);
        A.y = Y->base;
        A.k = K2->base;
        A.kc = K1->base;
        A.out = YN->base;
        A.bad = &rec->bad[1];
        A.minh = &rec->minh;
        if ((st = launch(c, MODE_S2, A))) return st;
        CK(cudaEventRecord(ev[2], c->stream));
        A = stage_args(c, MODE_S3, dt);
        A.y = YN->base;
        A.out = K4->base;
        A.bad = &rec->bad[2];
        if ((st = launch(c, MODE_S3, A))) return st;
        CK(cudaEventRecord(ev[3], c->stream));
        CK(cudaEventSynchronize(ev[3]));
        for (int k = 0; k < 3; ++k) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
            acc[k] += ms;
        }
    }
    for (int k = 0; k < 4; ++k) cudaEventDestroy(ev[k]);
    for (int k = 0; k < 3; ++k) ms3[k] = acc[k] / reps;
    return HSGN_OK;
}

// Mean device ms of the fused S12 kernel (stages 1 + 2) over `reps` launches
// on workspace copies of (y, k1) (caller state intact).
extern "C" hsgn_status hsgn_profile_fused(hsgn_ctx* c, const hsgn_state* y, const hsgn_state* k1, double dt,
                                          int32_t reps, double* ms) {
    if (!c || !y || !k1 || !ms || reps < 1) return HSGN_EINVAL;
    DeviceGuard dg_(c->device);
    hsgn_status st;
    if ((st = ensure_ws(c, 2))) return st;
    CK(cudaMemcpyAsync(c->ws[0].base - GHOST * c->grid.nx, y->base - GHOST * c->grid.nx, sizeof(double) * 5 * c->fs,
                       cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(c->ws[2].base - GHOST * c->grid.nx, k1->base - GHOST * c->grid.nx, sizeof(double) * 5 * c->fs,
                       cudaMemcpyDeviceToDevice, c->stream));
    reset_recs(c, 2);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    double acc = 0.0;
    for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(e0, c->stream));
        if ((st = enqueue_s12(c, &c->ws[0], &c->ws[2], &c->ws[6], &c->d_rec[1], nullptr, dt))) return st;
        CK(cudaEventRecord(e1, c->stream));
        CK(cudaEventSynchronize(e1));
        float m = 0.f;
        cudaEventElapsedTime(&m, e0, e1);
        acc += m;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms = acc / reps;
    return HSGN_OK;
}

// ------------------------------------------------------------------ in-process slab group
// The slab decomposition of DESIGN.md section 6 driven from ONE process: N
// slab contexts (on one or several devices) whose halo rows move by a pull
// kernel reading the neighbours' boundary rows through (peer) device
// pointers, ordered by CUDA events -- no spinning, so several slabs may share
// one GPU.  Used to test the multi-slab kernel path on a single B200, and as
// a single-process multi-GPU transport (NVLink peer reads).

struct hsgn_group {
    hsgn_grid grid{};
    int n = 0;
    std::vector<hsgn_ctx*> m;
    std::vector<int> j0, j1;
    std::vector<cudaEvent_t> evk, evp;  // per member: stage kernel done / halo pull done
    std::string err;
};

struct hsgn_gstate {
    std::vector<hsgn_state*> p;
};

namespace {

struct HaloPull {
    double* dst[10];
    const double* src[10];
    int nx, count;
};

__global__ void halo_pull_kernel(const HaloPull H) {
    const int k = blockIdx.y;
    if (k >= H.count) return;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < H.nx; i += gridDim.x * blockDim.x) H.dst[k][i] = H.src[k][i];
}

int g_dn(const hsgn_group* G, int r) {
    if (r > 0) return r - 1;
    return G->grid.kind_y == HSGN_BOUNDED ? -1 : G->n - 1;
}
int g_up(const hsgn_group* G, int r) {
    if (r + 1 < G->n) return r + 1;
    return G->grid.kind_y == HSGN_BOUNDED ? -1 : 0;
}

hsgn_status gfail(hsgn_group* G, hsgn_status s, const std::string& what) {
    G->err = what;
    return s;
}

// Fill the ghost rows of every member's part of `parts` (nf fields) from its
// neighbours, after their latest kernels (evk); record evp.
hsgn_status group_pull(hsgn_group* G, const std::vector<hsgn_state*>& parts, int nf) {
    for (int r = 0; r < G->n; ++r) {
        hsgn_ctx* c = G->m[r];
        const int dn = g_dn(G, r), up = g_up(G, r);
        cudaSetDevice(c->device);
        HaloPull H;
        H.nx = GHOST * G->grid.nx;  // GHOST contiguous rows per field and direction
        H.count = 0;
        const long long nx = G->grid.nx;
        for (int f = 0; f < nf; ++f) {
            if (dn >= 0) {
                const hsgn_ctx* d = G->m[dn];
                H.dst[H.count] = parts[r]->f(f) - GHOST * nx;
                H.src[H.count] = parts[dn]->f(f) + (long long)(d->ny_loc - GHOST) * nx;
                ++H.count;
            }
            if (up >= 0) {
                H.dst[H.count] = parts[r]->f(f) + (long long)c->ny_loc * nx;
                H.src[H.count] = parts[up]->f(f);
                ++H.count;
            }
        }
        if (dn >= 0) cudaStreamWaitEvent(c->stream, G->evk[dn], 0);
        if (up >= 0) cudaStreamWaitEvent(c->stream, G->evk[up], 0);
        if (H.count) halo_pull_kernel<<<dim3((H.nx + 255) / 256 < 64 ? (H.nx + 255) / 256 : 64, H.count), 256, 0,
                                        c->stream>>>(H);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return gfail(G, HSGN_ECUDA, cudaGetErrorString(e));
        cudaEventRecord(G->evp[r], c->stream);
    }
    return HSGN_OK;
}

// Before a member overwrites buffers its neighbours may still be reading.
void group_wait_pulls(hsgn_group* G, int r) {
    const int dn = g_dn(G, r), up = g_up(G, r);
    hsgn_ctx* c = G->m[r];
    if (dn >= 0) cudaStreamWaitEvent(c->stream, G->evp[dn], 0);
    if (up >= 0) cudaStreamWaitEvent(c->stream, G->evp[up], 0);
}

}  // namespace

extern "C" {

hsgn_status hsgn_group_create(const hsgn_grid* grid, const hsgn_phys* phys, const double* b_full, const int* devices,
                              int32_t n, hsgn_group** out) {
    DeviceRestore dr_;
    if (!grid || !phys || !b_full || !out || n < 1 || grid->ny < 2 * n) return HSGN_EINVAL;
    hsgn_group* G = new hsgn_group();
    G->grid = *grid;
    G->n = n;
    const int base = grid->ny / n, rem = grid->ny % n;  // slab.py partition(): first ranks take the remainder
    int j = 0;
    for (int r = 0; r < n; ++r) {
        const int k = base + (r < rem ? 1 : 0);
        G->j0.push_back(j);
        G->j1.push_back(j + k);
        j += k;
    }
    for (int r = 0; r < n; ++r) {
        hsgn_ctx* c = nullptr;
        const int dev = devices ? devices[r] : -1;
        hsgn_status s = hsgn_ctx_create_slab(grid, phys, b_full + (long long)G->j0[r] * grid->nx, dev, G->j0[r],
                                             G->j1[r], r, n, &c);
        if (s) {
            hsgn_group_destroy(G);
            return s;
        }
        c->in_group = 1;
        G->m.push_back(c);
        cudaEvent_t a, b;
        cudaSetDevice(c->device);
        cudaEventCreateWithFlags(&a, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&b, cudaEventDisableTiming);
        G->evk.push_back(a);
        G->evp.push_back(b);
    }
    for (int r = 0; r < n; ++r)  // peer access between neighbouring devices (no-op on one device)
        for (int q : {g_dn(G, r), g_up(G, r)})
            if (q >= 0 && G->m[q]->device != G->m[r]->device) {
                cudaSetDevice(G->m[r]->device);
                cudaDeviceEnablePeerAccess(G->m[q]->device, 0);
                cudaGetLastError();
            }
    // bathymetry ghost rows (static field, one pull)
    std::vector<hsgn_state*> bs(n);
    std::vector<hsgn_state> bstore(n);
    for (int r = 0; r < n; ++r) {
        bstore[r].base = G->m[r]->b;
        bstore[r].fs = G->m[r]->fs;
        bs[r] = &bstore[r];
        cudaSetDevice(G->m[r]->device);
        cudaStreamSynchronize(G->m[r]->stream);
        cudaEventRecord(G->evk[r], G->m[r]->stream);
    }
    hsgn_status s = group_pull(G, bs, 1);
    for (int r = 0; r < n; ++r) cudaStreamSynchronize(G->m[r]->stream);
    int b_lit = 0;  // the guard's b flag covers every slab
    for (int r = 0; r < n; ++r) b_lit |= G->m[r]->b_lit;
    for (int r = 0; r < n && b_lit; ++r)
        if (!G->m[r]->b_lit) {
            G->m[r]->b_lit = 1;
            setup_ctx(G->m[r]);
        }
    if (s) {
        hsgn_group_destroy(G);
        return s;
    }
    *out = G;
    return HSGN_OK;
}

hsgn_status hsgn_group_destroy(hsgn_group* G) {
    DeviceRestore dr_;
    if (!G) return HSGN_OK;
    for (int r = 0; r < (int)G->m.size(); ++r) {
        cudaSetDevice(G->m[r]->device);
        if (r < (int)G->evk.size()) cudaEventDestroy(G->evk[r]);
        if (r < (int)G->evp.size()) cudaEventDestroy(G->evp[r]);
        hsgn_ctx_destroy(G->m[r]);
    }
    delete G;
    return HSGN_OK;
}

const char* hsgn_group_last_error(const hsgn_group* G) { return G ? G->err.c_str() : "null group"; }

hsgn_status hsgn_group_state_alloc(hsgn_group* G, hsgn_gstate** out) {
    DeviceRestore dr_;
    if (!G || !out) return HSGN_EINVAL;
    hsgn_gstate* s = new hsgn_gstate();
    for (hsgn_ctx* c : G->m) {
        hsgn_state* p = nullptr;
        hsgn_status st = hsgn_state_alloc(c, &p);
        if (st) {
            hsgn_group_state_free(G, s);
            return st;
        }
        s->p.push_back(p);
    }
    *out = s;
    return HSGN_OK;
}

hsgn_status hsgn_group_state_free(hsgn_group* G, hsgn_gstate* s) {
    DeviceRestore dr_;
    if (!G || !s) return HSGN_EINVAL;
    for (size_t r = 0; r < s->p.size(); ++r) hsgn_state_free(G->m[r], s->p[r]);
    delete s;
    return HSGN_OK;
}

// host layout: the full grid (5 fields of nx*ny); each member takes its rows
hsgn_status hsgn_group_state_upload(hsgn_group* G, hsgn_gstate* s, const double* host) {
    DeviceRestore dr_;
    if (!G || !s || !host) return HSGN_EINVAL;
    const long long nx = G->grid.nx, n = nx * G->grid.ny;
    for (int r = 0; r < G->n; ++r) {
        hsgn_ctx* c = G->m[r];
        cudaSetDevice(c->device);
        for (int f = 0; f < 5; ++f)
            if (cudaMemcpyAsync(s->p[r]->f(f), host + f * n + G->j0[r] * nx, sizeof(double) * nx * c->ny_loc,
                                cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
                return gfail(G, HSGN_ECUDA, "upload");
        group_wait_pulls(G, r);
        cudaEventRecord(G->evk[r], c->stream);
    }
    hsgn_status st = group_pull(G, s->p, 5);
    for (hsgn_ctx* c : G->m) cudaStreamSynchronize(c->stream);
    return st;
}

hsgn_status hsgn_group_state_download(hsgn_group* G, const hsgn_gstate* s, double* host) {
    DeviceRestore dr_;
    if (!G || !s || !host) return HSGN_EINVAL;
    const long long nx = G->grid.nx, n = nx * G->grid.ny;
    for (int r = 0; r < G->n; ++r) {
        hsgn_ctx* c = G->m[r];
        cudaSetDevice(c->device);
        for (int f = 0; f < 5; ++f) {
            const cudaError_t e = cudaMemcpyAsync(host + f * n + G->j0[r] * nx, s->p[r]->f(f),
                                                  sizeof(double) * nx * c->ny_loc, cudaMemcpyDeviceToHost, c->stream);
            if (e != cudaSuccess) return gfail(G, HSGN_ECUDA, std::string("download: ") + cudaGetErrorString(e));
        }
    }
    for (hsgn_ctx* c : G->m) cudaStreamSynchronize(c->stream);
    return HSGN_OK;
}

// rhs on the decomposed grid (ghost rows of q must be current: upload does it)
hsgn_status hsgn_group_rhs(hsgn_group* G, double t, const hsgn_gstate* q, hsgn_gstate* out, int64_t* bad_nodes) {
    DeviceRestore dr_;
    if (!G || !q || !out) return HSGN_EINVAL;
    int64_t bad = 0;
    for (int r = 0; r < G->n; ++r) {
        hsgn_ctx* c = G->m[r];
        cudaSetDevice(c->device);
        hsgn_status s = ensure_recs(c, 1);
        if (s) return s;
        cudaMemsetAsync(&c->d_rec[0].bad[0], 0, sizeof(unsigned long long), c->stream);
        group_wait_pulls(G, r);
        if ((s = rhs_raw(c, t, q->p[r], out->p[r], false, &c->d_rec[0].bad[0]))) return s;
        cudaEventRecord(G->evk[r], c->stream);
    }
    hsgn_status s = group_pull(G, out->p, 5);
    if (s) return s;
    for (int r = 0; r < G->n; ++r) {
        hsgn_ctx* c = G->m[r];
        unsigned long long hb = 0;
        cudaMemcpyAsync(&hb, &c->d_rec[0].bad[0], sizeof hb, cudaMemcpyDeviceToHost, c->stream);
        cudaStreamSynchronize(c->stream);
        bad += (int64_t)hb;
    }
    if (bad_nodes) *bad_nodes = bad;
    return bad ? gfail(G, HSGN_EDEPTH, "non-positive depth") : HSGN_OK;
}

// `steps` fused fixed-step BS3 steps on (y, k1) in place, halo pulls after
// every stage (the NCCL schedule of enqueue_step with an in-process transport)
hsgn_status hsgn_group_bs3_fixed_steps(hsgn_group* G, hsgn_gstate* y, hsgn_gstate* k1, double t, double dt,
                                       int64_t steps, int64_t* steps_done) {
    DeviceRestore dr_;
    if (!G || !y || !k1 || steps < 0) return HSGN_EINVAL;
    const int n = G->n;
    for (hsgn_ctx* c : G->m) {
        cudaSetDevice(c->device);
        hsgn_status s = ensure_ws(c, 1);
        if (s) return s;
    }
    // work in each member's workspace: y -> ws[0], k1 -> ws[2]
    std::vector<hsgn_state*> Y[2], K[2], K2(n);
    for (int r = 0; r < n; ++r) {
        hsgn_ctx* c = G->m[r];
        Y[0].push_back(&c->ws[0]);
        Y[1].push_back(&c->ws[1]);
        K[0].push_back(&c->ws[2]);
        K[1].push_back(&c->ws[3]);
        K2[r] = &c->ws[4];
        cudaSetDevice(c->device);
        group_wait_pulls(G, r);
        cudaMemcpyAsync(c->ws[0].base - GHOST * c->grid.nx, y->p[r]->base - GHOST * c->grid.nx, sizeof(double) * 5 * c->fs,
                        cudaMemcpyDeviceToDevice, c->stream);
        cudaMemcpyAsync(c->ws[2].base - GHOST * c->grid.nx, k1->p[r]->base - GHOST * c->grid.nx, sizeof(double) * 5 * c->fs,
                        cudaMemcpyDeviceToDevice, c->stream);
        cudaEventRecord(G->evk[r], c->stream);
        cudaEventRecord(G->evp[r], c->stream);
    }
    int p = 0;
    int64_t done = 0;
    hsgn_status result = HSGN_OK;
    // the members' fixed-step structure: S12 + S3 (kernels 1, 2) or one
    // kernel per stage (kernels 1..3); halos pulled after every kernel
    const bool s12 = G->m[0]->fused == 3 && G->m[0]->source == 0;
    for (int64_t step = 0; step < steps; ++step) {
        for (int kern = 1; kern <= (s12 ? 2 : 3); ++kern) {
            for (int r = 0; r < n; ++r) {
                hsgn_ctx* c = G->m[r];
                cudaSetDevice(c->device);
                if (kern == 1) reset_recs(c, 1);
                group_wait_pulls(G, r);
                hsgn_status s;
                if (s12)
                    s = kern == 1 ? enqueue_s12(c, Y[p][r], K[p][r], Y[p ^ 1][r], &c->d_rec[0], nullptr, dt)
                                  : enqueue_s3_fixed(c, Y[p ^ 1][r], K[p ^ 1][r], &c->d_rec[0], dt);
                else
                    s = enqueue_stage(c, kern, Y[p][r], K[p][r], K2[r], Y[p ^ 1][r], K[p ^ 1][r], nullptr,
                                      &c->d_rec[0], nullptr, t, dt, false, 0, 0);
                if (s) return s;
                cudaEventRecord(G->evk[r], c->stream);
            }
            const std::vector<hsgn_state*>& produced =
                s12 ? (kern == 1 ? Y[p ^ 1] : K[p ^ 1]) : (kern == 1 ? K2 : (kern == 2 ? Y[p ^ 1] : K[p ^ 1]));
            hsgn_status s = group_pull(G, produced, 5);
            if (s) return s;
        }
        bool bad = false;
        for (int r = 0; r < n; ++r) {
            hsgn_ctx* c = G->m[r];
            StepRec rec;
            cudaSetDevice(c->device);
            cudaMemcpyAsync(&rec, &c->d_rec[0], sizeof rec, cudaMemcpyDeviceToHost, c->stream);
            cudaStreamSynchronize(c->stream);
            bad |= (rec.bad[0] | rec.bad[1] | rec.bad[2]) != 0;
            c->n_evals += 3;
        }
        if (bad) {
            result = gfail(G, HSGN_EDEPTH, "non-positive depth in fixed-step mode");
            break;
        }
        t = t + dt;
        p ^= 1;
        ++done;
    }
    for (int r = 0; r < n; ++r) {
        hsgn_ctx* c = G->m[r];
        cudaSetDevice(c->device);
        cudaMemcpyAsync(y->p[r]->base - GHOST * c->grid.nx, Y[p][r]->base - GHOST * c->grid.nx, sizeof(double) * 5 * c->fs,
                        cudaMemcpyDeviceToDevice, c->stream);
        cudaMemcpyAsync(k1->p[r]->base - GHOST * c->grid.nx, K[p][r]->base - GHOST * c->grid.nx, sizeof(double) * 5 * c->fs,
                        cudaMemcpyDeviceToDevice, c->stream);
        cudaStreamSynchronize(c->stream);
    }
    if (steps_done) *steps_done = done;
    return result;
}

// Decomposition-independent SBP-norm totals: per-slab row sums gathered in
// global row order, one outer sum (kind: 0 mass, 1 energy, 2 energy rate).
hsgn_status hsgn_group_reduce(hsgn_group* G, int32_t kind, const hsgn_gstate* q, const hsgn_gstate* qt,
                              double* out) {
    DeviceRestore dr_;
    if (!G || !q || !out || kind < 0 || kind > 2 || (kind == 2 && !qt)) return HSGN_EINVAL;
    std::vector<double> rows(G->grid.ny);
    for (int r = 0; r < G->n; ++r) {
        hsgn_status s = hsgn_row_sums(G->m[r], kind, q->p[r], qt ? qt->p[r] : nullptr, 0, rows.data() + G->j0[r]);
        if (s) return s;
    }
    *out = outer_sum(&G->grid, rows.data(), 0, G->grid.ny);
    return HSGN_OK;
}

}  // extern "C"
