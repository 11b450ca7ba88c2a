/*
 * oracle_abi.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C ABI shared by the two CPU checkers under oracle/:
 *   ref_*  : oracle/_ref/libhsgn_ref.so, the UNMODIFIED reference headers
 *            (/root/reference/proj/include/hsgn) compiled by oracle/Makefile
 *            through the thin adapter oracle/ref_capi.cpp;
 *   orc_*  : oracle/liboracle.so, the from-scratch C restatement in
 *            oracle/hsgn_oracle.c (pinned against ref_* and tests/golden/).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load these libraries.  The product path
 * (paper_2601_02540_b200) never links or calls them.
 *
 * Field layout everywhere: a state is 5 contiguous fp64 fields
 * (h, u, v, w, eta), each nx*ny, row-major with x fastest
 * (reference field.hpp:9-10, model.hpp:22-35).
 */
#ifndef HSGN_ORACLE_ABI_H
#define HSGN_ORACLE_ABI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* kind: 0 = periodic, 1 = bounded (reference grid.hpp:11) */
typedef struct {
    int32_t nx, ny;
    int32_t kind_x, kind_y;
    double x_min, x_max, y_min, y_max;
} orc_grid;

/* reference model.hpp:40-45 (b passed separately) */
typedef struct {
    double g, lambda, h_floor;
} orc_phys;

/* reference time_integration.hpp:18-29 */
typedef struct {
    double abs_tol, rel_tol, dt_initial, dt_max, safety, growth_cap, shrink_floor;
    int64_t max_steps;
    double fixed_dt, h_floor;
} orc_cfg;

/* reference time_integration.hpp:33-42 */
typedef struct {
    double t;
    int64_t accepted, rejected, rhs_evals, rhs_evals_setup;
    int32_t aborted;
    char reason[256];
} orc_record;

/* source_kind: 0 none, 1 manufactured (reference rhs.hpp:252-266 with
 * manufactured_generated.hpp:69-115). */

#ifdef __cplusplus
}
#endif
#endif
