/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference hot path
 * (proj/include/rimdp/omax.hpp, bellman.hpp, solver.hpp, property.hpp).
 *
 * Compiled by oracle/Makefile with -ffp-contract=off: every multiply and add
 * rounds separately, exactly like the reference built for x86-64 without
 * -march (no FMA instructions available).  Pinned by tests/test_oracle.py
 * against the reference library (oracle/_ref) and tests/golden fixtures. */
#define _GNU_SOURCE
#include "rimdp_port.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* Shortest round-trip decimal, the spirit of std::to_chars used by
 * NumericTraits::to_string (numeric.hpp:30-35). */
static void shortest(char* buf, size_t len, double x, int is_float) {
    for (int prec = 1; prec <= 17; ++prec) {
        snprintf(buf, len, "%.*g", prec, x);
        if (is_float ? ((float)strtod(buf, NULL) == (float)x) : (strtod(buf, NULL) == x)) return;
    }
}

#define T double
#define SFX f64
#define TOL 1e-9
#define FABS fabs
#include "rimdp_port_t.inc"
#undef T
#undef SFX
#undef TOL
#undef FABS

#define T float
#define SFX f32
#define TOL 1e-5f
#define FABS fabsf
#include "rimdp_port_t.inc"
#undef T
#undef SFX
#undef TOL
#undef FABS

/* Model handles carry no type tag; the Python side calls the matching
 * free function through port_model_free with the dtype it built. */
void port_model_free(void* h) {
    /* The two model layouts differ only in the element type of lower/upper,
     * and both free the same five buffers, so one implementation suffices. */
    port_model_free_impl_f64(h);
}
