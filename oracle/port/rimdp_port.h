/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference hot path.
 *
 * Used by tests/ as an independent checker and by bench.py as the "port"
 * CPU baseline when the reference library (oracle/_ref) is unavailable.
 * Never linked into the product.  Same extern "C" surface as
 * oracle/ref_capi.cpp with the prefix port_ (colptr is int64 here). */
#ifndef RIMDP_PORT_H
#define RIMDP_PORT_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct port_spec {
    int kind; /* 0 FTR, 1 ITR, 2 FTRA, 3 ITRA, 4 FTRew, 5 ITRew (property.hpp:14-59) */
    const int* reach;
    int nreach;
    const int* avoid;
    int navoid;
    const void* rewards;
    double discount;
    long long horizon;
    double eps;
    int pessimistic;
    int maximize;
    unsigned workers;
    long long max_iterations;
} port_spec;

typedef struct port_err {
    char msg[512];
    long long iterations;
    double residual;
    int violation_kind;
    long long violation_column;
} port_err;

enum { PORT_OK = 0, PORT_MODEL_ERROR = 1, PORT_NON_CONVERGENCE = 2, PORT_STATE_OUT_OF_RANGE = 3,
       PORT_INVALID_PROPERTY = 4, PORT_INVALID_POLICY = 5, PORT_OTHER = 9 };

#ifdef __cplusplus
}
#endif
#endif
