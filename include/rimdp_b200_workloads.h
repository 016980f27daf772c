/* rimdp_b200_workloads.h — host-side workload generators of the B200 engine.
 *
 * rimdp_random_imdp restates the reference generator random_imdp /
 * random_point_imdp (random_model.hpp:42-161) bit for bit (same
 * std::mt19937_64 stream, same rejection loop, same [0,0] dropping), so the
 * engine and the CPU reference ingest byte-identical models for BASELINE
 * configs 2-3.  Two-phase: generate (sizes out, opaque handle), then take
 * (copies into caller buffers and frees the handle).
 */
#ifndef RIMDP_B200_WORKLOADS_H
#define RIMDP_B200_WORKLOADS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rimdp_random_sizes {
    int32_t num_states;
    int32_t num_cols;
    int64_t nnz;
} rimdp_random_sizes;

/* dtype: 0 = f64, 1 = f32 (values drawn in double, converted like
 * NumericTraits<float>::from_double).  Returns 0 on success. */
int rimdp_random_imdp(int32_t num_states, int32_t actions, double density, double scale, uint64_t seed,
                      int32_t point, int32_t dtype, rimdp_random_sizes* sizes, void** handle);
int rimdp_random_imdp_take(void* handle, int32_t* stateptr, int64_t* colptr, int32_t* rowval, void* lower,
                           void* upper);

#ifdef __cplusplus
}
#endif
#endif
