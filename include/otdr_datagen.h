/* otdr_datagen.h -- seeded synthetic instances (host C++, in libotdr_dev.so).
 *
 * Restates the reference's generators so benchmarks and callers can build the
 * exact instances the reference tests and CLI use:
 *   otdr_gaussian_points    gaussian_problem's two clouds   datagen.cpp:21-35, :56-65
 *   otdr_adaptation_points  adaptation_problem's clouds     datagen.cpp:67-129
 * with the mt19937_64 / 53-bit uniform / Box-Muller stream of rng.hpp:14-45.
 * The cost itself is built on device by otdr_dev_build_sqdist_cost
 * (datagen.cpp:43-54 + problem.cpp:68-74); marginals are uniform (1/m, 1/n).
 */
#ifndef OTDR_DATAGEN_H
#define OTDR_DATAGEN_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* src: m x 2, tgt: n x 2, row-major fp64. */
void otdr_gaussian_points(int64_t m, int64_t n, uint64_t seed, double* src, double* tgt);

/* Returns 0, or 5 (OTDR_E_INVALID_ARG) for classes < 1 or fewer points than
 * classes. Labels are the class of each point (rows sorted by class). */
int otdr_adaptation_points(int64_t m, int64_t n, int classes, uint64_t seed, int identity_map,
                           double* src, double* tgt, int32_t* src_labels, int32_t* tgt_labels);

/* ncclGetUniqueId for row-sharded contexts (128 bytes). Returns 0 on success. */
int otdr_dev_nccl_unique_id(unsigned char* out128);

#ifdef __cplusplus
}
#endif
#endif
