/* otpr_oracle.h — TEST INFRASTRUCTURE ONLY (see otpr_oracle.c header).
 * CPU restatement of the reference assignment path; the parity checker. */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror the reference exception taxonomy
 * (include/otpr/errors.hpp:9-37 -> tools/otbench.cpp:187-209 exit codes) */
enum { ORC_OK = 0, ORC_PARAMETER = 2, ORC_INPUT = 3, ORC_NUMERICAL = 4, ORC_INVARIANT = 5 };

typedef struct {
  int64_t phases;
  int64_t sum_ni;
  int32_t swapped;
  int32_t full_match_termination;
  double cost;
} orc_stats;

uint64_t orc_splitmix64(uint64_t x);
void orc_raw_stream(uint64_t seed, int64_t count, uint64_t* out);
int orc_uniform_square_points(int32_t n, uint64_t seed, double* ax, double* ay,
                              double* bx, double* by);
double orc_points_cost(double ax, double ay, double bx, double by);
int orc_gen_uniform_square(int32_t n, uint64_t seed, double* cost);
int orc_mnist_sample(uint32_t count, int32_t n, uint64_t seed, uint32_t* picked);
int orc_mnist_cost(int32_t n, const uint8_t* images, double* cost);
int orc_gen_random_ot_rational(int32_t n_a, int32_t n_b, uint64_t seed,
                               int64_t* wa, int64_t* wb, double* cost);
int64_t orc_scaled_floor(double c, double eps);
int orc_validate_costs(int32_t n_a, int32_t n_b, const double* cost);
int orc_units(double eps, int32_t* unit_floor, int32_t* unit_ceil);
int orc_scale_round_costs(int32_t n_a, int32_t n_b, const double* cost, double eps,
                          int32_t* k, int32_t* unit_floor, int32_t* unit_ceil);
double orc_matching_cost(int32_t n_a, int32_t n_b, const double* cost,
                         const int32_t* match_of_a);
int orc_solve_assignment(int32_t n_a, int32_t n_b, const double* cost, double eps,
                         int32_t* match_of_a, int32_t* match_of_b, int64_t* y_a,
                         int64_t* y_b, int64_t* free_counts, int64_t free_cap,
                         orc_stats* st);
int orc_solve_rounded(int32_t n_a, int32_t n_b, const int32_t* kT, double eps,
                      int32_t* match_of_a, int32_t* match_of_b, int64_t* y_a,
                      int64_t* y_b, int64_t* free_counts, int64_t free_cap,
                      orc_stats* st);
uint64_t orc_fnv1a64(const void* data, int64_t nbytes, uint64_t h);

#ifdef __cplusplus
}
#endif
