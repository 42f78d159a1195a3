/*
 * placement_c.h -- C entry points of the host placement policy
 * (include/moesim/balance.hpp; the reference's proj/include/moesim/
 * balance.hpp:12-58, src/balance.cpp:59-165), exported by libmoesim_b200 for
 * C and Python hosts (paper_2303_06182_b200/ep.py).  Host only.
 *
 * Histories are E x B row-major double arrays (share[e*B + b] = fraction of
 * batch b's slots routed to expert e, LoadMatrix::share).  device_of is
 * int32 [E].  Return 0 on success, 1 for an invalid argument
 * (std::invalid_argument in the C++ API), 2 for any other failure; the message
 * is in moesim_placement_last_error().
 */
#ifndef MOESIM_PLACEMENT_C_H_
#define MOESIM_PLACEMENT_C_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* moesim_placement_last_error(void);
int moesim_contiguous_place(int E, int D, int32_t* device_of);
int moesim_greedy_place(const double* share, int E, int B, int D, int32_t* device_of);
int moesim_anticorr_place(const double* share, int E, int B, int D, double weight,
                          int32_t* device_of);
/* corr: E x E row-major */
int moesim_pearson_corr(const double* share, int E, int B, double* corr);
/* device_load (optional): D x B row-major */
int moesim_eval_balance(const int32_t* device_of, int E, int D, const double* share, int B,
                        double* device_load, double* max_load, double* avg_max_load,
                        double* objective);

#ifdef __cplusplus
}
#endif

#endif /* MOESIM_PLACEMENT_C_H_ */
