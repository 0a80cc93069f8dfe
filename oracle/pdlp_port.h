/*
 * pdlp_port.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's PDLP solve path
 * (/root/reference/proj/src/{solver,scaling,termination,lp_model,
 * sparse_matrix}.cpp), used as the CPU checker of the B200 engine and as
 * the "port" CPU baseline.  It exports the include/folp_c.h entry points
 * with the prefix folp_port_.  Presolve is not restated (it stays on the
 * host and is not part of the path): folp_port_solve requires an LP on
 * which presolve is the identity (no fixed, empty or crossed columns, no
 * empty rows) and fails with FOLP_E_INVALID_ARGUMENT otherwise.
 *
 * Every floating-point operation follows the reference's order, so on
 * x86-64 (-O2, no FMA) the results equal the compiled reference bit for
 * bit (pinned in tests/test_oracle_port.py).
 */
#ifndef PDLP_PORT_H_
#define PDLP_PORT_H_

#include "../include/folp_c.h"

#ifdef __cplusplus
extern "C" {
#endif

void folp_port_params_default(folp_params_c* params);
int folp_port_solve(const folp_lp_c* lp, const folp_params_c* params,
                    const double* x0, const double* y0, folp_result_c* out);
int folp_port_multiply(const folp_lp_c* lp, const double* x, double* out);
int folp_port_multiply_transpose(const folp_lp_c* lp, const double* y,
                                 double* out);
int folp_port_rescale(const folp_lp_c* lp, int64_t ruiz_iterations,
                      int32_t apply_pock_chambolle, double alpha,
                      double* row_scale, double* col_scale,
                      double* scaled_values, double* scaled_objective,
                      double* scaled_rhs, double* scaled_lower,
                      double* scaled_upper);
int folp_port_convergence_info(const folp_lp_c* lp, const double* x,
                               const double* y, folp_info_c* info);
int folp_port_normalized_duality_gap(const folp_lp_c* lp, const double* x,
                                     const double* y, double radius,
                                     double omega, double* gap);
int folp_port_adaptive_step(const folp_lp_c* lp, const double* x,
                            const double* y, double omega, double eta_hat,
                            int64_t k, double* x_next, double* y_next,
                            double* eta_used, double* eta_hat_next,
                            int64_t* trials, double* movement_sq,
                            double* cross_term);
int folp_port_malitsky_pock_step(const folp_lp_c* lp, const double* x,
                                 const double* y, double omega, double eta_prev,
                                 double theta_prev, const folp_params_c* params,
                                 double* x_next, double* y_next, double* eta_next,
                                 double* theta_next, int64_t* trials);
const char* folp_port_last_error(void);
/* Summation order of the scalar reductions: 0 = the reference's sequential
 * fold (default, bit-exact); 1 pairwise tree, 2 reversed, 3 tree + 256-entry
 * parts for long segment dots.  Non-zero orders only measure the reference's
 * reduction-order noise floor (tools/noise_floor.py).  Process-global. */
void folp_port_set_sum_order(int order);

#ifdef __cplusplus
}
#endif

#endif /* PDLP_PORT_H_ */
