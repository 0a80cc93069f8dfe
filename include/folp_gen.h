/*
 * folp_gen.h -- seeded generators for the five BASELINE.json configurations
 * (SURVEY.md section 8d).  Harness-side: both the B200 engine and the CPU
 * reference receive the same generated LP.  Randomness uses raw
 * std::mt19937_64 draws only (U[0,1) = (r >> 11) * 2^-53, Box-Muller
 * normals written out), like the reference's instance_gen.cpp:25-40, so the
 * instances are identical on every platform.
 *
 * `scale` (0 < scale <= 1) shrinks the row/column counts of a family while
 * keeping its structure (tests use small members of each family).
 */
#ifndef FOLP_GEN_H_
#define FOLP_GEN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct folp_gen_lp {
  int64_t num_rows, num_cols, num_inequality_rows, nnz;
  int64_t* row_start;  /* CSR, columns increasing */
  int64_t* row_cols;
  double* row_values;
  int64_t* col_start;  /* CSC, rows increasing */
  int64_t* col_rows;
  double* col_values;
  double* objective;
  double* right_hand_side;
  double* variable_lower;
  double* variable_upper;
  double objective_constant;
  int64_t max_row_len, max_col_len; /* structure statistics */
} folp_gen_lp;

/* cfg = 1..5 as in BASELINE.json "configs" (index + 1). NULL on error. */
folp_gen_lp* folp_gen_config(int32_t cfg, uint64_t seed, double scale);
void folp_gen_free(folp_gen_lp* lp);
const char* folp_gen_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* FOLP_GEN_H_ */
