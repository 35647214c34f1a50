/* TEST INFRASTRUCTURE ONLY — CPU oracle (restatement of the reference
 * dctfilter library). See dctf_oracle.c for the parity pin and citations. */
#ifndef DCTF_ORACLE_H
#define DCTF_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int or_dct_basis(int n, double* c);
void or_forward_2d(int n, const double* c, const double* x, double* out);
void or_inverse_2d(int n, const double* c, const double* y, double* out);
int or_row_symmetric(const double* w, int k);
int or_plan_pairs(const double* w, int k, int n, int padding, int* npairs, int* merged,
                  double* lefts, double* rights);
void or_apply_pairs(int n, int npairs, const double* lefts, const double* rights,
                    const double* x, double* out);
void or_convolve(int n, const double* w, int kr, int kc, int padding, const double* x,
                 double* out);
int or_quantize(double v);
size_t or_tile(const uint8_t* img, int w, int h, int n, double* blocks);
int or_assemble(const double* blocks, int w, int h, int n, uint8_t* out);
int or_filter_image(const uint8_t* img, int w, int h, const double* mw, int k, int padding,
                    int n, uint8_t* out, double* coef_in, double* coef_out, double* prequant);
int or_filter_image_spatial(const uint8_t* img, int w, int h, const double* mw, int kr, int kc,
                            int padding, int n, uint8_t* out, double* prequant);
int or_dense_operator(const double* mw, int kr, int kc, int n, int padding, double* hout);

#ifdef __cplusplus
}
#endif
#endif
