/* kohler_oracle.h — CPU restatement of the reference path (TEST INFRASTRUCTURE
 * ONLY; see kohler_oracle.c).  Not part of the product. */
#ifndef KOHLER_ORACLE_H
#define KOHLER_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORACLE_LEVELS 256
#define ORACLE_NO_BOUNDARY 1
#define ORACLE_INVALID_K 2

void oracle_pair_contribution(int lo, int hi, uint64_t *sum, uint64_t *card);
void oracle_curve_rows(const uint8_t *px, int w, int h, size_t pitch, int r0, int r1,
                       uint64_t *sum, uint64_t *card);
void oracle_fast_curve(const uint8_t *px, int w, int h, uint64_t *sum, uint64_t *card);
void oracle_fast_curve_blocks(const uint8_t *px, int w, int h, unsigned blocks,
                              uint64_t *sum, uint64_t *card);
void oracle_direct_curve(const uint8_t *px, int w, int h, uint64_t *sum, uint64_t *card);
void oracle_mean_contrast(const uint64_t *sum, const uint64_t *card, int n, double *values,
                          uint8_t *defined);
int oracle_optimal_threshold(const double *values, const uint8_t *defined, int n);
int oracle_top_k_local_maxima(const double *values, const uint8_t *defined, int n, int k,
                              int *out, int *out_count);
void oracle_identities(const uint8_t *px, int w, int h, uint64_t *tv, uint64_t *qs);
uint8_t oracle_luma601(unsigned r, unsigned g, unsigned b);
void oracle_rgb_to_gray(const uint8_t *rgb, int w, int h, size_t pitch, uint8_t *out);
int oracle_analyze(const uint8_t *px, int w, int h, int k, uint64_t *sum, uint64_t *card,
                   double *values, uint8_t *defined, int *t0, int *topk, int *topk_count);

#ifdef __cplusplus
}
#endif
#endif
