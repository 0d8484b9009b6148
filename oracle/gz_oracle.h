/* gz_oracle.h -- TEST INFRASTRUCTURE ONLY: CPU restatement of the reference codec
 * (/root/reference/pkg/src/gzccl/codec.py).  See gz_oracle.c. */
#ifndef GZ_ORACLE_H
#define GZ_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
enum { GZO_OK = 0, GZO_EBAD = -1, GZO_ENONFINITE = -2, GZO_ECAP = -3, GZO_EDECODE = -4 };
uint64_t gzo_compress_bound(uint64_t n);
int gzo_check_eb(double eb);
int64_t gzo_first_nonfinite(const float *x, uint64_t n);
int gzo_compress(const float *x, uint64_t n, double eb, uint8_t *out, uint64_t cap, uint64_t *out_len,
                 uint64_t *block_offsets, int64_t *bad_index, int threads);
int gzo_parse_header(const uint8_t *blob, uint64_t len, uint64_t *n, double *eb, char *msg, int msglen);
int gzo_walk(const uint8_t *payload, uint64_t psize, uint64_t n, uint64_t *starts, char *msg, int msglen);
int gzo_decompress(const uint8_t *blob, uint64_t len, float *y, uint64_t ycap, uint64_t *n_out, char *msg, int msglen,
                   int threads);
#ifdef __cplusplus
}
#endif
#endif
