/*
 * s5g_gen.h -- C5 corpus generator (libs5gen.so).  Bench and test
 * infrastructure only: it produces the synthetic input BASELINE.json
 * configs[4] describes; it is not part of the sort or of the drop-in
 * boundary (include/s5g.h).  Strings n0 .. n0+n-1 of the counter-based
 * definition in paper_1403_2056_b200/csrc/s5g_gen.cu; handles are offsets
 * relative to the first generated string.
 */
#ifndef S5G_GEN_H
#define S5G_GEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
/* Arena bytes (terminators included) of strings n0 .. n0+n-1. */
int64_t s5gen_nodup_bytes(int64_t n0, int64_t n, uint64_t seed);
/* Host (OpenMP): handles[n] and/or buf[s5gen_nodup_bytes] (either may be NULL). */
int s5gen_nodup_host(int64_t n0, int64_t n, uint64_t seed, uint8_t *buf, int64_t *handles);
/* Device: the same bytes into device buf / handles (synchronous on stream). */
int s5gen_nodup_device(int64_t n0, int64_t n, uint64_t seed, uint8_t *buf, int64_t *handles,
                       void *stream);
const char *s5gen_last_error(void);
#ifdef __cplusplus
}
#endif
#endif
