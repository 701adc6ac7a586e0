/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the dnnp hot path.
 *
 * A plain-C restatement of the reference CPU algorithms in
 * /root/reference/pkg/src/dnnp (conv.py implicit engine, gemm.py tiled
 * engine, intdiv.py magic division, nnops.py, tensor.py).  It is used by
 * tests/ as the checker, by __graft_entry__.smoke() as the checker, and by
 * bench.py's cpu_baseline / --impl reference legs as the timed CPU
 * implementation of the reference algorithm.  The product library never
 * links, loads or calls it.
 *
 * Parity pin: tests/test_oracle_golden.py checks every routine against the
 * golden vectors generated from the reference package itself
 * (tests/golden/gen_golden.py) and against the reference's own
 * known-answer tests (intdiv constants, Fig.1 example, pooling KATs).
 *
 * Tensor geometry arrays: 8 int64 {n, c, h, w, sn, sc, sh, sw}.
 * Filter geometry: 4 int64 {k, c, r, s} (dense KCRS).
 * Conv geometry: 6 int64 {u, v, pad_h, pad_w, mode(0=conv,1=xcorr), accumulate}.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MIN(a, b) ((a) < (b) ? (a) : (b))
#define MAX(a, b) ((a) > (b) ? (a) : (b))
#define CAT_(a, b) a##b
#define CAT(a, b) CAT_(a, b)

typedef struct { int64_t n, c, h, w, sn, sc, sh, sw; } ov4;
static ov4 ov4_of(const int64_t *g)
{
    ov4 v = {g[0], g[1], g[2], g[3], g[4], g[5], g[6], g[7]};
    return v;
}
#define OFF(v, n_, c_, h_, w_) ((n_) * (v).sn + (c_) * (v).sc + (h_) * (v).sh + (w_) * (v).sw)
#define FOR4(v)                                  \
    for (int64_t n = 0; n < (v).n; n++)          \
        for (int64_t c = 0; c < (v).c; c++)      \
            for (int64_t h = 0; h < (v).h; h++)  \
                for (int64_t w = 0; w < (v).w; w++)

/* ---- magic division (intdiv.py:33-101) ----------------------------------- */
typedef struct { uint32_t d, mul, shift, add; } omagic;

omagic oracle_make_divider(uint32_t d)
{
    omagic m = {d, 1, 0, 0};
    if (d <= 1) return m;  /* degenerate d == 1 (intdiv.py:89-92) */
    const unsigned __int128 word = (unsigned __int128)1 << 32;
    const unsigned __int128 nc = (word / d) * d - 1;
    unsigned __int128 mul = 0;
    int p;
    for (p = 32; p <= 64; p++) {
        unsigned __int128 tp = (unsigned __int128)1 << p, rem = (tp - 1) % d;
        if (tp > nc * (d - 1 - rem)) { mul = (tp + d - 1 - rem) / d; break; }
    }
    m.shift = (uint32_t)(p - 32);
    if (mul < word) { m.mul = (uint32_t)mul; m.add = 0; }
    else { m.mul = (uint32_t)(mul - word); m.add = 1; }
    return m;
}

static inline uint32_t oracle_div(uint32_t n, const omagic *m)
{
    if (m->d == 1) return n;
    uint32_t t = (uint32_t)(((uint64_t)n * m->mul) >> 32);
    return m->add ? (t + ((n - t) >> 1)) >> (m->shift - 1) : t >> m->shift;
}
static inline void oracle_divmod(uint32_t n, const omagic *m, uint32_t *q, uint32_t *r)
{
    *q = oracle_div(n, m);
    *r = n - *q * m->d;
}

/* exported for tests: (multiplier, shift, add) of make_divider(d) */
void oracle_divider_constants(uint32_t d, uint32_t *out3)
{
    omagic m = oracle_make_divider(d);
    out3[0] = m.mul; out3[1] = m.shift; out3[2] = m.add;
}
/* exported for tests: quotients of n[i] / d through the magic path */
void oracle_divide_many(uint32_t d, const uint32_t *n, uint32_t *q, int64_t count)
{
    omagic m = oracle_make_divider(d);
    for (int64_t i = 0; i < count; i++) q[i] = oracle_div(n[i], &m);
}

/* output_extent (conv.py:165-179) */
static int oracle_output_extent(int64_t in, int64_t filt, int64_t stride, int64_t pad, int64_t *out)
{
    if (in < 1 || filt < 1 || stride < 1 || pad < 0) return 0;
    int64_t numer = in - filt + 1 + 2 * pad;
    if (numer < 1) return 0;
    *out = (numer + stride - 1) / stride;
    return 1;
}
int64_t oracle_output_extent_c(int64_t in, int64_t filt, int64_t stride, int64_t pad)
{
    int64_t o;
    return oracle_output_extent(in, filt, stride, pad, &o) ? o : -1;
}

#define REAL float
#define SFX f32
#define EXP expf
#define TANH tanhf
#define FABS fabsf
#include "oracle_impl.h"
#undef REAL
#undef SFX
#undef EXP
#undef TANH
#undef FABS

#define REAL double
#define SFX f64
#define EXP exp
#define TANH tanh
#define FABS fabs
#include "oracle_impl.h"
