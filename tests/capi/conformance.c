/*
 * C conformance program for libdnnp.so, written against include/dnnp.h the
 * way a reference caller uses pkg/capi (reference tests: capi/tests/test_capi.c,
 * capi/examples/conv_example.c).  It exercises descriptor round trips, the
 * status contract for NULLs / zero extents / huge strides / aliasing /
 * double destroy, numeric known answers (Fig.1 example golden bytes, exact
 * f64 1x1 product, engine agreement, max-pool KAT, layout round trip) and
 * concurrent calls from four threads on disjoint outputs.
 *
 * Usage: conformance [--status-only]   (status-only skips compute checks,
 * for hosts without a GPU).  Exit code = number of failed checks.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "dnnp.h"

static int n_pass, n_fail;
static dnnp_handle H;

#define EXPECT(cond, name)                                          \
    do {                                                            \
        if (cond) { n_pass++; printf("ok   %s\n", name); }          \
        else { n_fail++; printf("FAIL %s (%s)\n", name, dnnp_last_error()); } \
    } while (0)

static void descriptors(void)
{
    dnnp_tensor_desc t = NULL;
    dnnp_elem_type et;
    int64_t n, c, h, w, sn, sc, sh, sw;
    EXPECT(dnnp_tensor_desc_create(&t) == DNNP_STATUS_OK, "tensor create");
    EXPECT(dnnp_tensor_desc_get(t, &et, &n, &c, &h, &w, &sn, &sc, &sh, &sw) == DNNP_STATUS_BAD_PARAM,
           "get before set");
    EXPECT(dnnp_tensor_desc_set(t, DNNP_F32, 2, 3, 4, 5) == DNNP_STATUS_OK, "set dense");
    EXPECT(dnnp_tensor_desc_get(t, &et, &n, &c, &h, &w, &sn, &sc, &sh, &sw) == DNNP_STATUS_OK &&
               sn == 60 && sc == 20 && sh == 5 && sw == 1 && et == DNNP_F32,
           "dense strides");
    EXPECT(dnnp_tensor_desc_set_ex(t, DNNP_F64, 2, 3, 4, 5, 60, 1, 15, 3) == DNNP_STATUS_OK,
           "NHWC strides");
    EXPECT(dnnp_tensor_desc_set_ex(t, DNNP_F64, 4, 4, 4, 4, INT64_MAX / 2, 1, 1, 1) ==
               DNNP_STATUS_BAD_PARAM, "span guard");
    EXPECT(dnnp_tensor_desc_set(t, DNNP_F64, 0, 1, 1, 1) == DNNP_STATUS_BAD_PARAM, "zero extent");
    EXPECT(dnnp_tensor_desc_set(t, (dnnp_elem_type)5, 1, 1, 1, 1) == DNNP_STATUS_BAD_PARAM,
           "bad element type");
    EXPECT(dnnp_tensor_desc_destroy(t) == DNNP_STATUS_OK, "tensor destroy");
    EXPECT(dnnp_tensor_desc_destroy(t) == DNNP_STATUS_BAD_PARAM, "double destroy");
    EXPECT(dnnp_tensor_desc_destroy(NULL) == DNNP_STATUS_BAD_PARAM, "destroy NULL");

    dnnp_filter_desc f;
    dnnp_conv_desc cv;
    dnnp_pooling_desc pd;
    int64_t k, r, s, u, v, ph, pw, wh, ww, shh, sww;
    dnnp_conv_mode mode;
    dnnp_pool_kind kind;
    int acc;
    dnnp_filter_desc_create(&f);
    EXPECT(dnnp_filter_desc_set(f, DNNP_F64, 8, 4, 3, 2) == DNNP_STATUS_OK &&
               dnnp_filter_desc_get(f, &et, &k, &c, &r, &s) == DNNP_STATUS_OK && k == 8 &&
               c == 4 && r == 3 && s == 2,
           "filter round trip");
    dnnp_conv_desc_create(&cv);
    EXPECT(dnnp_conv_desc_set(cv, 2, 3, 1, 0, DNNP_CROSS_CORRELATION, 5) == DNNP_STATUS_OK &&
               dnnp_conv_desc_get(cv, &u, &v, &ph, &pw, &mode, &acc) == DNNP_STATUS_OK &&
               u == 2 && v == 3 && ph == 1 && pw == 0 && mode == DNNP_CROSS_CORRELATION &&
               acc == 1,
           "conv round trip (accumulate normalised to 1)");
    EXPECT(dnnp_conv_desc_set(cv, 1, 1, -1, 0, DNNP_CONVOLUTION, 0) == DNNP_STATUS_BAD_PARAM,
           "negative pad");
    dnnp_pooling_desc_create(&pd);
    EXPECT(dnnp_pooling_desc_set(pd, DNNP_POOL_MAX, 3, 2, 2, 1, 1, 0) == DNNP_STATUS_OK &&
               dnnp_pooling_desc_get(pd, &kind, &wh, &ww, &shh, &sww, &ph, &pw) ==
                   DNNP_STATUS_OK && wh == 3 && ww == 2 && shh == 2 && sww == 1 && ph == 1,
           "pooling round trip");
    EXPECT(dnnp_pooling_desc_set(pd, (dnnp_pool_kind)3, 1, 1, 1, 1, 0, 0) == DNNP_STATUS_BAD_PARAM,
           "bad pool kind");
    dnnp_filter_desc_destroy(f);
    dnnp_conv_desc_destroy(cv);
    dnnp_pooling_desc_destroy(pd);
}

static void compute_statuses(void)
{
    dnnp_tensor_desc a, b;
    dnnp_filter_desc f;
    dnnp_conv_desc cv;
    double x[64] = {0}, y[64] = {0}, one = 1.0, zero = 0.0;
    dnnp_tensor_desc_create(&a);
    dnnp_tensor_desc_create(&b);
    dnnp_tensor_desc_set(a, DNNP_F64, 1, 1, 4, 4);
    dnnp_tensor_desc_set(b, DNNP_F64, 1, 1, 4, 4);
    EXPECT(dnnp_activation_forward(H, DNNP_ACTIVATION_RELU, a, NULL, b, y) == DNNP_STATUS_BAD_PARAM,
           "NULL input buffer");
    EXPECT(dnnp_activation_forward(NULL, DNNP_ACTIVATION_RELU, a, x, b, y) == DNNP_STATUS_BAD_PARAM,
           "NULL handle");
    EXPECT(dnnp_activation_forward(H, (dnnp_activation_kind)9, a, x, b, y) == DNNP_STATUS_BAD_PARAM,
           "bad activation kind");
    dnnp_tensor_desc_set_ex(b, DNNP_F64, 1, 2, 2, 2, 8, 0, 2, 1);
    EXPECT(dnnp_activation_forward(H, DNNP_ACTIVATION_RELU, b, x, b, y) == DNNP_STATUS_BAD_PARAM,
           "aliasing strides at compute");
    dnnp_tensor_desc_set_ex(b, DNNP_F64, 1, 1, 4, 4, 16, 16, -4, 1);
    EXPECT(dnnp_activation_forward(H, DNNP_ACTIVATION_RELU, a, x, b, y) ==
               DNNP_STATUS_SHAPE_MISMATCH, "negative reach is shape_mismatch");
    dnnp_tensor_desc_set(b, DNNP_F64, 1, 1, 4, 3);
    EXPECT(dnnp_activation_forward(H, DNNP_ACTIVATION_RELU, a, x, b, y) ==
               DNNP_STATUS_SHAPE_MISMATCH, "extent mismatch");
    dnnp_tensor_desc_set(b, DNNP_F64, 1, 1, 4, 4);
    dnnp_filter_desc_create(&f);
    dnnp_filter_desc_set(f, DNNP_F64, 1, 3, 2, 2);
    dnnp_conv_desc_create(&cv);
    dnnp_conv_desc_set(cv, 1, 1, 0, 0, DNNP_CONVOLUTION, 0);
    EXPECT(dnnp_convolution_forward(H, &one, a, x, f, x, cv, DNNP_ENGINE_IMPLICIT, &zero, b, y) ==
               DNNP_STATUS_SHAPE_MISMATCH, "channel mismatch");
    EXPECT(dnnp_convolution_forward(H, &one, a, x, f, x, cv, (dnnp_engine)3, &zero, b, y) ==
               DNNP_STATUS_BAD_PARAM, "bad engine");
    EXPECT(dnnp_convolution_forward(H, NULL, a, x, f, x, cv, DNNP_ENGINE_IMPLICIT, &zero, b, y) ==
               DNNP_STATUS_BAD_PARAM, "NULL alpha");
    dnnp_filter_desc_set(f, DNNP_F64, 1, 1, 5, 5);
    EXPECT(dnnp_convolution_forward(H, &one, a, x, f, x, cv, DNNP_ENGINE_IMPLICIT, &zero, b, y) ==
               DNNP_STATUS_SHAPE_MISMATCH, "empty output");
    EXPECT(dnnp_transform(H, &one, a, x, &zero, b, x) == DNNP_STATUS_SHAPE_MISMATCH,
           "overlapping transform");
    dnnp_tensor_desc_destroy(a);
    dnnp_tensor_desc_destroy(b);
    dnnp_filter_desc_destroy(f);
    dnnp_conv_desc_destroy(cv);
}

/* Fig.1 sized example (conv_example.c): the golden bytes of the reference
 * native path are [7, -36, 10, -11, -5, 5, 25, -9]. */
static void fig1_example(void)
{
    float x[27], f[24], y[8], alpha = 1.0f, beta = 0.0f;
    const float golden[8] = {7, -36, 10, -11, -5, 5, 25, -9};
    int i;
    int64_t on, ok, op, oq;
    dnnp_tensor_desc xd, yd;
    dnnp_filter_desc fd;
    dnnp_conv_desc cd;
    for (i = 0; i < 27; i++) x[i] = (float)((i % 11) - 5);
    for (i = 0; i < 24; i++) f[i] = (float)(((i * 3) % 7) - 3);
    dnnp_tensor_desc_create(&xd);
    dnnp_tensor_desc_set(xd, DNNP_F32, 1, 3, 3, 3);
    dnnp_filter_desc_create(&fd);
    dnnp_filter_desc_set(fd, DNNP_F32, 2, 3, 2, 2);
    dnnp_conv_desc_create(&cd);
    dnnp_conv_desc_set(cd, 1, 1, 0, 0, DNNP_CONVOLUTION, 0);
    EXPECT(dnnp_conv_output_shape(xd, fd, cd, &on, &ok, &op, &oq) == DNNP_STATUS_OK && on == 1 &&
               ok == 2 && op == 2 && oq == 2, "output shape");
    dnnp_tensor_desc_create(&yd);
    dnnp_tensor_desc_set(yd, DNNP_F32, 1, 2, 2, 2);
    EXPECT(dnnp_convolution_forward(H, &alpha, xd, x, fd, f, cd, DNNP_ENGINE_IMPLICIT, &beta, yd, y) ==
               DNNP_STATUS_OK, "fig1 forward");
    EXPECT(memcmp(y, golden, sizeof y) == 0, "fig1 output bit-identical to reference golden");
    dnnp_tensor_desc_destroy(xd);
    dnnp_tensor_desc_destroy(yd);
    dnnp_filter_desc_destroy(fd);
    dnnp_conv_desc_destroy(cd);
}

static void numerics(void)
{
    /* exact f64 1x1 product */
    {
        dnnp_tensor_desc a, b;
        dnnp_filter_desc f;
        dnnp_conv_desc cv;
        double x = 3.5, w = -2.0, y = 99.0, one = 1.0, zero = 0.0;
        dnnp_tensor_desc_create(&a);
        dnnp_tensor_desc_create(&b);
        dnnp_tensor_desc_set(a, DNNP_F64, 1, 1, 1, 1);
        dnnp_tensor_desc_set(b, DNNP_F64, 1, 1, 1, 1);
        dnnp_filter_desc_create(&f);
        dnnp_filter_desc_set(f, DNNP_F64, 1, 1, 1, 1);
        dnnp_conv_desc_create(&cv);
        dnnp_conv_desc_set(cv, 1, 1, 0, 0, DNNP_CONVOLUTION, 0);
        EXPECT(dnnp_convolution_forward(H, &one, a, &x, f, &w, cv, DNNP_ENGINE_DIRECT, &zero, b, &y) ==
                   DNNP_STATUS_OK && y == -7.0, "f64 1x1 exact");
        dnnp_tensor_desc_destroy(a);
        dnnp_tensor_desc_destroy(b);
        dnnp_filter_desc_destroy(f);
        dnnp_conv_desc_destroy(cv);
    }
    /* all engine values agree (one kernel family) */
    {
        enum { N = 1, C = 2, HH = 5, W = 5, K = 3, R = 3, S = 3, P = 3, Q = 3 };
        double x[N * C * HH * W], f[K * C * R * S], y0[27], y1[27], y2[27], one = 1, zero = 0;
        dnnp_tensor_desc xd, yd;
        dnnp_filter_desc fd;
        dnnp_conv_desc cd;
        int i, same = 1;
        for (i = 0; i < N * C * HH * W; i++) x[i] = ((i * 13) % 17) / 4.0 - 2.0;
        for (i = 0; i < K * C * R * S; i++) f[i] = ((i * 5) % 11) / 2.0 - 2.5;
        dnnp_tensor_desc_create(&xd);
        dnnp_tensor_desc_set(xd, DNNP_F64, N, C, HH, W);
        dnnp_tensor_desc_create(&yd);
        dnnp_tensor_desc_set(yd, DNNP_F64, N, K, P, Q);
        dnnp_filter_desc_create(&fd);
        dnnp_filter_desc_set(fd, DNNP_F64, K, C, R, S);
        dnnp_conv_desc_create(&cd);
        dnnp_conv_desc_set(cd, 1, 1, 0, 0, DNNP_CROSS_CORRELATION, 0);
        EXPECT(dnnp_convolution_forward(H, &one, xd, x, fd, f, cd, DNNP_ENGINE_EXPLICIT, &zero, yd, y0) == 0 &&
                   dnnp_convolution_forward(H, &one, xd, x, fd, f, cd, DNNP_ENGINE_IMPLICIT, &zero, yd, y1) == 0 &&
                   dnnp_convolution_forward(H, &one, xd, x, fd, f, cd, DNNP_ENGINE_DIRECT, &zero, yd, y2) == 0,
               "three engine values run");
        for (i = 0; i < 27; i++) same &= (y0[i] == y1[i]) && (y1[i] == y2[i]);
        EXPECT(same, "engines agree bitwise");
        dnnp_tensor_desc_destroy(xd);
        dnnp_tensor_desc_destroy(yd);
        dnnp_filter_desc_destroy(fd);
        dnnp_conv_desc_destroy(cd);
    }
    /* max pooling KAT and layout round trip */
    {
        dnnp_pooling_desc pd;
        dnnp_tensor_desc xd, yd, nchw, nhwc;
        double x[16], y[4], src[24], mid[24], back[24], one = 1, zero = 0;
        int64_t am[4];
        int i, eq = 1;
        for (i = 0; i < 16; i++) x[i] = (double)((i * 7) % 16);
        dnnp_pooling_desc_create(&pd);
        dnnp_pooling_desc_set(pd, DNNP_POOL_MAX, 2, 2, 2, 2, 0, 0);
        dnnp_tensor_desc_create(&xd);
        dnnp_tensor_desc_set(xd, DNNP_F64, 1, 1, 4, 4);
        dnnp_tensor_desc_create(&yd);
        dnnp_tensor_desc_set(yd, DNNP_F64, 1, 1, 2, 2);
        EXPECT(dnnp_pooling_forward(H, pd, xd, x, yd, y, am) == DNNP_STATUS_OK && y[0] == 12 &&
                   y[1] == 14 && y[2] == 15 && y[3] == 13, "max pool values");
        EXPECT(am[0] == 4 && am[1] == 2 && am[2] == 9 && am[3] == 11, "max pool argmax (logical)");
        for (i = 0; i < 24; i++) src[i] = i * 0.5 - 3.0;
        dnnp_tensor_desc_create(&nchw);
        dnnp_tensor_desc_set(nchw, DNNP_F64, 2, 3, 2, 2);
        dnnp_tensor_desc_create(&nhwc);
        dnnp_tensor_desc_set_ex(nhwc, DNNP_F64, 2, 3, 2, 2, 12, 1, 6, 3);
        EXPECT(dnnp_transform(H, &one, nchw, src, &zero, nhwc, mid) == 0 &&
                   dnnp_transform(H, &one, nhwc, mid, &zero, nchw, back) == 0, "transform both ways");
        for (i = 0; i < 24; i++) eq &= back[i] == src[i];
        EXPECT(eq, "layout round trip is the identity");
        dnnp_pooling_desc_destroy(pd);
        dnnp_tensor_desc_destroy(xd);
        dnnp_tensor_desc_destroy(yd);
        dnnp_tensor_desc_destroy(nchw);
        dnnp_tensor_desc_destroy(nhwc);
    }
}

struct warg { dnnp_tensor_desc d; const double *x; double *y; int bad; };

static void *worker(void *p)
{
    struct warg *a = p;
    for (int i = 0; i < 50; i++)
        if (dnnp_activation_forward(H, DNNP_ACTIVATION_RELU, a->d, a->x, a->d, a->y) != 0) a->bad = 1;
    return NULL;
}

static void concurrency(void)
{
    double x[64], y[4][64];
    pthread_t th[4];
    struct warg args[4];
    dnnp_tensor_desc d;
    int i, t, ok = 1, vals = 1;
    for (i = 0; i < 64; i++) x[i] = (i % 2) ? i : -i;
    dnnp_tensor_desc_create(&d);
    dnnp_tensor_desc_set(d, DNNP_F64, 1, 1, 8, 8);
    for (t = 0; t < 4; t++) {
        args[t].d = d; args[t].x = x; args[t].y = y[t]; args[t].bad = 0;
        pthread_create(&th[t], NULL, worker, &args[t]);
    }
    for (t = 0; t < 4; t++) { pthread_join(th[t], NULL); ok &= !args[t].bad; }
    for (t = 0; t < 4; t++)
        for (i = 0; i < 64; i++) vals &= y[t][i] == (x[i] > 0 ? x[i] : 0.0);
    EXPECT(ok, "concurrent calls ok");
    EXPECT(vals, "concurrent results correct");
    dnnp_tensor_desc_destroy(d);
}

int main(int argc, char **argv)
{
    int status_only = argc > 1 && strcmp(argv[1], "--status-only") == 0;
    dnnp_tensor_desc x;
    dnnp_filter_desc f;
    dnnp_conv_desc c;
    int64_t on;
    dnnp_tensor_desc_create(&x);
    dnnp_filter_desc_create(&f);
    dnnp_conv_desc_create(&c);
    dnnp_tensor_desc_set(x, DNNP_F32, 1, 1, 3, 3);
    dnnp_filter_desc_set(f, DNNP_F32, 1, 1, 2, 2);
    dnnp_conv_desc_set(c, 1, 1, 0, 0, DNNP_CONVOLUTION, 0);
    EXPECT(dnnp_conv_output_shape(x, f, c, &on, NULL, NULL, NULL) == DNNP_STATUS_BAD_PARAM,
           "output_shape before first create");
    EXPECT(dnnp_version() == DNNP_VERSION && DNNP_VERSION == 100, "version");
    EXPECT(strcmp(dnnp_status_string(DNNP_STATUS_SHAPE_MISMATCH), "shape_mismatch") == 0,
           "status strings");
    EXPECT(dnnp_create(NULL) == DNNP_STATUS_BAD_PARAM, "create(NULL)");
    EXPECT(dnnp_create(&H) == DNNP_STATUS_OK, "create");
    EXPECT(dnnp_conv_output_shape(x, f, c, &on, NULL, NULL, NULL) == DNNP_STATUS_OK && on == 1,
           "output_shape after create");
    EXPECT(dnnp_set_threads(H, 0) == DNNP_STATUS_BAD_PARAM, "threads < 1");
    EXPECT(dnnp_set_threads(H, 4) == DNNP_STATUS_OK, "set threads");
    dnnp_tensor_desc_destroy(x);
    dnnp_filter_desc_destroy(f);
    dnnp_conv_desc_destroy(c);
    descriptors();
    compute_statuses();
    if (!status_only) {
        fig1_example();
        numerics();
        concurrency();
    }
    EXPECT(dnnp_destroy(H) == DNNP_STATUS_OK, "destroy");
    EXPECT(dnnp_destroy(H) == DNNP_STATUS_BAD_PARAM, "double destroy handle");
    printf("%d passed, %d failed\n", n_pass, n_fail);
    return n_fail;
}
