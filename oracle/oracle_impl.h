/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle.  Included twice by oracle.c
 * with REAL = float / double and SFX = f32 / f64.  Every routine restates
 * the reference algorithm of pkg/src/dnnp (file:line cited per function);
 * nothing in the product links or calls this code.
 */

/* ---- implicit-GEMM forward (conv.py:538-562 + gemm.py:140-207) ------------
 * O_m[K x NPQ] = F_m[K x CRS] . D_m[CRS x NPQ]; D_m is never stored: each
 * tile is gathered from x through the magic-divider decode of
 * _LoweredMap.fill (conv.py:269-356).  Tiles (min(128,K), min(512,NPQ),
 * min(256,CRS)) as _conv_tile (conv.py:468-470); output tiles are spread
 * over `threads` workers like gemm.py:174-181. */

typedef struct {
    const ov4 *xv; const REAL *x; const REAL *f; REAL *o;
    int64_t N, C, H, W, K, R, S, P, Q, u, v, ph, pw; int flip;
    int64_t tm, tn, tk;
    int64_t nti, ntj;
    int worker, nworkers;
} CAT(fwd_job_, SFX);

static void *CAT(fwd_worker_, SFX)(void *arg)
{
    CAT(fwd_job_, SFX) *jb = arg;
    const int64_t rows = jb->C * jb->R * jb->S, cols = jb->N * jb->P * jb->Q;
    const int64_t tm = jb->tm, tn = jb->tn, tk = jb->tk;
    omagic drs = oracle_make_divider((uint32_t)(jb->R * jb->S)), ds = oracle_make_divider((uint32_t)jb->S);
    omagic dpq = oracle_make_divider((uint32_t)(jb->P * jb->Q)), dq = oracle_make_divider((uint32_t)jb->Q);
    REAL *at = calloc(tm * tk, sizeof(REAL)), *bt = calloc(tk * tn, sizeof(REAL));
    REAL *acc = calloc(tm * tn, sizeof(REAL)), *prod = calloc(tm * tn, sizeof(REAL));
    int64_t *coff = malloc(tn * 8), *chc = malloc(tn * 8), *cwc = malloc(tn * 8);
    int64_t *roff = malloc(tk * 8), *rhr = malloc(tk * 8), *rwr = malloc(tk * 8);
    const ov4 *xv = jb->xv;
    int64_t job = 0;
    for (int64_t ti = 0; ti < jb->nti; ti++) {
        for (int64_t tj = 0; tj < jb->ntj; tj++, job++) {
            if (job % jb->nworkers != jb->worker) continue;
            const int64_t i0 = ti * tm, j0 = tj * tn;
            const int64_t mi = MIN(tm, jb->K - i0), mj = MIN(tn, cols - j0);
            memset(acc, 0, sizeof(REAL) * tm * tn);
            /* column terms of this column range (conv.py:282-289) */
            for (int64_t j = 0; j < mj; j++) {
                uint32_t n, rem, p, q;
                oracle_divmod((uint32_t)(j0 + j), &dpq, &n, &rem);
                oracle_divmod(rem, &dq, &p, &q);
                chc[j] = (int64_t)p * jb->u - jb->ph;
                cwc[j] = (int64_t)q * jb->v - jb->pw;
                coff[j] = (int64_t)n * xv->sn + chc[j] * xv->sh + cwc[j] * xv->sw;
            }
            for (int64_t k0 = 0; k0 < rows; k0 += tk) {
                const int64_t mk = MIN(tk, rows - k0);
                /* filter tile F_m[i0:i0+mi, k0:k0+mk] (zero padded) */
                memset(at, 0, sizeof(REAL) * tm * tk);
                for (int64_t i = 0; i < mi; i++)
                    for (int64_t k = 0; k < mk; k++)
                        at[i * tk + k] = jb->f[(i0 + i) * rows + k0 + k];
                /* row terms (conv.py:269-280) */
                for (int64_t k = 0; k < mk; k++) {
                    uint32_t c, rs, r, s;
                    oracle_divmod((uint32_t)(k0 + k), &drs, &c, &rs);
                    oracle_divmod(rs, &ds, &r, &s);
                    rhr[k] = jb->flip ? jb->R - 1 - (int64_t)r : (int64_t)r;
                    rwr[k] = jb->flip ? jb->S - 1 - (int64_t)s : (int64_t)s;
                    roff[k] = (int64_t)c * xv->sc + rhr[k] * xv->sh + rwr[k] * xv->sw;
                }
                /* gather D_m tile with the zero mask (conv.py:340-356) */
                memset(bt, 0, sizeof(REAL) * tk * tn);
                for (int64_t k = 0; k < mk; k++)
                    for (int64_t j = 0; j < mj; j++) {
                        int64_t h = rhr[k] + chc[j], w = rwr[k] + cwc[j];
                        if (h >= 0 && h < jb->H && w >= 0 && w < jb->W)
                            bt[k * tn + j] = jb->x[roff[k] + coff[j]];
                    }
                /* prod = a_t . b_t ; acc += prod (gemm.py:170-171) */
                memset(prod, 0, sizeof(REAL) * tm * tn);
                for (int64_t i = 0; i < mi; i++)
                    for (int64_t k = 0; k < mk; k++) {
                        const REAL a = at[i * tk + k];
                        REAL *pr = prod + i * tn;
                        const REAL *br = bt + k * tn;
                        for (int64_t j = 0; j < mj; j++) pr[j] += a * br[j];
                    }
                for (int64_t i = 0; i < mi; i++)
                    for (int64_t j = 0; j < mj; j++) acc[i * tn + j] += prod[i * tn + j];
            }
            for (int64_t i = 0; i < mi; i++)
                for (int64_t j = 0; j < mj; j++) jb->o[(i0 + i) * cols + j0 + j] = acc[i * tn + j];
        }
    }
    free(at); free(bt); free(acc); free(prod);
    free(coff); free(chc); free(cwc); free(roff); free(rhr); free(rwr);
    return NULL;
}

int CAT(oracle_conv_forward_, SFX)(const int64_t *xg, const REAL *x, const int64_t *fg,
                                   const REAL *f, const int64_t *cg, const int64_t *yg, REAL *y,
                                   double alpha, double beta, int threads)
{
    ov4 xv = ov4_of(xg), yv = ov4_of(yg);
    const int64_t K = fg[0], R = fg[2], S = fg[3];
    int64_t P, Q;
    if (!oracle_output_extent(xv.h, R, cg[0], cg[2], &P) || !oracle_output_extent(xv.w, S, cg[1], cg[3], &Q))
        return 2;
    const int64_t cols = xv.n * P * Q, rows = xv.c * R * S;
    REAL *o = malloc(sizeof(REAL) * K * cols);
    CAT(fwd_job_, SFX) base = {&xv, x, f, o, xv.n, xv.c, xv.h, xv.w, K, R, S, P, Q,
                               cg[0], cg[1], cg[2], cg[3], cg[4] == 0, 0, 0, 0, 0, 0, 0, 1};
    base.tm = MIN(128, K); base.tn = MIN(512, cols); base.tk = MIN(256, rows);
    base.nti = (K + base.tm - 1) / base.tm; base.ntj = (cols + base.tn - 1) / base.tn;
    if (threads < 1) threads = 1;
    pthread_t th[256];
    CAT(fwd_job_, SFX) jobs[256];
    if (threads > 256) threads = 256;
    for (int t = 0; t < threads; t++) {
        jobs[t] = base; jobs[t].worker = t; jobs[t].nworkers = threads;
        if (threads == 1) CAT(fwd_worker_, SFX)(&jobs[t]);
        else pthread_create(&th[t], NULL, CAT(fwd_worker_, SFX), &jobs[t]);
    }
    if (threads > 1) for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
    /* accumulate forces beta = 1; _combine (conv.py:552-562) */
    if (cg[5]) beta = 1.0;
    for (int64_t n = 0; n < xv.n; n++)
        for (int64_t k = 0; k < K; k++)
            for (int64_t p = 0; p < P; p++)
                for (int64_t q = 0; q < Q; q++) {
                    REAL fresh = o[k * cols + (n * P + p) * Q + q];
                    if (alpha != 1.0) fresh = fresh * (REAL)alpha;
                    REAL *d = y + OFF(yv, n, k, p, q);
                    if (beta == 0.0) *d = fresh;
                    else { if (beta != 1.0) *d = *d * (REAL)beta; *d = *d + fresh; }
                }
    free(o);
    return 0;
}

/* ---- implicit backward-data (conv.py:646-670) -------------------------------
 * gemm_stream(F_m^T [CRS x K], dy_map [K x NPQ]) with serial scatter-add of
 * every finished tile into dx (np.add.at in row-major tile order).  The dy
 * tile is gathered like _OutputGradMap.fill (conv.py:408-425). */
int CAT(oracle_conv_backward_data_, SFX)(const int64_t *fg, const REAL *f, const int64_t *dyg,
                                         const REAL *dy, const int64_t *cg, const int64_t *dxg,
                                         REAL *dx)
{
    ov4 dyv = ov4_of(dyg), dxv = ov4_of(dxg);
    const int64_t K = fg[0], C = fg[1], R = fg[2], S = fg[3];
    int64_t P, Q;
    if (!oracle_output_extent(dxv.h, R, cg[0], cg[2], &P) || !oracle_output_extent(dxv.w, S, cg[1], cg[3], &Q))
        return 2;
    const int64_t rows = C * R * S, cols = dxv.n * P * Q;
    const int64_t tm = MIN(128, rows), tn = MIN(512, cols), tk = MIN(256, K);
    const int flip = cg[4] == 0;
    omagic drs = oracle_make_divider((uint32_t)(R * S)), ds = oracle_make_divider((uint32_t)S);
    omagic dpq = oracle_make_divider((uint32_t)(P * Q)), dq = oracle_make_divider((uint32_t)Q);
    if (!cg[5])
        for (int64_t n = 0; n < dxv.n; n++) for (int64_t c = 0; c < C; c++)
            for (int64_t h = 0; h < dxv.h; h++) for (int64_t w = 0; w < dxv.w; w++)
                dx[OFF(dxv, n, c, h, w)] = 0;
    REAL *acc = malloc(sizeof(REAL) * tm * tn), *prod = malloc(sizeof(REAL) * tm * tn);
    REAL *bt = malloc(sizeof(REAL) * tk * tn);
    int64_t *coff = malloc(8 * tn), *cn = malloc(8 * tn), *chc = malloc(8 * tn), *cwc = malloc(8 * tn);
    for (int64_t i0 = 0; i0 < rows; i0 += tm)
        for (int64_t j0 = 0; j0 < cols; j0 += tn) {
            const int64_t mi = MIN(tm, rows - i0), mj = MIN(tn, cols - j0);
            for (int64_t j = 0; j < mj; j++) {
                uint32_t n, rem, p, q;
                oracle_divmod((uint32_t)(j0 + j), &dpq, &n, &rem);
                oracle_divmod(rem, &dq, &p, &q);
                cn[j] = n;
                coff[j] = (int64_t)n * dyv.sn + (int64_t)p * dyv.sh + (int64_t)q * dyv.sw;
                chc[j] = (int64_t)p * cg[0] - cg[2];
                cwc[j] = (int64_t)q * cg[1] - cg[3];
            }
            memset(acc, 0, sizeof(REAL) * tm * tn);
            for (int64_t k0 = 0; k0 < K; k0 += tk) {
                const int64_t mk = MIN(tk, K - k0);
                for (int64_t k = 0; k < mk; k++)
                    for (int64_t j = 0; j < mj; j++) bt[k * tn + j] = dy[(k0 + k) * dyv.sc + coff[j]];
                memset(prod, 0, sizeof(REAL) * tm * tn);
                for (int64_t i = 0; i < mi; i++)
                    for (int64_t k = 0; k < mk; k++) {
                        /* F_m^T[i][k] = f[k][i] (zero-copy transposed view, gemm.py:74-77) */
                        const REAL a = f[(k0 + k) * rows + i0 + i];
                        REAL *pr = prod + i * tn;
                        const REAL *br = bt + k * tn;
                        for (int64_t j = 0; j < mj; j++) pr[j] += a * br[j];
                    }
                for (int64_t i = 0; i < mi * tn; i++) acc[i] += prod[i];
            }
            /* scatter (conv.py:654-665) */
            for (int64_t i = 0; i < mi; i++) {
                uint32_t c, rs, r, s;
                oracle_divmod((uint32_t)(i0 + i), &drs, &c, &rs);
                oracle_divmod(rs, &ds, &r, &s);
                const int64_t hr = flip ? R - 1 - (int64_t)r : (int64_t)r;
                const int64_t wr = flip ? S - 1 - (int64_t)s : (int64_t)s;
                for (int64_t j = 0; j < mj; j++) {
                    const int64_t h = hr + chc[j], w = wr + cwc[j];
                    if (h >= 0 && h < dxv.h && w >= 0 && w < dxv.w)
                        dx[OFF(dxv, cn[j], c, h, w)] += acc[i * tn + j];
                }
            }
        }
    free(acc); free(prod); free(bt); free(coff); free(cn); free(chc); free(cwc);
    return 0;
}

/* ---- implicit backward-filter (conv.py:710-717) -----------------------------
 * gemm(dy_map [K x NPQ], lowered^T [NPQ x CRS], df [K x CRS]), tiles
 * _conv_tile(K, NPQ, CRS); beta = accumulate; output tiles spread over
 * `threads` workers (gemm.py:174-181). */
typedef struct {
    const ov4 *xv, *dyv; const REAL *x, *dy; REAL *df; const int64_t *cg;
    int64_t K, C, R, S, P, Q; int worker, nworkers;
} CAT(wgrad_job_, SFX);

static void *CAT(wgrad_worker_, SFX)(void *arg)
{
    CAT(wgrad_job_, SFX) *jb = arg;
    const ov4 xv = *jb->xv, dyv = *jb->dyv;
    const int64_t K = jb->K, R = jb->R, S = jb->S, P = jb->P, Q = jb->Q;
    const int64_t *cg = jb->cg;
    const int64_t crs = jb->C * R * S, npq = xv.n * P * Q;
    const int64_t tm = MIN(128, K), tn = MIN(512, crs), tk = MIN(256, npq);
    const int flip = cg[4] == 0;
    omagic drs = oracle_make_divider((uint32_t)(R * S)), ds = oracle_make_divider((uint32_t)S);
    omagic dpq = oracle_make_divider((uint32_t)(P * Q)), dq = oracle_make_divider((uint32_t)Q);
    REAL *acc = malloc(sizeof(REAL) * tm * tn), *prod = malloc(sizeof(REAL) * tm * tn);
    REAL *bt = malloc(sizeof(REAL) * tk * tn), *at = malloc(sizeof(REAL) * tm * tk);
    int64_t *roff = malloc(8 * tn), *rhr = malloc(8 * tn), *rwr = malloc(8 * tn);
    int64_t *koff = malloc(8 * tk), *kdy = malloc(8 * tk), *khc = malloc(8 * tk), *kwc = malloc(8 * tk);
    int64_t job = 0;
    for (int64_t i0 = 0; i0 < K; i0 += tm)
        for (int64_t j0 = 0; j0 < crs; j0 += tn, job++) {
            if (job % jb->nworkers != jb->worker) continue;
            const int64_t mi = MIN(tm, K - i0), mj = MIN(tn, crs - j0);
            for (int64_t j = 0; j < mj; j++) {
                uint32_t c, rs, r, s;
                oracle_divmod((uint32_t)(j0 + j), &drs, &c, &rs);
                oracle_divmod(rs, &ds, &r, &s);
                rhr[j] = flip ? R - 1 - (int64_t)r : (int64_t)r;
                rwr[j] = flip ? S - 1 - (int64_t)s : (int64_t)s;
                roff[j] = (int64_t)c * xv.sc + rhr[j] * xv.sh + rwr[j] * xv.sw;
            }
            memset(acc, 0, sizeof(REAL) * tm * tn);
            for (int64_t k0 = 0; k0 < npq; k0 += tk) {
                const int64_t mk = MIN(tk, npq - k0);
                for (int64_t k = 0; k < mk; k++) {
                    uint32_t n, rem, p, q;
                    oracle_divmod((uint32_t)(k0 + k), &dpq, &n, &rem);
                    oracle_divmod(rem, &dq, &p, &q);
                    khc[k] = (int64_t)p * cg[0] - cg[2];
                    kwc[k] = (int64_t)q * cg[1] - cg[3];
                    koff[k] = (int64_t)n * xv.sn + khc[k] * xv.sh + kwc[k] * xv.sw;
                    kdy[k] = (int64_t)n * dyv.sn + (int64_t)p * dyv.sh + (int64_t)q * dyv.sw;
                }
                for (int64_t i = 0; i < mi; i++)
                    for (int64_t k = 0; k < mk; k++) at[i * tk + k] = jb->dy[kdy[k] + (i0 + i) * dyv.sc];
                for (int64_t k = 0; k < mk; k++)
                    for (int64_t j = 0; j < mj; j++) {
                        const int64_t h = rhr[j] + khc[k], w = rwr[j] + kwc[k];
                        bt[k * tn + j] = (h >= 0 && h < xv.h && w >= 0 && w < xv.w)
                                             ? jb->x[roff[j] + koff[k]] : 0;
                    }
                memset(prod, 0, sizeof(REAL) * tm * tn);
                for (int64_t i = 0; i < mi; i++)
                    for (int64_t k = 0; k < mk; k++) {
                        const REAL a = at[i * tk + k];
                        REAL *pr = prod + i * tn;
                        const REAL *br = bt + k * tn;
                        for (int64_t j = 0; j < mj; j++) pr[j] += a * br[j];
                    }
                for (int64_t i = 0; i < mi * tn; i++) acc[i] += prod[i];
            }
            for (int64_t i = 0; i < mi; i++)
                for (int64_t j = 0; j < mj; j++) {
                    REAL *d = jb->df + (i0 + i) * crs + j0 + j;
                    if (cg[5]) *d = *d + acc[i * tn + j];
                    else *d = acc[i * tn + j];
                }
        }
    free(acc); free(prod); free(bt); free(at); free(roff); free(rhr); free(rwr);
    free(koff); free(kdy); free(khc); free(kwc);
    return NULL;
}

int CAT(oracle_conv_backward_filter_, SFX)(const int64_t *xg, const REAL *x, const int64_t *dyg,
                                           const REAL *dy, const int64_t *cg, const int64_t *fg,
                                           REAL *df, int threads)
{
    ov4 xv = ov4_of(xg), dyv = ov4_of(dyg);
    int64_t P, Q;
    if (!oracle_output_extent(xv.h, fg[2], cg[0], cg[2], &P) || !oracle_output_extent(xv.w, fg[3], cg[1], cg[3], &Q))
        return 2;
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    CAT(wgrad_job_, SFX) jobs[256];
    for (int t = 0; t < threads; t++) {
        CAT(wgrad_job_, SFX) j = {&xv, &dyv, x, dy, df, cg, fg[0], fg[1], fg[2], fg[3], P, Q, t, threads};
        jobs[t] = j;
        if (threads == 1) CAT(wgrad_worker_, SFX)(&jobs[t]);
        else pthread_create(&th[t], NULL, CAT(wgrad_worker_, SFX), &jobs[t]);
    }
    if (threads > 1) for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
    return 0;
}

/* ---- bias gradient (conv.py:754-760) -------------------------------------- */
int CAT(oracle_conv_backward_bias_, SFX)(const int64_t *dyg, const REAL *dy, REAL *db)
{
    ov4 v = ov4_of(dyg);
    for (int64_t k = 0; k < v.c; k++) {
        REAL s = 0;
        for (int64_t n = 0; n < v.n; n++)
            for (int64_t h = 0; h < v.h; h++)
                for (int64_t w = 0; w < v.w; w++) s += dy[OFF(v, n, k, h, w)];
        db[k] = s;
    }
    return 0;
}

/* ---- activation (nnops.py:54-88) ------------------------------------------ */
int CAT(oracle_activation_forward_, SFX)(int kind, const int64_t *xg, const REAL *x,
                                         const int64_t *yg, REAL *y)
{
    ov4 xv = ov4_of(xg), yv = ov4_of(yg);
    FOR4(xv) {
        REAL a = x[OFF(xv, n, c, h, w)], r;
        if (kind == 1) r = (a > 0 || a != a) ? a : 0;
        else if (kind == 2) r = TANH(a);
        else { REAL e = EXP(-FABS(a)); r = a >= 0 ? (REAL)1 / ((REAL)1 + e) : e / ((REAL)1 + e); }
        y[OFF(yv, n, c, h, w)] = r;
    }
    return 0;
}

int CAT(oracle_activation_backward_, SFX)(int kind, const int64_t *yg, const REAL *y,
                                          const int64_t *dyg, const REAL *dy, const int64_t *dxg,
                                          REAL *dx)
{
    ov4 yv = ov4_of(yg), dyv = ov4_of(dyg), dxv = ov4_of(dxg);
    FOR4(yv) {
        volatile REAL a = y[OFF(yv, n, c, h, w)], d = dy[OFF(dyv, n, c, h, w)];
        volatile REAL r, t;
        if (kind == 1) { r = d * (a > 0 ? (REAL)1 : (REAL)0); }
        else if (kind == 2) { t = a * a; t = (REAL)1 - t; r = d * t; }
        else { t = d * a; r = (REAL)1 - a; r = t * r; }
        dx[OFF(dxv, n, c, h, w)] = r;
    }
    return 0;
}

/* ---- softmax (nnops.py:91-117) -------------------------------------------- */
int CAT(oracle_softmax_forward_, SFX)(int mode, const int64_t *xg, const REAL *x,
                                      const int64_t *yg, REAL *y)
{
    ov4 xv = ov4_of(xg), yv = ov4_of(yg);
    if (mode == 0) {
        for (int64_t n = 0; n < xv.n; n++) {
            REAL m = -INFINITY, s = 0;
            for (int64_t c = 0; c < xv.c; c++) for (int64_t h = 0; h < xv.h; h++) for (int64_t w = 0; w < xv.w; w++) {
                REAL a = x[OFF(xv, n, c, h, w)]; if (a > m || a != a) m = a; }
            for (int64_t c = 0; c < xv.c; c++) for (int64_t h = 0; h < xv.h; h++) for (int64_t w = 0; w < xv.w; w++)
                s += EXP(x[OFF(xv, n, c, h, w)] - m);
            for (int64_t c = 0; c < xv.c; c++) for (int64_t h = 0; h < xv.h; h++) for (int64_t w = 0; w < xv.w; w++)
                y[OFF(yv, n, c, h, w)] = EXP(x[OFF(xv, n, c, h, w)] - m) / s;
        }
    } else {
        for (int64_t n = 0; n < xv.n; n++) for (int64_t h = 0; h < xv.h; h++) for (int64_t w = 0; w < xv.w; w++) {
            REAL m = -INFINITY, s = 0;
            for (int64_t c = 0; c < xv.c; c++) { REAL a = x[OFF(xv, n, c, h, w)]; if (a > m || a != a) m = a; }
            for (int64_t c = 0; c < xv.c; c++) s += EXP(x[OFF(xv, n, c, h, w)] - m);
            for (int64_t c = 0; c < xv.c; c++) y[OFF(yv, n, c, h, w)] = EXP(x[OFF(xv, n, c, h, w)] - m) / s;
        }
    }
    return 0;
}

int CAT(oracle_softmax_backward_, SFX)(int mode, const int64_t *yg, const REAL *y,
                                       const int64_t *dyg, const REAL *dy, const int64_t *dxg,
                                       REAL *dx)
{
    ov4 yv = ov4_of(yg), dyv = ov4_of(dyg), dxv = ov4_of(dxg);
    if (mode == 0) {
        for (int64_t n = 0; n < yv.n; n++) {
            REAL dot = 0;
            for (int64_t c = 0; c < yv.c; c++) for (int64_t h = 0; h < yv.h; h++) for (int64_t w = 0; w < yv.w; w++)
                dot += y[OFF(yv, n, c, h, w)] * dy[OFF(dyv, n, c, h, w)];
            for (int64_t c = 0; c < yv.c; c++) for (int64_t h = 0; h < yv.h; h++) for (int64_t w = 0; w < yv.w; w++)
                dx[OFF(dxv, n, c, h, w)] = y[OFF(yv, n, c, h, w)] * (dy[OFF(dyv, n, c, h, w)] - dot);
        }
    } else {
        for (int64_t n = 0; n < yv.n; n++) for (int64_t h = 0; h < yv.h; h++) for (int64_t w = 0; w < yv.w; w++) {
            REAL dot = 0;
            for (int64_t c = 0; c < yv.c; c++) dot += y[OFF(yv, n, c, h, w)] * dy[OFF(dyv, n, c, h, w)];
            for (int64_t c = 0; c < yv.c; c++)
                dx[OFF(dxv, n, c, h, w)] = y[OFF(yv, n, c, h, w)] * (dy[OFF(dyv, n, c, h, w)] - dot);
        }
    }
    return 0;
}

/* ---- pooling (nnops.py:150-246) ------------------------------------------- */
int CAT(oracle_pool_forward_, SFX)(const int64_t *pg, const int64_t *xg, const REAL *x,
                                   const int64_t *yg, REAL *y, int64_t *argmax)
{
    /* pg: kind, wh, ww, sh, sw, ph, pw */
    ov4 xv = ov4_of(xg), yv = ov4_of(yg);
    int64_t P, Q;
    if (!oracle_output_extent(xv.h, pg[1], pg[3], pg[5], &P) || !oracle_output_extent(xv.w, pg[2], pg[4], pg[6], &Q))
        return 2;
    for (int64_t n = 0; n < xv.n; n++) for (int64_t c = 0; c < xv.c; c++)
        for (int64_t p = 0; p < P; p++) for (int64_t q = 0; q < Q; q++) {
            int64_t hs0 = p * pg[3] - pg[5], ws0 = q * pg[4] - pg[6];
            int64_t hs = MAX(0, hs0), he = MIN(xv.h, hs0 + pg[1]);
            int64_t ws = MAX(0, ws0), we = MIN(xv.w, ws0 + pg[2]);
            if (hs >= he || ws >= we) return 2;  /* EmptyWindow */
            REAL out;
            if (pg[0] == 0) {
                REAL best = x[OFF(xv, n, c, hs, ws)]; int64_t bh = hs, bw = ws;
                for (int64_t h = hs; h < he; h++) for (int64_t w = ws; w < we; w++) {
                    REAL a = x[OFF(xv, n, c, h, w)];
                    if (best != best) continue;
                    if (a != a || a > best) { best = a; bh = h; bw = w; }
                }
                out = best;
                if (argmax) argmax[((n * xv.c + c) * P + p) * Q + q] = ((n * xv.c + c) * xv.h + bh) * xv.w + bw;
            } else {
                REAL s = 0;
                for (int64_t h = hs; h < he; h++) for (int64_t w = ws; w < we; w++) s += x[OFF(xv, n, c, h, w)];
                out = s / (REAL)((he - hs) * (we - ws));
            }
            y[OFF(yv, n, c, p, q)] = out;
        }
    return 0;
}

int CAT(oracle_pool_backward_, SFX)(const int64_t *pg, const int64_t *dyg, const REAL *dy,
                                    const int64_t *dxg, REAL *dx, const int64_t *argmax)
{
    ov4 dyv = ov4_of(dyg), dxv = ov4_of(dxg);
    const int64_t P = dyv.h, Q = dyv.w;
    FOR4(dxv) dx[OFF(dxv, n, c, h, w)] = 0;
    if (pg[0] == 0) {
        /* np.add.at in flat (n, c, p, q) order */
        const int64_t H = dxv.h, W = dxv.w, C = dxv.c;
        for (int64_t n = 0; n < dyv.n; n++) for (int64_t c = 0; c < C; c++)
            for (int64_t p = 0; p < P; p++) for (int64_t q = 0; q < Q; q++) {
                int64_t a = argmax[((n * C + c) * P + p) * Q + q];
                int64_t ww = a % W, hh = (a / W) % H, cc = (a / (W * H)) % C, nn = a / (W * H * C);
                REAL *t = dx + OFF(dxv, nn, cc, hh, ww);
                *t = *t + dy[OFF(dyv, n, c, p, q)];
            }
    } else {
        for (int64_t p = 0; p < P; p++) for (int64_t q = 0; q < Q; q++) {
            int64_t hs0 = p * pg[3] - pg[5], ws0 = q * pg[4] - pg[6];
            int64_t hs = MAX(0, hs0), he = MIN(dxv.h, hs0 + pg[1]);
            int64_t ws = MAX(0, ws0), we = MIN(dxv.w, ws0 + pg[2]);
            int64_t cnt = (he - hs) * (we - ws);
            if (cnt <= 0) return 2;
            for (int64_t n = 0; n < dyv.n; n++) for (int64_t c = 0; c < dyv.c; c++) {
                REAL g = dy[OFF(dyv, n, c, p, q)] / (REAL)cnt;
                for (int64_t h = hs; h < he; h++) for (int64_t w = ws; w < we; w++) {
                    REAL *t = dx + OFF(dxv, n, c, h, w);
                    *t = *t + g;
                }
            }
        }
    }
    return 0;
}

/* ---- transform / add_broadcast (tensor.py:241-271) ------------------------ */
int CAT(oracle_transform_, SFX)(const int64_t *sg, const REAL *s, const int64_t *dg, REAL *d,
                                double alpha, double beta)
{
    ov4 sv = ov4_of(sg), dv = ov4_of(dg);
    FOR4(sv) {
        volatile REAL as = s[OFF(sv, n, c, h, w)] * (REAL)alpha;
        REAL *t = d + OFF(dv, n, c, h, w);
        if (beta == 0) *t = as;
        else { volatile REAL b = *t * (REAL)beta; *t = b + as; }
    }
    return 0;
}

int CAT(oracle_add_broadcast_, SFX)(const int64_t *bg, const REAL *b, const int64_t *og, REAL *o,
                                    double alpha, double beta)
{
    ov4 bv = ov4_of(bg), ov = ov4_of(og);
    FOR4(ov) {
        int64_t bn = bv.n == 1 ? 0 : n, bc = bv.c == 1 ? 0 : c, bh = bv.h == 1 ? 0 : h, bw = bv.w == 1 ? 0 : w;
        volatile REAL ab = b[OFF(bv, bn, bc, bh, bw)] * (REAL)alpha;
        REAL *t = o + OFF(ov, n, c, h, w);
        if (beta == 0) *t = ab;
        else { volatile REAL x = *t * (REAL)beta; *t = x + ab; }
    }
    return 0;
}
