/*
 * oracle.c -- CPU ORACLE for arXiv 1605.02164 (MCSF). TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library. The product path (libbfvec.so and the
 * Python binding) never links, loads or calls it. It shares no code, headers
 * or constants with paper_1605_02164_b200/csrc.
 *
 * Plain fp64, no blocking/fusion/reordering beyond what the paper states.
 * OpenMP parallelises independent rows only (results are independent of the
 * thread count: each output element is computed by one thread in a fixed
 * order).
 *
 *   oracle_mcsf_alg1  -- Algorithm 1 step by step, with the
 *                        Gaussian convolutions done separably (PAPER.md:204,
 *                        "using separability") and the real-part convention
 *                        of DESIGN.md reading R4 at the final division.
 *   oracle_direct     -- the exact bilateral filter Eq. (2)-(3)
 *                         on the square window of PAPER.md:46.
 *
 * Boundary (paper silent; reading R1): half-sample symmetric
 * reflection, period 2n, applied per axis.
 *
 * Both functions work on a row SLAB of the full image so that bounded samples
 * of very large images (config 5) can be computed: the slab holds image rows
 * [slab_row0, slab_row0 + slab_rows) of a full image of height H; the outputs
 * are rows [out_row0, out_row0 + out_rows). Every (reflected) input row an
 * output needs must lie in the slab, else the call returns -2.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* half-sample symmetric reflection into [0, n) (reading R1) */
static long refl(long i, long n) {
    long p = 2 * n;
    i %= p;
    if (i < 0) i += p;
    return i < n ? i : p - 1 - i;
}

static int check_slab(int H, int slab_row0, int slab_rows, int out_row0, int out_rows, int r) {
    if (out_row0 < 0 || out_rows < 0 || out_row0 + out_rows > H) return -1;
    if (slab_row0 < 0 || slab_rows < 1 || slab_row0 + slab_rows > H) return -1;
    for (long y = out_row0; y < (long)out_row0 + out_rows; ++y)
        for (long m = -r; m <= r; ++m) {
            long yy = refl(y - m, H);
            if (yy < slab_row0 || yy >= (long)slab_row0 + slab_rows) return -2;
        }
    return 0;
}

/*
 * Algorithm 1 (MCSF).
 *   f      planar float (d, slab_rows, W), rows of the full image
 *   Q      d x d row-major, orthogonal; alpha[d] > 0   (Eq. (4))
 *   Y      T x d integers Y_k^(t) = N - 2 X_k^(t)
 *   w      2r+1 separable spatial taps, w[m + r] for m in [-r, r]
 *   P      out (d, out_rows, W)  Re of the accumulated numerator
 *   Z      out (out_rows, W)     Re of the accumulated denominator
 *   Pim/Zim optional imaginary parts (may be NULL)
 * The 1/T factors of Eq. (15)-(19) cancel in the division and are omitted as
 * in Algorithm 1 (reading R13), so P and Z are raw sums over t.
 */
int oracle_mcsf_alg1(int H, int W, int d, const float *f, int slab_row0, int slab_rows,
                     int out_row0, int out_rows, const double *Q, const double *alpha, int N,
                     int T, const int *Y, int r, const double *w, double *P, double *Z,
                     double *Pim, double *Zim) {
    int rc = check_slab(H, slab_row0, slab_rows, out_row0, out_rows, r);
    if (rc) return rc;
    const long S = (long)slab_rows * W;   /* slab pixels */
    const long O = (long)out_rows * W;    /* output pixels */
    const int nplanes = 1 + d;            /* H and the d components of G */

    /* L212-214: gamma_k = alpha_k / sqrt(N) */
    double *gamma = (double *)malloc(sizeof(double) * d);
    for (int k = 0; k < d; ++k) gamma[k] = alpha[k] / sqrt((double)N);

    double *g = (double *)malloc(sizeof(double) * d * S);         /* g = Q^T f */
    double *Hre = (double *)malloc(sizeof(double) * S);
    double *Him = (double *)malloc(sizeof(double) * S);
    double *Gre = (double *)malloc(sizeof(double) * d * S);
    double *Gim = (double *)malloc(sizeof(double) * d * S);
    /* horizontal-pass output (slab rows) and full 2-D convolution (output rows)
     * for the 2*(1+d) real planes: plane p = 0 is H, p = 1+c is G_c */
    double *hre = (double *)malloc(sizeof(double) * nplanes * S);
    double *him = (double *)malloc(sizeof(double) * nplanes * S);
    double *bre = (double *)malloc(sizeof(double) * nplanes * O);
    double *bim = (double *)malloc(sizeof(double) * nplanes * O);
    if (!gamma || !g || !Hre || !Him || !Gre || !Gim || !hre || !him || !bre || !bim) {
        free(gamma); free(g); free(Hre); free(Him); free(Gre); free(Gim);
        free(hre); free(him); free(bre); free(bim);
        return -3;
    }

    /* L215-219: g(i) = Q^T f(i); P(i) = 0; Z(i) = 0 */
#pragma omp parallel for schedule(static)
    for (long i = 0; i < S; ++i)
        for (int k = 0; k < d; ++k) {
            double s = 0.0;
            for (int c = 0; c < d; ++c) s += Q[c * d + k] * (double)f[(long)c * S + i];
            g[(long)k * S + i] = s;
        }
    for (long i = 0; i < (long)d * O; ++i) { P[i] = 0.0; if (Pim) Pim[i] = 0.0; }
    for (long i = 0; i < O; ++i) { Z[i] = 0.0; if (Zim) Zim[i] = 0.0; }

    for (int t = 0; t < T; ++t) {                                   /* L220 */
        const int *Yt = Y + (long)t * d;                            /* L221 (draws passed in) */
        /* L222-225: H(i) = prod_k exp(iota (N - 2 X_k) gamma_k g_k(i)) */
#pragma omp parallel for schedule(static)
        for (long i = 0; i < S; ++i) {
            double hr = 1.0, hi = 0.0;
            for (int k = 0; k < d; ++k) {
                double a = (double)Yt[k] * gamma[k] * g[(long)k * S + i];
                double er = cos(a), ei = sin(a);
                double nr = hr * er - hi * ei, ni = hr * ei + hi * er;
                hr = nr; hi = ni;
            }
            Hre[i] = hr; Him[i] = hi;
            /* L226: G(i) = H(i) f(i) */
            for (int c = 0; c < d; ++c) {
                double fc = (double)f[(long)c * S + i];
                Gre[(long)c * S + i] = hr * fc;
                Gim[(long)c * S + i] = hi * fc;
            }
        }
        /* L227: Gbar = w * G, Hbar = w * H. Separable: omega(j) = w(j_y) w(j_x).
         * Horizontal pass: A(y,x) = sum_m w(m) X(y, rho(x - m)) on every slab row. */
#pragma omp parallel for schedule(static)
        for (long yy = 0; yy < slab_rows; ++yy)
            for (int p = 0; p < nplanes; ++p) {
                const double *xr = (p == 0 ? Hre : Gre + (long)(p - 1) * S) + yy * W;
                const double *xi = (p == 0 ? Him : Gim + (long)(p - 1) * S) + yy * W;
                double *ar = hre + (long)p * S + yy * W;
                double *ai = him + (long)p * S + yy * W;
                for (long x = 0; x < W; ++x) {
                    double sr = 0.0, si = 0.0;
                    for (long m = -r; m <= r; ++m) {
                        long xx = refl(x - m, W);
                        sr += w[m + r] * xr[xx];
                        si += w[m + r] * xi[xx];
                    }
                    ar[x] = sr; ai[x] = si;
                }
            }
        /* Vertical pass on the output rows: B(y,x) = sum_m w(m) A(rho(y - m), x). */
#pragma omp parallel for schedule(static)
        for (long oy = 0; oy < out_rows; ++oy)
            for (int p = 0; p < nplanes; ++p) {
                double *br = bre + (long)p * O + oy * W;
                double *bi = bim + (long)p * O + oy * W;
                for (long x = 0; x < W; ++x) { br[x] = 0.0; bi[x] = 0.0; }
                for (long m = -r; m <= r; ++m) {
                    long sy = refl(out_row0 + oy - m, H) - slab_row0;
                    const double *ar = hre + (long)p * S + sy * W;
                    const double *ai = him + (long)p * S + sy * W;
                    for (long x = 0; x < W; ++x) { br[x] += w[m + r] * ar[x]; bi[x] += w[m + r] * ai[x]; }
                }
            }
        /* L228-229: P += conj(H) Gbar ; Z += conj(H) Hbar */
#pragma omp parallel for schedule(static)
        for (long oi = 0; oi < O; ++oi) {
            long si = (long)(out_row0 - slab_row0) * W + oi;   /* same pixel in the slab */
            double hr = Hre[si], hi = Him[si];
            double zr = bre[oi], zi = bim[oi];
            Z[oi] += hr * zr + hi * zi;
            if (Zim) Zim[oi] += hr * zi - hi * zr;
            for (int c = 0; c < d; ++c) {
                double gr = bre[(long)(1 + c) * O + oi], gi = bim[(long)(1 + c) * O + oi];
                P[(long)c * O + oi] += hr * gr + hi * gi;
                if (Pim) Pim[(long)c * O + oi] += hr * gi - hi * gr;
            }
        }
    }
    free(gamma); free(g); free(Hre); free(Him); free(Gre); free(Gim);
    free(hre); free(him); free(bre); free(bim);
    return 0;
}

/*
 * Exact bilateral filter, Eq. (2)-(3), window [-r, r]^2
 * (PAPER.md:46), phi(x) = exp(-x^T C^{-1} x / 2) (Eq. (1)),
 * omega(j) = w(j_y) w(j_x) (normalised taps; the scale cancels, reading R3).
 *   Cinv  d x d row-major inverse covariance
 *   out   (d, out_rows, W)
 */
int oracle_direct(int H, int W, int d, const float *f, int slab_row0, int slab_rows,
                  int out_row0, int out_rows, const double *Cinv, int r, const double *w,
                  double *out) {
    int rc = check_slab(H, slab_row0, slab_rows, out_row0, out_rows, r);
    if (rc) return rc;
    const long S = (long)slab_rows * W;
    const long O = (long)out_rows * W;
#pragma omp parallel for schedule(dynamic, 1)
    for (long oy = 0; oy < out_rows; ++oy) {
        double fi[16], x[16], num[16];
        long y = out_row0 + oy;
        for (long xi = 0; xi < W; ++xi) {
            for (int c = 0; c < d; ++c) fi[c] = (double)f[(long)c * S + (y - slab_row0) * W + xi];
            double den = 0.0;
            for (int c = 0; c < d; ++c) num[c] = 0.0;
            for (long jy = -r; jy <= r; ++jy) {
                long sy = refl(y - jy, H) - slab_row0;
                for (long jx = -r; jx <= r; ++jx) {
                    long sx = refl(xi - jx, W);
                    double fj[16];
                    for (int c = 0; c < d; ++c) {
                        fj[c] = (double)f[(long)c * S + sy * W + sx];
                        x[c] = fj[c] - fi[c];
                    }
                    double q = 0.0;
                    for (int a = 0; a < d; ++a)
                        for (int b = 0; b < d; ++b) q += x[a] * Cinv[a * d + b] * x[b];
                    double wt = w[jy + r] * w[jx + r] * exp(-0.5 * q);
                    den += wt;
                    for (int c = 0; c < d; ++c) num[c] += wt * fj[c];
                }
            }
            for (int c = 0; c < d; ++c) out[(long)c * O + oy * W + xi] = num[c] / den;
        }
    }
    return 0;
}

int oracle_version(void) { return 1; }
