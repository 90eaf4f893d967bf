/*
 * filter_host.c -- minimal C user of libbfvec.so: filter a synthetic colour image held in HOST
 * memory with the Monte Carlo shiftable filter (bf_vec_filter_host copies it in and out), compare
 * with the exact bilateral filter is left to the Python tools. No CUDA headers needed.
 *
 *   gcc -O2 -I include examples/filter_host.c -L paper_1605_02164_b200 -lbfvec \
 *       -Wl,-rpath,$PWD/paper_1605_02164_b200 -o filter_host && ./filter_host
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "bfvec.h"

int main(void) {
    const int H = 256, W = 320, d = 3, N = 20, M = 64;
    const double sigma_s = 3.0;
    const double C[9] = {40.0 * 40.0, 0, 0, 0, 40.0 * 40.0, 0, 0, 0, 40.0 * 40.0};   /* sigma_r = 40 */
    float *f = malloc(sizeof(float) * d * H * W), *out = malloc(sizeof(float) * d * H * W);
    for (int c = 0; c < d; ++c)                      /* four flat quadrants + a ripple */
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x)
                f[(c * H + y) * W + x] = (float)(60.0 * (c + 1) * ((y < H / 2) + (x < W / 2)) +
                                                 10.0 * sin(0.3 * x + c));
    bf_vec_plan_t plan;
    bf_status_t st = bf_vec_plan(H, W, d, sigma_s, C, N, M, 42, &plan);
    if (st < 0) { fprintf(stderr, "plan: %s\n", bf_vec_status_string(st)); return 1; }
    st = bf_vec_sample_freqs(plan, NULL);
    if (st >= 0) st = bf_vec_filter_host(plan, f, out, NULL);
    if (st < 0) { fprintf(stderr, "filter: %s\n", bf_vec_status_string(st)); bf_vec_plan_destroy(plan); return 1; }
    float zmin; long long nsmall;
    bf_vec_diag(plan, &zmin, &nsmall);
    double mean_abs = 0.0;
    for (long i = 0; i < (long)d * H * W; ++i) mean_abs += fabs(out[i] - f[i]);
    printf("filtered %dx%dx%d, M=%d: mean |S - f| = %.3f, min Z/M = %.3f, %lld small-Z pixels\n", H, W, d, M,
           mean_abs / ((double)d * H * W), zmin, nsmall);
    bf_vec_plan_destroy(plan);
    free(f);
    free(out);
    return 0;
}
