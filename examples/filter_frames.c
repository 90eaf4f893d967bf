/*
 * filter_frames.c -- a stream of host frames through bf_vec_filter_host_async: each frame's input
 * copy and the previous frame's output copy overlap the current frame's kernels (two plan-owned
 * copy streams, alternating device slots); one bf_vec_host_sync at the end. The caller keeps every
 * frame's buffers alive until then. Frames are plain malloc memory here (the copies are then
 * staged by the driver); pinned memory (cudaHostAlloc) makes them truly asynchronous. Checks that
 * every frame equals the synchronous bf_vec_filter_host result bit for bit. No CUDA headers needed.
 *
 *   gcc -O2 -I include examples/filter_frames.c -L paper_1605_02164_b200 -lbfvec \
 *       -Wl,-rpath,$PWD/paper_1605_02164_b200 -lm -o filter_frames && ./filter_frames
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "bfvec.h"

int main(void) {
    enum { FRAMES = 6 };
    const int H = 256, W = 320, d = 3, N = 20, M = 64;
    const size_t n = (size_t)d * H * W;
    const double C[9] = {40.0 * 40.0, 0, 0, 0, 40.0 * 40.0, 0, 0, 0, 40.0 * 40.0};
    float *in[FRAMES], *out[FRAMES], *ref = malloc(sizeof(float) * n);
    for (int k = 0; k < FRAMES; ++k) {   /* a moving ripple over flat quadrants */
        in[k] = malloc(sizeof(float) * n);
        out[k] = malloc(sizeof(float) * n);
        for (int c = 0; c < d; ++c)
            for (int y = 0; y < H; ++y)
                for (int x = 0; x < W; ++x)
                    in[k][(c * H + y) * W + x] = (float)(60.0 * (c + 1) * ((y < H / 2) + (x < W / 2)) +
                                                         10.0 * sin(0.3 * x + 0.5 * k + c));
    }
    bf_vec_plan_t plan;
    bf_status_t st = bf_vec_plan(H, W, d, 3.0, C, N, M, 7, &plan);
    if (st >= 0) st = bf_vec_sample_freqs(plan, NULL);
    for (int k = 0; k < FRAMES && st >= 0; ++k) st = bf_vec_filter_host_async(plan, in[k], out[k], NULL);
    if (st >= 0) st = bf_vec_host_sync(plan);
    if (st < 0) { fprintf(stderr, "frames: %s\n", bf_vec_status_string(st)); return 1; }
    int same = 1;
    for (int k = 0; k < FRAMES; ++k) {
        if (bf_vec_filter_host(plan, in[k], ref, NULL) < 0) return 1;
        same &= memcmp(ref, out[k], sizeof(float) * n) == 0;
    }
    printf("%d frames %dx%dx%d through bf_vec_filter_host_async: %s the synchronous results\n", FRAMES, H, W, d,
           same ? "bitwise equal to" : "DIFFERENT from");
    bf_vec_plan_destroy(plan);
    for (int k = 0; k < FRAMES; ++k) { free(in[k]); free(out[k]); }
    free(ref);
    return same ? 0 : 1;
}
