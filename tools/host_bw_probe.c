// Host write bandwidth probe: expand a sparse frame (bitmask + packed 5-float
// pixels) into 3 fp32 planes with T threads, pre-faulted destination.
//   gcc -O3 -march=native -pthread tools/host_bw_probe.c -o /tmp/host_bw && /tmp/host_bw <hit_frac>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#define W 1920
#define H 1080
#define NPIX (W * H)
static float *rgb, *alp, *dep, *packed;
static uint32_t *mask, *prefix;
static int T;
static void *work(void *arg) {
    const long id = (long)arg;
    const long words = NPIX / 32, per = (words + T - 1) / T, w0 = id * per, w1 = w0 + per < words ? w0 + per : words;
    for (long w = w0; w < w1; ++w) {
        uint32_t m = mask[w];
        const float *src = packed + 5L * prefix[w];
        for (int b = 0; b < 32; ++b) {
            const long p = w * 32 + b;
            if (m >> b & 1) {
                rgb[3 * p] = src[0]; rgb[3 * p + 1] = src[1]; rgb[3 * p + 2] = src[2];
                alp[p] = src[3]; dep[p] = src[4]; src += 5;
            } else {
                rgb[3 * p] = 0; rgb[3 * p + 1] = 0; rgb[3 * p + 2] = 0; alp[p] = 0; dep[p] = 0;
            }
        }
    }
    return 0;
}
static double now() { struct timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec + 1e-9 * t.tv_nsec; }
int main(int argc, char **argv) {
    double hit = argc > 1 ? atof(argv[1]) : 0.33;
    rgb = malloc(12L * NPIX); alp = malloc(4L * NPIX); dep = malloc(4L * NPIX);
    packed = malloc(20L * NPIX); mask = malloc(NPIX / 8); prefix = malloc(NPIX / 8);
    memset(rgb, 1, 12L * NPIX); memset(alp, 1, 4L * NPIX); memset(dep, 1, 4L * NPIX); memset(packed, 1, 20L * NPIX);
    uint32_t c = 0;  // a central disc of hits, like a performer
    for (long w = 0; w < NPIX / 32; ++w) {
        uint32_t m = 0;
        for (int b = 0; b < 32; ++b) {
            long p = w * 32 + b; double x = (double)(p % W) / W - 0.5, y = (double)(p / W) / H - 0.5;
            if (x * x + y * y < hit / 3.14159) m |= 1u << b;
        }
        mask[w] = m; prefix[w] = c; c += __builtin_popcount(m);
    }
    printf("hit fraction %.3f, memcpy 41.5MB 1 thread: ", (double)c / NPIX);
    double t0 = now(); for (int i = 0; i < 10; ++i) memcpy(packed, rgb, 12L * NPIX); printf("%.1f GB/s\n", 10 * 12.0 * NPIX / (now() - t0) / 1e9);
    for (T = 1; T <= 32; T *= 2) {
        pthread_t th[64];
        double best = 1e9;
        for (int it = 0; it < 8; ++it) {
            double a = now();
            for (long i = 0; i < T; ++i) pthread_create(&th[i], 0, work, (void *)i);
            for (int i = 0; i < T; ++i) pthread_join(th[i], 0);
            double d = now() - a; if (d < best) best = d;
        }
        printf("threads %2d: expand %.3f ms (%.1f GB/s written)\n", T, best * 1e3, 20.0 * NPIX / best / 1e9);
    }
    return 0;
}
