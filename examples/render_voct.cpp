// render_voct.cpp -- the C ABI from a non-Python host: a .voct file straight
// to the GPU (vv_voct_upload), one frame through the fused camera kernel
// (vv_render_camera), rgb/alpha/depth back to the host, a binary PPM out.
//
//   render_voct <tree.voct> <frame> <width> <height> <out.ppm> [<out.f32>]
//
// The camera is look_at((1.6, 1.3, 0.9) -> bbox centre), focal 1.08 * max(W, H)
// (the benchmark camera of SURVEY.md 8(d)); <out.f32> receives the raw
// (H, W, 5) float32 [r, g, b, alpha, depth] planes for comparisons.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "voxvid_b200.h"

static int die(const char *what, int rc) {
    std::fprintf(stderr, "%s failed (%d): %s\n", what, rc, vv_last_error());
    return 1;
}

static void cross(const double *a, const double *b, double *c) {
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}
static void normalize(double *v) {
    const double n = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    for (int i = 0; i < 3; ++i) v[i] /= n;
}

int main(int argc, char **argv) {
    if (argc < 6) {
        std::fprintf(stderr, "usage: %s tree.voct frame width height out.ppm [out.f32]\n", argv[0]);
        return 2;
    }
    const int frame = std::atoi(argv[2]), W = std::atoi(argv[3]), H = std::atoi(argv[4]);
    FILE *f = std::fopen(argv[1], "rb");
    if (!f) return std::perror(argv[1]), 1;
    std::fseek(f, 0, SEEK_END);
    const long len = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    std::vector<unsigned char> buf((size_t)len);
    if (std::fread(buf.data(), 1, buf.size(), f) != buf.size()) return std::perror("read"), 1;
    std::fclose(f);

    vv_tree *tree = nullptr;
    vv_voct_info info;
    int rc = vv_voct_upload(buf.data(), buf.size(), 0, &tree, &info);
    if (rc) return die("vv_voct_upload", rc);
    std::printf("tree: depth %d, %lld leaves, %d frames, n_max %d\n", info.depth, (long long)info.n_leaves,
                info.frames, info.n_max);

    // Camera.look_at (render.py:97-125): rows of R are right, down, forward
    const double eye[3] = {1.6, 1.3, 0.9};
    const double tgt[3] = {info.bbox_lo[0] + 0.5 * info.side, info.bbox_lo[1] + 0.5 * info.side,
                           info.bbox_lo[2] + 0.5 * info.side};
    double fwd[3] = {tgt[0] - eye[0], tgt[1] - eye[1], tgt[2] - eye[2]}, up[3] = {0, 0, 1}, right[3], down[3];
    normalize(fwd);
    cross(fwd, up, right);
    normalize(right);
    cross(fwd, right, down);
    vv_camera cam;
    cam.width = W;
    cam.height = H;
    cam.fx = cam.fy = 1.08 * (W > H ? W : H);
    cam.cx = 0.5 * W;
    cam.cy = 0.5 * H;
    const double c2w[16] = {right[0], down[0], fwd[0], eye[0], right[1], down[1], fwd[1], eye[1],
                            right[2], down[2], fwd[2], eye[2], 0, 0, 0, 1};
    for (int i = 0; i < 16; ++i) cam.c2w[i] = c2w[i];

    const size_t npix = (size_t)W * H;
    float *d = nullptr;
    if (cudaMalloc(&d, 5 * npix * sizeof(float)) != cudaSuccess) return die("cudaMalloc", -1);
    rc = vv_render_camera(tree, frame, nullptr, nullptr, &cam, d, d + 3 * npix, d + 4 * npix, nullptr);
    if (rc) return die("vv_render_camera", rc);
    std::vector<float> h(5 * npix);
    if (cudaMemcpy(h.data(), d, h.size() * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess)
        return die("cudaMemcpy", -1);

    FILE *o = std::fopen(argv[5], "wb");
    if (!o) return std::perror(argv[5]), 1;
    std::fprintf(o, "P6\n%d %d\n255\n", W, H);
    for (size_t p = 0; p < npix; ++p)
        for (int c = 0; c < 3; ++c) {  // composite over black, gamma-free 8-bit
            const float v = h[3 * p + c] * h[3 * npix + p];
            std::fputc((int)std::lround(255.0f * (v < 0 ? 0 : v > 1 ? 1 : v)), o);
        }
    std::fclose(o);
    if (argc > 6) {  // raw planes (H, W, 5) for comparisons
        FILE *r = std::fopen(argv[6], "wb");
        std::vector<float> il(5 * npix);
        for (size_t p = 0; p < npix; ++p) {
            for (int c = 0; c < 3; ++c) il[5 * p + c] = h[3 * p + c];
            il[5 * p + 3] = h[3 * npix + p];
            il[5 * p + 4] = h[4 * npix + p];
        }
        std::fwrite(il.data(), sizeof(float), il.size(), r);
        std::fclose(r);
    }
    double cover = 0;
    for (size_t p = 0; p < npix; ++p) cover += h[3 * npix + p] > 0.5f;
    std::printf("frame %d: %dx%d, %.1f%% of pixels opaque -> %s\n", frame, W, H, 100.0 * cover / npix, argv[5]);
    cudaFree(d);
    vv_tree_free(tree);
    return 0;
}
