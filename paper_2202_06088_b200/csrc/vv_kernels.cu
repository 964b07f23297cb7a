// vv_kernels.cu -- sm_100a kernels and the device half of the C ABI
// (include/voxvid_b200.h).
//
// Kernels (all one-thread-per-ray/pixel, shared-memory traversal stacks):
//   k_render_rays    render_kernel (kernels.py:410-652) over explicit rays
//   k_render_camera  Camera.rays + render_kernel + finalize_layer, fused
//                    (render.py:74-83, 218-240); also the tile-sharded form
//   k_render_scene   render_instance x L + Algorithm 1 + background
//                    (compose.py:373-475, render.py:243-251), fused per pixel
//   k_build_slice    build_slice_kernel (kernels.py:397-407)
//   k_count / k_collect  count/collect_segments_kernel (kernels.py:313-367)
//   k_repack         payload rows -> padded [w_sigma] / [w_gamma | w_hh] planes
#include <cuda_runtime.h>
#include <math.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "../../include/voxvid_b200.h"
#include "vv_device.cuh"
#include "vv_host_common.h"

using namespace vv;

struct vv_tree {
    int device;
    TreeView view;
    int64_t n_leaves, n_internal;
    int32_t frames, C, K, S, n_max, depth;
    bool has_edits;
    int64_t bytes;
    // owned device allocations
    int32_t *d_child;
    float4 *d_sig, *d_rest, *d_edit_rgb;
    int2 *d_edit_t;
    float *d_a, *d_b;
};

struct vv_slice {
    const vv_tree *tree;
    int device;
    int32_t frame;
    double *d_sigma;
    float4 *d_q;
    int q4;
    int64_t n_leaves;
};

#define VV_CUDA(call)                                                                          \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess)                                                                 \
            return set_error(VV_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));      \
    } while (0)

namespace {

constexpr int kBlock = 128;
constexpr int kMaxInst = 16;

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

Consts make_consts(int n_max) {
    HostTables t;
    build_tables(n_max, t);
    Consts c;
    memset(&c, 0, sizeof(c));
    for (int i = 0; i < t.n_pairs && i < 16; ++i) c.pair_norm[i] = (float)t.pair_norm[i];
    for (int i = 0; i < t.s && i < 16; ++i) c.sh_pref[i] = (float)t.sh_pref[i];
    return c;
}

CamView make_cam(const vv_camera &c) {
    CamView v;
    v.width = c.width;
    v.height = c.height;
    v.fx = c.fx;
    v.fy = c.fy;
    v.cx = c.cx;
    v.cy = c.cy;
    v.r00 = c.c2w[0]; v.r01 = c.c2w[1]; v.r02 = c.c2w[2];
    v.r10 = c.c2w[4]; v.r11 = c.c2w[5]; v.r12 = c.c2w[6];
    v.r20 = c.c2w[8]; v.r21 = c.c2w[9]; v.r22 = c.c2w[10];
    v.ox = c.c2w[3];
    v.oy = c.c2w[7];
    v.oz = c.c2w[11];
    return v;
}

// cooperative load of the frame's A/B rows (kernels read them for every leaf)
__device__ __forceinline__ void load_rows(const TreeView &T, int frame, float *sA, float *sB) {
    for (int c = threadIdx.x; c < kMaxC; c += blockDim.x) {
        const bool in = c < T.C;
        sA[c] = in ? T.basis_a[(size_t)frame * T.C + c] : 0.0f;
        sB[c] = in ? T.basis_b[(size_t)frame * T.C + c] : 0.0f;
    }
}

// ------------------------------------------------------------------ rays
struct RaysParams {
    TreeView T;
    SliceView S;
    Consts K;
    int frame;
    double early_stop, edit_weight, tmin, tmax;
    const double *origins, *dirs;
    int64_t n;
    double *premult, *alpha, *tbar;
    int32_t *used, *pops, *shaded;
    const int64_t *visit_start;
    int64_t *visit_leaf;
};

template <int NMAX, bool CACHED, bool EDITS, class Entry, bool VISITS>
__global__ void __launch_bounds__(kBlock) k_render_rays(const __grid_constant__ RaysParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ float sA[kMaxC], sB[kMaxC];
    load_rows(p.T, p.frame, sA, sB);
    __syncthreads();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= p.n) return;
    Entry *stk = reinterpret_cast<Entry *>(smem_raw) + threadIdx.x;
    const double ox = p.origins[3 * r], oy = p.origins[3 * r + 1], oz = p.origins[3 * r + 2];
    const double dx = p.dirs[3 * r], dy = p.dirs[3 * r + 1], dz = p.dirs[3 * r + 2];
    FrameCtx F{sA, sB, p.frame, p.early_stop, p.edit_weight};
    Shader<NMAX, CACHED, EDITS, VISITS> sh(p.T, p.S, F, p.K, (float)dx, (float)dy, (float)dz);
    if (VISITS) sh.visit = p.visit_leaf + p.visit_start[r];
    Ray ray;
    if (ray_setup(p.T, ox, oy, oz, dx, dy, dz, p.tmin, p.tmax, ray))
        traverse<Entry>(p.T.child, p.T.depth, ray, stk, blockDim.x, sh);
    if (VISITS) return;
    p.premult[3 * r + 0] = sh.acc0;
    p.premult[3 * r + 1] = sh.acc1;
    p.premult[3 * r + 2] = sh.acc2;
    p.alpha[r] = sh.aacc;
    p.tbar[r] = sh.tacc;
    if (p.used) p.used[r] = sh.used;
    if (p.pops) p.pops[r] = sh.pops;
    if (p.shaded) p.shaded[r] = sh.shaded;
}

// ------------------------------------------------------------------ camera
struct CamParams {
    TreeView T;
    SliceView S;
    Consts K;
    CamView cam;
    int frame;
    double early_stop, edit_weight, tmin, tmax, far_plane, alpha_floor;
    float *rgb, *alpha, *depth;
    // tile mode (packed != null)
    float *packed;
    int tile, shard, n_shards, tiles_x;
};

// block = 16x8 pixels; warp = 16x2 pixels (spatially coherent rays)
__device__ __forceinline__ void block_pixel(int bx, int by, int &ix, int &iy) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    ix = bx * 16 + (lane & 15);
    iy = by * 8 + w * 2 + (lane >> 4);
}

template <int NMAX, bool CACHED, bool EDITS, class Entry>
__global__ void __launch_bounds__(kBlock) k_render_camera(const __grid_constant__ CamParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ float sA[kMaxC], sB[kMaxC];
    load_rows(p.T, p.frame, sA, sB);
    __syncthreads();
    int ix, iy;
    int64_t slot = -1;  // tile mode: packed output slot
    if (p.packed) {
        const int sub_per_tile = (p.tile / 16) * (p.tile / 8);
        const int my_tile = blockIdx.x / sub_per_tile;
        const int sub = blockIdx.x % sub_per_tile;
        const int tile_id = my_tile * p.n_shards + p.shard;
        const int tx0 = (tile_id % p.tiles_x) * p.tile, ty0 = (tile_id / p.tiles_x) * p.tile;
        int lx, ly;
        block_pixel(sub % (p.tile / 16), sub / (p.tile / 16), lx, ly);
        ix = tx0 + lx;
        iy = ty0 + ly;
        slot = (int64_t)my_tile * p.tile * p.tile + (int64_t)ly * p.tile + lx;
    } else {
        block_pixel(blockIdx.x, blockIdx.y, ix, iy);
    }
    const bool inside = ix < p.cam.width && iy < p.cam.height;
    float r = 0.f, g = 0.f, b = 0.f, a = 0.f, d = (float)p.far_plane;
    if (inside) {
        double dx, dy, dz;
        camera_ray(p.cam, ix, iy, dx, dy, dz);
        Entry *stk = reinterpret_cast<Entry *>(smem_raw) + threadIdx.x;
        FrameCtx F{sA, sB, p.frame, p.early_stop, p.edit_weight};
        Shader<NMAX, CACHED, EDITS, false> sh(p.T, p.S, F, p.K, (float)dx, (float)dy, (float)dz);
        Ray ray;
        if (ray_setup(p.T, p.cam.ox, p.cam.oy, p.cam.oz, dx, dy, dz, p.tmin, p.tmax, ray))
            traverse<Entry>(p.T.child, p.T.depth, ray, stk, blockDim.x, sh);
        finalize(sh.acc0, sh.acc1, sh.acc2, sh.aacc, sh.tacc, 1.0, false, p.alpha_floor, p.far_plane,
                 r, g, b, a, d);
    }
    if (p.packed) {
        float *o = p.packed + slot * 5;
        o[0] = r; o[1] = g; o[2] = b; o[3] = a; o[4] = d;
        return;
    }
    if (!inside) return;
    const int64_t pix = (int64_t)iy * p.cam.width + ix;
    if (p.rgb) {
        p.rgb[3 * pix + 0] = r;
        p.rgb[3 * pix + 1] = g;
        p.rgb[3 * pix + 2] = b;
    }
    if (p.alpha) p.alpha[pix] = a;
    if (p.depth) p.depth[pix] = d;
}

__global__ void k_unpack_tiles(const float *__restrict__ packed, int width, int height, int tile,
                               int n_shards, int tiles_x, int tiles_total, float *rgb, float *alpha,
                               float *depth) {
    const int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pix >= (int64_t)width * height) return;
    const int ix = (int)(pix % width), iy = (int)(pix / width);
    const int tid = (iy / tile) * tiles_x + (ix / tile);
    const int shard = tid % n_shards, k = tid / n_shards;
    const int per_shard = (tiles_total + n_shards - 1) / n_shards;
    const int64_t slot = ((int64_t)shard * per_shard + k) * tile * tile + (int64_t)(iy % tile) * tile + (ix % tile);
    const float *s = packed + slot * 5;
    if (rgb) {
        rgb[3 * pix + 0] = s[0];
        rgb[3 * pix + 1] = s[1];
        rgb[3 * pix + 2] = s[2];
    }
    if (alpha) alpha[pix] = s[3];
    if (depth) depth[pix] = s[4];
}

// ------------------------------------------------------------------ scene
struct InstView {
    TreeView T;
    CamView cam;      // mode 0: pulled-back pose
    double inv[12];   // mode 1: rows of inv(affine)[:3, :4]
    int frame, mode;
};

struct SceneParams {
    Consts K;
    CamView cam;
    InstView inst[kMaxInst];
    int n_inst;
    double early_stop, edit_weight, tmin, tmax, far_plane, alpha_floor;
    double bg0, bg1, bg2;
    float *image, *alpha, *depth;
};

template <int NMAX, class Entry>
__global__ void __launch_bounds__(kBlock) k_render_scene(const __grid_constant__ SceneParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ float sA[kMaxInst][kMaxC], sB[kMaxInst][kMaxC];
    for (int i = 0; i < p.n_inst; ++i) load_rows(p.inst[i].T, p.inst[i].frame, sA[i], sB[i]);
    __syncthreads();
    int ix, iy;
    block_pixel(blockIdx.x, blockIdx.y, ix, iy);
    if (ix >= p.cam.width || iy >= p.cam.height) return;
    Entry *stk = reinterpret_cast<Entry *>(smem_raw) + threadIdx.x;
    double cdx, cdy, cdz;
    camera_ray(p.cam, ix, iy, cdx, cdy, cdz);
    // blended state (compose.py:386-405): I (3), D, A
    double I0 = 0, I1 = 0, I2 = 0, D = 0, A = 0;
    for (int i = 0; i < p.n_inst; ++i) {
        const InstView &v = p.inst[i];
        double ox, oy, oz, dx, dy, dz, scale = 1.0;
        bool scaled = false;
        if (v.mode == 0) {
            camera_ray(v.cam, ix, iy, dx, dy, dz);
            ox = v.cam.ox;
            oy = v.cam.oy;
            oz = v.cam.oz;
        } else {
            // o_t = o @ inv3^T + t ; d_raw = d @ inv3^T ; d_t = d_raw/|d_raw|
            const double *m = v.inv;
            ox = xadd(xadd(xadd(xmul(p.cam.ox, m[0]), xmul(p.cam.oy, m[1])), xmul(p.cam.oz, m[2])), m[3]);
            oy = xadd(xadd(xadd(xmul(p.cam.ox, m[4]), xmul(p.cam.oy, m[5])), xmul(p.cam.oz, m[6])), m[7]);
            oz = xadd(xadd(xadd(xmul(p.cam.ox, m[8]), xmul(p.cam.oy, m[9])), xmul(p.cam.oz, m[10])), m[11]);
            const double r0 = xadd(xadd(xmul(cdx, m[0]), xmul(cdy, m[1])), xmul(cdz, m[2]));
            const double r1 = xadd(xadd(xmul(cdx, m[4]), xmul(cdy, m[5])), xmul(cdz, m[6]));
            const double r2 = xadd(xadd(xmul(cdx, m[8]), xmul(cdy, m[9])), xmul(cdz, m[10]));
            const double nrm = sqrt(xadd(xadd(xmul(r0, r0), xmul(r1, r1)), xmul(r2, r2)));
            dx = xdiv(r0, nrm);
            dy = xdiv(r1, nrm);
            dz = xdiv(r2, nrm);
            scale = xdiv(1.0, nrm);
            scaled = true;
        }
        FrameCtx F{sA[i], sB[i], v.frame, p.early_stop, p.edit_weight};
        SliceView S{nullptr, nullptr, 0};
        Shader<NMAX, false, true, false> sh(v.T, S, F, p.K, (float)dx, (float)dy, (float)dz);
        Ray ray;
        if (ray_setup(v.T, ox, oy, oz, dx, dy, dz, p.tmin, p.tmax, ray))
            traverse<Entry>(v.T.child, v.T.depth, ray, stk, blockDim.x, sh);
        // finalize_layer in float64
        const double al = sh.aacc;
        const double safe = al > 1e-300 ? al : 1e-300;
        double li0 = 0, li1 = 0, li2 = 0;
        if (al > 0.0) {
            li0 = xdiv(sh.acc0, safe);
            li1 = xdiv(sh.acc1, safe);
            li2 = xdiv(sh.acc2, safe);
        }
        double t = xdiv(sh.tacc, safe);
        if (scaled) t = xmul(t, scale);
        const double ld = al >= p.alpha_floor ? t : p.far_plane;
        if (i == 0) {
            I0 = li0; I1 = li1; I2 = li2; D = ld; A = al;
        } else {
            // Algorithm 1 (compose.py:393-404); ties go to the incoming layer
            const double om_ai = xsub(1.0, al), om_a = xsub(1.0, A);
            if (ld <= D) {
                I0 = xadd(xmul(al, li0), xmul(xmul(om_ai, A), I0));
                I1 = xadd(xmul(al, li1), xmul(xmul(om_ai, A), I1));
                I2 = xadd(xmul(al, li2), xmul(xmul(om_ai, A), I2));
                D = ld;
            } else {
                I0 = xadd(xmul(A, I0), xmul(xmul(om_a, al), li0));
                I1 = xadd(xmul(A, I1), xmul(xmul(om_a, al), li1));
                I2 = xadd(xmul(A, I2), xmul(xmul(om_a, al), li2));
            }
            A = xadd(A, xmul(al, om_a));
        }
    }
    if (p.n_inst > 1) {  // unpremultiply the blend (compose.py:457-460)
        const double safe = A > 1e-300 ? A : 1e-300;
        if (A > 0.0) {
            I0 = xdiv(I0, safe);
            I1 = xdiv(I1, safe);
            I2 = xdiv(I2, safe);
        } else {
            I0 = I1 = I2 = 0.0;
        }
    }
    // composite_background: a * rgb + (1 - a) * bg (render.py:243-251)
    const double om = xsub(1.0, A);
    const int64_t pix = (int64_t)iy * p.cam.width + ix;
    p.image[3 * pix + 0] = (float)xadd(xmul(A, I0), xmul(om, p.bg0));
    p.image[3 * pix + 1] = (float)xadd(xmul(A, I1), xmul(om, p.bg1));
    p.image[3 * pix + 2] = (float)xadd(xmul(A, I2), xmul(om, p.bg2));
    if (p.alpha) p.alpha[pix] = (float)A;
    if (p.depth) p.depth[pix] = (float)D;
}

// ------------------------------------------------------------------ slice
struct SliceParams {
    TreeView T;
    Consts K;
    int frame;
    int64_t n_leaves;
    double *sigma;
    float4 *q;
    int q4;
};

template <int NMAX>
__global__ void __launch_bounds__(256) k_build_slice(const __grid_constant__ SliceParams p) {
    __shared__ float sA[kMaxC], sB[kMaxC];
    load_rows(p.T, p.frame, sA, sB);
    __syncthreads();
    const int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (L >= p.n_leaves) return;
    constexpr int Q4 = Basis<NMAX>::Q4;
    float q[4 * Q4];
#pragma unroll
    for (int i = 0; i < 4 * Q4; ++i) q[i] = 0.0f;
    double sigma;
    slice_leaf<NMAX>(p.T, (uint32_t)L, sA, sB, p.K, sigma, q);
    p.sigma[L] = sigma;
    float4 *o = p.q + L * p.q4;
#pragma unroll
    for (int i = 0; i < Q4; ++i) o[i] = make_float4(q[4 * i], q[4 * i + 1], q[4 * i + 2], q[4 * i + 3]);
}

// ------------------------------------------------------------------ traversal only
struct SegParams {
    TreeView T;
    const double *origins, *dirs;
    int64_t n;
    double tmin, tmax;
    int64_t *count;
    const int64_t *ray_start;
    int64_t *seg_leaf;
    double *seg_t0, *seg_t1;
};

template <class Entry, bool COLLECT>
__global__ void __launch_bounds__(kBlock) k_segments(const __grid_constant__ SegParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= p.n) return;
    Entry *stk = reinterpret_cast<Entry *>(smem_raw) + threadIdx.x;
    Ray ray;
    const bool hit = ray_setup(p.T, p.origins[3 * r], p.origins[3 * r + 1], p.origins[3 * r + 2],
                               p.dirs[3 * r], p.dirs[3 * r + 1], p.dirs[3 * r + 2], p.tmin, p.tmax, ray);
    if (COLLECT) {
        const int64_t b = p.ray_start[r];
        CollectVisitor v{p.seg_leaf + b, p.seg_t0 + b, p.seg_t1 + b, 0, p.ray_start[r + 1] - b};
        if (hit) traverse<Entry>(p.T.child, p.T.depth, ray, stk, blockDim.x, v);
    } else {
        CountVisitor v;
        if (hit) traverse<Entry>(p.T.child, p.T.depth, ray, stk, blockDim.x, v);
        p.count[r] = v.count;
    }
}

// ------------------------------------------------------------------ repack
// leaf rows (P = 2C + 3K floats) -> sig plane (sig4 float4 per row) and
// rest plane ([w_gamma pad to 4 | w_hh pad to 4], rest4 float4 per row)
__global__ void k_repack(const float *__restrict__ src, int64_t rows, int P, int C, int K3, int sig4,
                         int rest4, int hh_off4, float *sig, float *rest) {
    const int sigw = 4 * sig4, restw = 4 * rest4;
    const int64_t total = rows * (int64_t)(sigw + restw);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / (sigw + restw);
        const int j = (int)(i % (sigw + restw));
        const float *s = src + row * P;
        if (j < sigw) {
            sig[row * sigw + j] = j < C ? s[j] : 0.0f;
        } else {
            const int k = j - sigw;
            float v = 0.0f;
            if (k < C) v = s[C + k];
            else if (k >= 4 * hh_off4 && k < 4 * hh_off4 + K3) v = s[2 * C + (k - 4 * hh_off4)];
            rest[row * restw + k] = v;
        }
    }
}

// ------------------------------------------------------------------ dispatch helpers
template <class F>
int with_nmax(int nmax, F &&f) {
    switch (nmax) {
        case 0: return f(std::integral_constant<int, 0>());
        case 1: return f(std::integral_constant<int, 1>());
        case 2: return f(std::integral_constant<int, 2>());
        case 3: return f(std::integral_constant<int, 3>());
        default: return set_error(VV_E_UNSUPPORTED, "n_max %d not supported on device (max 3)", nmax);
    }
}

size_t stack_bytes(int depth, bool wide) {
    return (size_t)stack_cap(depth) * kBlock * (wide ? sizeof(EntryW) : sizeof(EntryN));
}

template <class Kern>
int prep_smem(Kern k, size_t smem) {
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return set_error(VV_E_CUDA, "smem attribute: %s", cudaGetErrorString(e));
    }
    return VV_OK;
}

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(VV_E_CUDA, "%s launch failed: %s", what, cudaGetErrorString(e));
    return VV_OK;
}

int check_frame(const vv_tree *t, int frame) {
    if (frame < 0 || frame >= t->frames)
        return set_error(VV_E_INVALID, "frame %d out of range [0, %d)", frame, t->frames);
    return VV_OK;
}

int check_cache(const vv_tree *t, const vv_slice *c, int frame) {
    if (!c) return VV_OK;
    if (c->tree != t) return set_error(VV_E_INVALID, "cache belongs to a different tree");
    if (c->frame != frame) return set_error(VV_E_INVALID, "cache built for frame %d, not %d", c->frame, frame);
    return VV_OK;
}

vv_render_opts default_opts() {
    vv_render_opts o;
    o.early_stop = 1e-4;
    o.far_plane = 1e9;
    o.alpha_floor = 1e-3;
    o.edit_weight = 1.0;
    o.tmin = 0.0;
    o.tmax = 1e30;
    return o;
}

SliceView slice_view(const vv_slice *c) {
    SliceView s{nullptr, nullptr, 0};
    if (c) {
        s.sigma = c->d_sigma;
        s.q = c->d_q;
        s.q4 = c->q4;
    }
    return s;
}

int tree_alloc_common(const vv_tree_desc *d, int device, vv_tree **out, bool host_src) {
    if (!d || !out) return set_error(VV_E_INVALID, "null argument");
    if (d->depth < 1 || d->depth > kMaxDepth)
        return set_error(VV_E_UNSUPPORTED, "depth %d outside [1, %d]", d->depth, kMaxDepth);
    if (d->n_max < 0 || d->n_max > kMaxNmax)
        return set_error(VV_E_UNSUPPORTED, "n_max %d outside [0, %d]", d->n_max, kMaxNmax);
    if (d->coeff_count < 1 || d->coeff_count > kMaxC)
        return set_error(VV_E_UNSUPPORTED, "coeff_count %d outside [1, %d]", d->coeff_count, kMaxC);
    if (d->frames < 1) return set_error(VV_E_INVALID, "frames must be >= 1");
    if (d->n_internal < 1) return set_error(VV_E_INVALID, "node table must have >= 1 row");
    if (d->n_leaves < 0 || d->n_leaves > 0x7fffffffLL) return set_error(VV_E_INVALID, "bad n_leaves");
    if (!(d->side > 0)) return set_error(VV_E_INVALID, "bbox side must be positive");
    if ((d->edit_rgb == nullptr) != (d->edit_t == nullptr))
        return set_error(VV_E_INVALID, "edit_rgb and edit_t must both be set or both be NULL");
    DeviceGuard g(device);
    vv_tree *t = new vv_tree();
    memset(t, 0, sizeof(*t));
    t->device = device;
    t->n_leaves = d->n_leaves;
    t->n_internal = d->n_internal;
    t->frames = d->frames;
    t->C = d->coeff_count;
    t->n_max = d->n_max;
    t->K = (d->n_max + 1) * (d->n_max + 2) * (2 * d->n_max + 3) / 6;
    t->S = (d->n_max + 1) * (d->n_max + 1);
    t->depth = d->depth;
    t->has_edits = d->edit_rgb != nullptr;
    const int C = t->C, K3 = 3 * t->K;
    const int P = 2 * C + K3;
    const int sig4 = (C + 3) / 4;
    const int hh_off4 = (C + 3) / 4;
    const int rest4 = hh_off4 + (K3 + 3) / 4;
    const int64_t nl = d->n_leaves, nrows = std::max<int64_t>(nl, 1);
    auto fail = [&](int rc) {
        vv_tree_free(t);
        return rc;
    };
    auto alloc = [&](void **p, size_t bytes) -> int {
        cudaError_t e = cudaMalloc(p, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return set_error(VV_E_NOMEM, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
        }
        t->bytes += (int64_t)bytes;
        return VV_OK;
    };
    int rc;
    const size_t child_b = (size_t)d->n_internal * 8 * sizeof(int32_t);
    if ((rc = alloc((void **)&t->d_child, child_b))) return fail(rc);
    if ((rc = alloc((void **)&t->d_sig, (size_t)nrows * sig4 * sizeof(float4)))) return fail(rc);
    if ((rc = alloc((void **)&t->d_rest, (size_t)nrows * rest4 * sizeof(float4)))) return fail(rc);
    const size_t ab = (size_t)d->frames * C * sizeof(float);
    if ((rc = alloc((void **)&t->d_a, ab))) return fail(rc);
    if ((rc = alloc((void **)&t->d_b, ab))) return fail(rc);
    const cudaMemcpyKind kind = host_src ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    cudaError_t e;
    if ((e = cudaMemcpy(t->d_child, d->node_child, child_b, kind)) != cudaSuccess ||
        (e = cudaMemcpy(t->d_a, d->basis_a, ab, kind)) != cudaSuccess ||
        (e = cudaMemcpy(t->d_b, d->basis_b, ab, kind)) != cudaSuccess)
        return fail(set_error(VV_E_CUDA, "tree copy failed: %s", cudaGetErrorString(e)));
    if (t->has_edits && nl > 0) {
        if ((rc = alloc((void **)&t->d_edit_rgb, (size_t)nl * sizeof(float4)))) return fail(rc);
        if ((rc = alloc((void **)&t->d_edit_t, (size_t)nl * sizeof(int2)))) return fail(rc);
        if ((e = cudaMemcpy(t->d_edit_rgb, d->edit_rgb, nl * sizeof(float4), kind)) != cudaSuccess ||
            (e = cudaMemcpy(t->d_edit_t, d->edit_t, nl * sizeof(int2), kind)) != cudaSuccess)
            return fail(set_error(VV_E_CUDA, "edit copy failed: %s", cudaGetErrorString(e)));
    }
    // payload rows -> padded planes, chunked through a device staging buffer
    if (nl > 0) {
        const int64_t row_b = (int64_t)P * sizeof(float);
        const int64_t chunk = host_src ? std::max<int64_t>(1, std::min<int64_t>(nl, (256ll << 20) / row_b)) : nl;
        float *stage = nullptr;
        if (host_src) {
            if (cudaMalloc(&stage, chunk * row_b) != cudaSuccess) {
                cudaGetLastError();
                return fail(set_error(VV_E_NOMEM, "staging allocation failed"));
            }
        }
        for (int64_t r0 = 0; r0 < nl; r0 += chunk) {
            const int64_t rows = std::min(chunk, nl - r0);
            const float *src = d->leaf_data + r0 * P;
            if (host_src) {
                if ((e = cudaMemcpy(stage, src, rows * row_b, cudaMemcpyHostToDevice)) != cudaSuccess) {
                    cudaFree(stage);
                    return fail(set_error(VV_E_CUDA, "payload upload failed: %s", cudaGetErrorString(e)));
                }
                src = stage;
            }
            k_repack<<<1184, 256>>>(src, rows, P, C, K3, sig4, rest4, hh_off4,
                                    reinterpret_cast<float *>(t->d_sig + r0 * sig4),
                                    reinterpret_cast<float *>(t->d_rest + r0 * rest4));
            if ((e = cudaGetLastError()) != cudaSuccess) {
                if (stage) cudaFree(stage);
                return fail(set_error(VV_E_CUDA, "repack launch failed: %s", cudaGetErrorString(e)));
            }
        }
        e = cudaDeviceSynchronize();
        if (stage) cudaFree(stage);
        if (e != cudaSuccess) return fail(set_error(VV_E_CUDA, "repack failed: %s", cudaGetErrorString(e)));
    }
    TreeView &v = t->view;
    v.child = t->d_child;
    v.sig = t->d_sig;
    v.rest = t->d_rest;
    v.edit_rgb = t->d_edit_rgb;
    v.edit_t = t->d_edit_t;
    v.basis_a = t->d_a;
    v.basis_b = t->d_b;
    v.lo0 = d->bbox_lo[0];
    v.lo1 = d->bbox_lo[1];
    v.lo2 = d->bbox_lo[2];
    v.side = d->side;
    v.depth = d->depth;
    v.C = C;
    v.sig4 = sig4;
    v.rest4 = rest4;
    v.hh_off4 = hh_off4;
    v.frames = d->frames;
    v.nmax = d->n_max;
    *out = t;
    return VV_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

int vv_device_count(int *count) {
    cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) {
        *count = 0;
        return set_error(VV_E_CUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
    }
    return VV_OK;
}

int vv_tree_upload(const vv_tree_desc *host, int device, vv_tree **out) {
    return tree_alloc_common(host, device, out, true);
}

int vv_tree_bind(const vv_tree_desc *dev, int device, vv_tree **out) {
    return tree_alloc_common(dev, device, out, false);
}

int vv_tree_free(vv_tree *t) {
    if (!t) return VV_OK;
    DeviceGuard g(t->device);
    cudaFree(t->d_child);
    cudaFree(t->d_sig);
    cudaFree(t->d_rest);
    cudaFree(t->d_edit_rgb);
    cudaFree(t->d_edit_t);
    cudaFree(t->d_a);
    cudaFree(t->d_b);
    delete t;
    return VV_OK;
}

int vv_tree_info(const vv_tree *t, int64_t *n_leaves, int64_t *n_internal, int32_t *depth, int32_t *frames,
                 int64_t *device_bytes) {
    if (!t) return set_error(VV_E_INVALID, "null tree");
    if (n_leaves) *n_leaves = t->n_leaves;
    if (n_internal) *n_internal = t->n_internal;
    if (depth) *depth = t->depth;
    if (frames) *frames = t->frames;
    if (device_bytes) *device_bytes = t->bytes;
    return VV_OK;
}

int vv_slice_build(const vv_tree *t, int32_t frame, void *stream, vv_slice **out) {
    if (!t || !out) return set_error(VV_E_INVALID, "null argument");
    int rc = check_frame(t, frame);
    if (rc) return rc;
    DeviceGuard g(t->device);
    vv_slice *s = new vv_slice();
    s->tree = t;
    s->device = t->device;
    s->frame = frame;
    s->n_leaves = t->n_leaves;
    s->q4 = (3 * t->S + 3) / 4;
    const int64_t nrows = std::max<int64_t>(t->n_leaves, 1);
    if (cudaMalloc(&s->d_sigma, nrows * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&s->d_q, nrows * s->q4 * sizeof(float4)) != cudaSuccess) {
        cudaGetLastError();
        vv_slice_free(s);
        return set_error(VV_E_NOMEM, "slice allocation failed");
    }
    if (t->n_leaves > 0) {
        SliceParams p;
        p.T = t->view;
        p.K = make_consts(t->n_max);
        p.frame = frame;
        p.n_leaves = t->n_leaves;
        p.sigma = s->d_sigma;
        p.q = s->d_q;
        p.q4 = s->q4;
        const unsigned grid = (unsigned)((t->n_leaves + 255) / 256);
        cudaStream_t st = (cudaStream_t)stream;
        rc = with_nmax(t->n_max, [&](auto N) {
            k_build_slice<decltype(N)::value><<<grid, 256, 0, st>>>(p);
            return check_launch("build_slice");
        });
        if (rc) {
            vv_slice_free(s);
            return rc;
        }
    }
    *out = s;
    return VV_OK;
}

int vv_slice_free(vv_slice *s) {
    if (!s) return VV_OK;
    DeviceGuard g(s->device);
    cudaFree(s->d_sigma);
    cudaFree(s->d_q);
    delete s;
    return VV_OK;
}

int vv_slice_frame(const vv_slice *s, int32_t *frame) {
    if (!s || !frame) return set_error(VV_E_INVALID, "null argument");
    *frame = s->frame;
    return VV_OK;
}

int vv_slice_export(const vv_slice *s, double *sigma, float *q, void *stream) {
    if (!s) return set_error(VV_E_INVALID, "null slice");
    DeviceGuard g(s->device);
    cudaStream_t st = (cudaStream_t)stream;
    const int S3 = 3 * s->tree->S;
    if (sigma) VV_CUDA(cudaMemcpyAsync(sigma, s->d_sigma, s->n_leaves * sizeof(double), cudaMemcpyDeviceToDevice, st));
    if (q && s->n_leaves > 0)
        VV_CUDA(cudaMemcpy2DAsync(q, S3 * sizeof(float), s->d_q, s->q4 * sizeof(float4), S3 * sizeof(float),
                                  s->n_leaves, cudaMemcpyDeviceToDevice, st));
    return VV_OK;
}

static int render_rays_impl(const vv_tree *t, int32_t frame, const vv_slice *cache, const vv_render_opts *o,
                            const double *origins, const double *dirs, int64_t n, double *premult,
                            double *alpha, double *tbar, int32_t *used, int32_t *pops, int32_t *shaded,
                            const int64_t *visit_start, int64_t *visit_leaf, void *stream) {
    if (!t) return set_error(VV_E_INVALID, "null tree");
    int rc = check_frame(t, frame);
    if (rc) return rc;
    if ((rc = check_cache(t, cache, frame))) return rc;
    if (n == 0) return VV_OK;
    if (!origins || !dirs) return set_error(VV_E_INVALID, "null ray arrays");
    const bool visits = visit_leaf != nullptr;
    if (!visits && (!premult || !alpha || !tbar)) return set_error(VV_E_INVALID, "null output arrays");
    DeviceGuard g(t->device);
    const vv_render_opts opts = o ? *o : default_opts();
    RaysParams p;
    memset(&p, 0, sizeof(p));
    p.T = t->view;
    p.S = slice_view(cache);
    p.K = make_consts(t->n_max);
    p.frame = frame;
    p.early_stop = opts.early_stop;
    p.edit_weight = opts.edit_weight;
    p.tmin = opts.tmin;
    p.tmax = opts.tmax;
    p.origins = origins;
    p.dirs = dirs;
    p.n = n;
    p.premult = premult;
    p.alpha = alpha;
    p.tbar = tbar;
    p.used = used;
    p.pops = pops;
    p.shaded = shaded;
    p.visit_start = visit_start;
    p.visit_leaf = visit_leaf;
    const bool wide = t->depth > kNarrowDepth;
    const size_t smem = stack_bytes(t->depth, wide);
    const unsigned grid = (unsigned)((n + kBlock - 1) / kBlock);
    cudaStream_t st = (cudaStream_t)stream;
    const bool cached = cache != nullptr, edits = t->has_edits;
    return with_nmax(t->n_max, [&](auto N) {
        constexpr int NM = decltype(N)::value;
        auto launch = [&](auto kern) {
            int r = prep_smem(kern, smem);
            if (r) return r;
            kern<<<grid, kBlock, smem, st>>>(p);
            return check_launch("render_rays");
        };
#define VV_RAYS_DISPATCH(ENTRY, VIS)                                                              \
    if (cached) {                                                                                 \
        if (edits) return launch(k_render_rays<NM, true, true, ENTRY, VIS>);                      \
        return launch(k_render_rays<NM, true, false, ENTRY, VIS>);                                \
    } else {                                                                                      \
        if (edits) return launch(k_render_rays<NM, false, true, ENTRY, VIS>);                     \
        return launch(k_render_rays<NM, false, false, ENTRY, VIS>);                               \
    }
        if (wide) {
            if (visits) { VV_RAYS_DISPATCH(EntryW, true) }
            else { VV_RAYS_DISPATCH(EntryW, false) }
        } else {
            if (visits) { VV_RAYS_DISPATCH(EntryN, true) }
            else { VV_RAYS_DISPATCH(EntryN, false) }
        }
#undef VV_RAYS_DISPATCH
    });
}

int vv_render_rays(const vv_tree *t, int32_t frame, const vv_slice *cache, const vv_render_opts *opts,
                   const double *origins, const double *dirs, int64_t n, double *premult, double *alpha,
                   double *tbar, int32_t *used, int32_t *pops, int32_t *shaded, void *stream) {
    return render_rays_impl(t, frame, cache, opts, origins, dirs, n, premult, alpha, tbar, used, pops, shaded,
                            nullptr, nullptr, stream);
}

int vv_render_rays_visits(const vv_tree *t, int32_t frame, const vv_slice *cache, const vv_render_opts *opts,
                          const double *origins, const double *dirs, int64_t n, const int64_t *visit_start,
                          int64_t *visit_leaf, void *stream) {
    if (!visit_start || !visit_leaf) return set_error(VV_E_INVALID, "null visit arrays");
    return render_rays_impl(t, frame, cache, opts, origins, dirs, n, nullptr, nullptr, nullptr, nullptr, nullptr,
                            nullptr, visit_start, visit_leaf, stream);
}

static int render_camera_impl(const vv_tree *t, int32_t frame, const vv_slice *cache, const vv_render_opts *o,
                              const vv_camera *cam, float *rgb, float *alpha, float *depth, float *packed,
                              int tile, int shard, int n_shards, void *stream) {
    if (!t || !cam) return set_error(VV_E_INVALID, "null argument");
    int rc = check_frame(t, frame);
    if (rc) return rc;
    if ((rc = check_cache(t, cache, frame))) return rc;
    if (cam->width <= 0 || cam->height <= 0) return set_error(VV_E_INVALID, "bad camera size");
    if (packed && (tile <= 0 || tile % 16 != 0 || n_shards < 1 || shard < 0 || shard >= n_shards))
        return set_error(VV_E_INVALID, "bad tile arguments (tile must be a positive multiple of 16)");
    DeviceGuard g(t->device);
    const vv_render_opts opts = o ? *o : default_opts();
    CamParams p;
    memset(&p, 0, sizeof(p));
    p.T = t->view;
    p.S = slice_view(cache);
    p.K = make_consts(t->n_max);
    p.cam = make_cam(*cam);
    p.frame = frame;
    p.early_stop = opts.early_stop;
    p.edit_weight = opts.edit_weight;
    p.tmin = opts.tmin;
    p.tmax = opts.tmax;
    p.far_plane = opts.far_plane;
    p.alpha_floor = opts.alpha_floor;
    p.rgb = rgb;
    p.alpha = alpha;
    p.depth = depth;
    dim3 grid;
    if (packed) {
        p.packed = packed;
        p.tile = tile;
        p.shard = shard;
        p.n_shards = n_shards;
        p.tiles_x = (cam->width + tile - 1) / tile;
        const int tiles_y = (cam->height + tile - 1) / tile;
        const int total = p.tiles_x * tiles_y;
        const int mine = total > shard ? (total - shard + n_shards - 1) / n_shards : 0;
        if (mine == 0) return VV_OK;
        grid = dim3((unsigned)(mine * (tile / 16) * (tile / 8)));
    } else {
        grid = dim3((unsigned)((cam->width + 15) / 16), (unsigned)((cam->height + 7) / 8));
    }
    const bool wide = t->depth > kNarrowDepth;
    const size_t smem = stack_bytes(t->depth, wide);
    cudaStream_t st = (cudaStream_t)stream;
    const bool cached = cache != nullptr, edits = t->has_edits;
    return with_nmax(t->n_max, [&](auto N) {
        constexpr int NM = decltype(N)::value;
        auto launch = [&](auto kern) {
            int r = prep_smem(kern, smem);
            if (r) return r;
            kern<<<grid, kBlock, smem, st>>>(p);
            return check_launch("render_camera");
        };
#define VV_CAM_DISPATCH(ENTRY)                                                                    \
    if (cached) {                                                                                 \
        if (edits) return launch(k_render_camera<NM, true, true, ENTRY>);                         \
        return launch(k_render_camera<NM, true, false, ENTRY>);                                   \
    } else {                                                                                      \
        if (edits) return launch(k_render_camera<NM, false, true, ENTRY>);                        \
        return launch(k_render_camera<NM, false, false, ENTRY>);                                  \
    }
        if (wide) { VV_CAM_DISPATCH(EntryW) }
        else { VV_CAM_DISPATCH(EntryN) }
#undef VV_CAM_DISPATCH
    });
}

int vv_render_camera(const vv_tree *t, int32_t frame, const vv_slice *cache, const vv_render_opts *opts,
                     const vv_camera *cam, float *rgb, float *alpha, float *depth, void *stream) {
    return render_camera_impl(t, frame, cache, opts, cam, rgb, alpha, depth, nullptr, 0, 0, 1, stream);
}

int vv_render_camera_tiles(const vv_tree *t, int32_t frame, const vv_slice *cache, const vv_render_opts *opts,
                           const vv_camera *cam, int32_t tile, int32_t shard, int32_t n_shards, float *packed,
                           void *stream) {
    if (!packed) return set_error(VV_E_INVALID, "null packed output");
    return render_camera_impl(t, frame, cache, opts, cam, nullptr, nullptr, nullptr, packed, tile, shard, n_shards,
                              stream);
}

int vv_unpack_tiles(const float *packed_all, int32_t width, int32_t height, int32_t tile, int32_t n_shards,
                    float *rgb, float *alpha, float *depth, void *stream) {
    if (!packed_all || width <= 0 || height <= 0 || tile <= 0 || n_shards < 1)
        return set_error(VV_E_INVALID, "bad unpack arguments");
    const int tiles_x = (width + tile - 1) / tile, tiles_y = (height + tile - 1) / tile;
    const int64_t npix = (int64_t)width * height;
    k_unpack_tiles<<<(unsigned)((npix + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        packed_all, width, height, tile, n_shards, tiles_x, tiles_x * tiles_y, rgb, alpha, depth);
    return check_launch("unpack_tiles");
}

int vv_render_scene(const vv_instance *inst, int32_t n_inst, const vv_render_opts *o, const vv_camera *cam,
                    const double *background, float *image, float *alpha, float *depth, void *stream) {
    if (!inst || !cam || !image || !background) return set_error(VV_E_INVALID, "null argument");
    if (n_inst < 1) return set_error(VV_E_INVALID, "scene has no visible instances");
    if (n_inst > kMaxInst) return set_error(VV_E_UNSUPPORTED, "at most %d instances per fused scene", kMaxInst);
    const vv_tree *t0 = inst[0].tree;
    if (!t0) return set_error(VV_E_INVALID, "null tree");
    int max_depth = 0;
    for (int i = 0; i < n_inst; ++i) {
        const vv_tree *t = inst[i].tree;
        if (!t) return set_error(VV_E_INVALID, "null tree in instance %d", i);
        if (t->device != t0->device) return set_error(VV_E_INVALID, "instances on different devices");
        if (t->n_max != t0->n_max) return set_error(VV_E_UNSUPPORTED, "mixed n_max in one fused scene");
        int rc = check_frame(t, inst[i].frame);
        if (rc) return rc;
        max_depth = std::max(max_depth, t->depth);
    }
    DeviceGuard g(t0->device);
    const vv_render_opts opts = o ? *o : default_opts();
    SceneParams p;
    memset(&p, 0, sizeof(p));
    p.K = make_consts(t0->n_max);
    p.cam = make_cam(*cam);
    p.n_inst = n_inst;
    for (int i = 0; i < n_inst; ++i) {
        InstView &v = p.inst[i];
        v.T = inst[i].tree->view;
        v.frame = inst[i].frame;
        v.mode = inst[i].mode;
        vv_camera c2 = *cam;
        memcpy(c2.c2w, inst[i].pose, sizeof(c2.c2w));
        v.cam = make_cam(c2);
        for (int k = 0; k < 12; ++k) v.inv[k] = inst[i].inv[k];
    }
    p.early_stop = opts.early_stop;
    p.edit_weight = opts.edit_weight;
    p.tmin = opts.tmin;
    p.tmax = opts.tmax;
    p.far_plane = opts.far_plane;
    p.alpha_floor = opts.alpha_floor;
    p.bg0 = background[0];
    p.bg1 = background[1];
    p.bg2 = background[2];
    p.image = image;
    p.alpha = alpha;
    p.depth = depth;
    const bool wide = max_depth > kNarrowDepth;
    const size_t smem = stack_bytes(max_depth, wide);
    dim3 grid((unsigned)((cam->width + 15) / 16), (unsigned)((cam->height + 7) / 8));
    cudaStream_t st = (cudaStream_t)stream;
    return with_nmax(t0->n_max, [&](auto N) {
        constexpr int NM = decltype(N)::value;
        auto launch = [&](auto kern) {
            int r = prep_smem(kern, smem);
            if (r) return r;
            kern<<<grid, kBlock, smem, st>>>(p);
            return check_launch("render_scene");
        };
        if (wide) return launch(k_render_scene<NM, EntryW>);
        return launch(k_render_scene<NM, EntryN>);
    });
}

static int segments_impl(const vv_tree *t, const double *origins, const double *dirs, int64_t n, double tmin,
                         double tmax, int64_t *count, const int64_t *ray_start, int64_t *seg_leaf, double *t0,
                         double *t1, void *stream) {
    if (!t) return set_error(VV_E_INVALID, "null tree");
    if (n == 0) return VV_OK;
    DeviceGuard g(t->device);
    SegParams p;
    p.T = t->view;
    p.origins = origins;
    p.dirs = dirs;
    p.n = n;
    p.tmin = tmin;
    p.tmax = tmax;
    p.count = count;
    p.ray_start = ray_start;
    p.seg_leaf = seg_leaf;
    p.seg_t0 = t0;
    p.seg_t1 = t1;
    const bool wide = t->depth > kNarrowDepth;
    const size_t smem = stack_bytes(t->depth, wide);
    const unsigned grid = (unsigned)((n + kBlock - 1) / kBlock);
    cudaStream_t st = (cudaStream_t)stream;
    auto launch = [&](auto kern) {
        int r = prep_smem(kern, smem);
        if (r) return r;
        kern<<<grid, kBlock, smem, st>>>(p);
        return check_launch("segments");
    };
    const bool collect = seg_leaf != nullptr;
    if (wide) return collect ? launch(k_segments<EntryW, true>) : launch(k_segments<EntryW, false>);
    return collect ? launch(k_segments<EntryN, true>) : launch(k_segments<EntryN, false>);
}

int vv_count_segments(const vv_tree *t, const double *origins, const double *dirs, int64_t n, double tmin,
                      double tmax, int64_t *count, void *stream) {
    if (!count) return set_error(VV_E_INVALID, "null count");
    return segments_impl(t, origins, dirs, n, tmin, tmax, count, nullptr, nullptr, nullptr, nullptr, stream);
}

int vv_collect_segments(const vv_tree *t, const double *origins, const double *dirs, int64_t n, double tmin,
                        double tmax, const int64_t *ray_start, int64_t *seg_leaf, double *seg_t0, double *seg_t1,
                        void *stream) {
    if (!ray_start || !seg_leaf || !seg_t0 || !seg_t1) return set_error(VV_E_INVALID, "null output");
    return segments_impl(t, origins, dirs, n, tmin, tmax, nullptr, ray_start, seg_leaf, seg_t0, seg_t1, stream);
}

}  // extern "C"
