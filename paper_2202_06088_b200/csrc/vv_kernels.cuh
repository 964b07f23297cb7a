// vv_kernels.cuh -- kernel templates and their parameter blocks.
//
// Kernels (one thread per ray/pixel, shared-memory traversal stacks):
//   k_render_rays    render_kernel (kernels.py:410-652) over explicit rays
//   k_render_camera  Camera.rays + render_kernel + finalize_layer, fused
//                    (render.py:74-83, 218-240); also the tile-sharded form
//   k_render_scene   render_instance x L + Algorithm 1 + background
//                    (compose.py:373-475, render.py:243-251), fused per pixel
//   k_build_slice    build_slice_kernel (kernels.py:397-407)
//   k_segments       count/collect_segments_kernel (kernels.py:313-367)
//   k_repack         payload rows -> padded [w_sigma] / [w_gamma | w_hh] planes
//   k_unpack_tiles   tile slabs (multi-GPU gather) -> images
// Instantiations live in vv_launch_*.cu (compiled in parallel); the C ABI in
// vv_api.cu calls the launch_* entry points declared at the bottom.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <type_traits>

#include "../../include/voxvid_b200.h"
#include "vv_device.cuh"
#include "vv_host_common.h"

namespace vvk {
using namespace vv;

constexpr int kBlock = 128;
constexpr int kMaxInst = 16;
#ifndef VV_CAM_MINB
#define VV_CAM_MINB 4  // min resident 128-thread blocks per SM for the render kernels
#endif

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

template <int NMAX, int CACHED, bool EDITS, class Entry, bool VISITS>
__global__ void __launch_bounds__(kBlock, VV_CAM_MINB) k_render_rays(const __grid_constant__ RaysParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ float sA[kMaxC], sB[kMaxC];
    load_rows(p.T, p.frame, sA, sB);
    __syncthreads();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= p.n) return;
    const double ox = p.origins[3 * r], oy = p.origins[3 * r + 1], oz = p.origins[3 * r + 2];
    const double dx = p.dirs[3 * r], dy = p.dirs[3 * r + 1], dz = p.dirs[3 * r + 2];
    FrameCtx F{sA, sB, p.frame, p.early_stop, p.edit_weight, nz_chunks(sA, p.T.C), nz_chunks(sB, p.T.C)};
    Shader<NMAX, CACHED, EDITS, VISITS, true> sh(p.T, p.S, F, p.K, (float)dx, (float)dy, (float)dz);
    if (VISITS) sh.visit = p.visit_leaf + p.visit_start[r];
    Ray ray;
    if (ray_setup(p.T, ox, oy, oz, dx, dy, dz, p.tmin, p.tmax, ray))
        traverse<Entry>(p.T.child, p.T.depth, ray, smem_raw, sh);
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

// ------------------------------------------------------------------ coverage
// Pixels whose ray can reach a leaf of a tree: the union of the projected
// rectangles of its 64-leaf chunk boxes (k_coverage, vv_launch_mask.cu; one
// pixel of margin; a box reaching behind the eye covers everything).  A ray
// outside it meets no leaf cell, so its result is exactly the empty pixel
// (premult 0, alpha 0, tbar 0 -> rgb 0, alpha 0, depth far_plane) and the
// kernels skip its setup and walk; a layer of such a ray enters Algorithm 1
// with exactly those values.
struct CoverView {
    const uint32_t *fine;   // (height, words): bit per pixel, small boxes; null: everything covered
    const uint8_t *coarse;  // (ceil(h/16), cw): 16x16-pixel tiles of large boxes
    const int *all;         // a box reached behind the eye: everything covered
    int words, cw;
};
__device__ __forceinline__ bool covered(const CoverView &c, int ix, int iy) {
    if (!c.fine) return true;
    if ((__ldg(c.fine + (size_t)iy * c.words + (ix >> 5)) >> (ix & 31)) & 1u) return true;
    return __ldg(c.coarse + (size_t)(iy >> 4) * c.cw + (ix >> 4)) != 0 || __ldg(c.all) != 0;
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
    // tile mode (tile > 0): this shard's tiles only, written packed (packed
    // != null) or straight into the image planes above (which may be a peer
    // GPU's memory mapped through CUDA IPC)
    float *packed;
    int tile, shard, n_shards, tiles_x;
    int peer;                     // image planes live on another GPU: fence at exit
    int blocks_x;                 // tiles per row (image mode)
    // image mode renders the pixel rectangle [rx0, rx1) x [ry0, ry1) of the
    // full-size planes (the whole image, or one rank's region)
    int rx0, ry0, rx1, ry1;
    // optional launch order of the rectangle's blocks (a permutation of
    // 0..grid-1, costliest first: the expensive blocks do not form the tail
    // of a short region kernel)
    const int32_t *block_order;
    // persistent warps (work != null, image / region mode): a resident grid
    // whose warps take the rectangle's warp chunks (32 rays each) one at a
    // time from the counter *work (zeroed before the launch), in
    // block_order when given -- SM slots never idle while chunks remain
    int *work;   // [next chunk, warps finished]: the last warp out resets both
    int n_work;  // warp chunks in the rectangle
    // optional (persistent mode): per-block walk cost of this render (leaf
    // samples + 1 per ray, atomically summed per warp) -- a camera plan's
    // launch order for the next frame (vv_camera_plan)
    uint32_t *block_cost;
    // optional (image mode): per row band of band_rows rows, the warp chunks
    // finished (each warp fences its stores, then adds 1) -- the copy
    // stream of vv_render_camera_to_host waits on these and copies each
    // band to the host while the rest of the frame renders
    unsigned *band_done;
    int band_rows;
    int band_first;  // rows of band 0 (a short first band starts the copies sooner); 0: band_rows
    CoverView cov;  // image / region mode: pixels that can reach the tree
    int cx0, cy0, cx1, cy1;  // image / region mode: pixel rectangle of the tree's occupied box (inclusive)
    // optional per-pixel leaf-sample counts (render_kernel's consumed
    // segments, up to and including the early-stop one; image mode): written
    // by the production instantiation itself, so its walk is checked
    // bit-exactly against the oracle
    int32_t *used;
    // visible-set slices (VIS kernels, image / region mode): a warp chunk
    // holding a pixel whose walk met a leaf outside the set is listed --
    // (tile x0, tile y0, chunk in tile, lane mask) -- and k_camera_rewalk
    // walks those pixels again per sample, then counts the chunk for its band
    int4 *deferred;
    int *n_deferred;
    // the tree's own child table, for the deferred pixels' walk when T.child
    // is a visible-set walk table (leaves outside the set -> a stand-in row)
    const int32_t *child_full;
};

// band of a row offset from the rectangle's top (banded host copies)
__device__ __forceinline__ int band_of(const CamParams &p, int dy) {
    const int f = p.band_first > 0 ? p.band_first : p.band_rows;
    return dy < f ? 0 : 1 + (dy - f) / p.band_rows;
}

// block = 16x8 pixels; warp = 16x2 pixels (spatially coherent rays)
__device__ __forceinline__ void block_pixel(int bx, int by, int &ix, int &iy) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    ix = bx * 16 + (lane & 15);
    iy = by * 8 + w * 2 + (lane >> 4);
}

// Block work unit: a kTW x kTH pixel tile (one ray per thread); warps take
// VV_CHUNK_W-wide chunks of it.
#ifndef VV_CHUNK_W
#define VV_CHUNK_W 4  // warp chunk = VV_CHUNK_W x (32 / VV_CHUNK_W) pixels (4 x 8 measured best)
#endif
#ifndef VV_CAM_TH
#define VV_CAM_TH 8  // camera block = 16 x VV_CAM_TH pixels, one thread each
#endif
#ifndef VV_CAM_TW
#define VV_CAM_TW 16  // camera block width in pixels
#endif
constexpr int kTW = VV_CAM_TW, kTH = VV_CAM_TH, kTileRays = kTW * kTH;
constexpr int kCamMinBlocks = VV_CAM_MINB * kBlock / kTileRays;  // same warps per SM for any tile height
static_assert(kTileRays % 32 == 0 && kTH % (32 / VV_CHUNK_W) == 0 && kTW % VV_CHUNK_W == 0,
              "camera tile must hold whole warp chunks");

// block -> tile origin (image mode: row-major tiles; tile mode: sub-tiles of
// this shard's tiles); local ray id -> pixel and output slot
__device__ __forceinline__ void block_origin(const CamParams &p, int &x0, int &y0, long long &my_tile, int &lx0,
                                             int &ly0) {
    if (p.tile) {
        const int subs_x = p.tile / kTW, subs = subs_x * (p.tile / kTH);
        my_tile = blockIdx.x / subs;
        const int sub = blockIdx.x % subs;
        lx0 = (sub % subs_x) * kTW;
        ly0 = (sub / subs_x) * kTH;
        const long long tile_id = my_tile * p.n_shards + p.shard;
        x0 = (int)(tile_id % p.tiles_x) * p.tile + lx0;
        y0 = (int)(tile_id / p.tiles_x) * p.tile + ly0;
    } else {
        my_tile = 0;
        lx0 = ly0 = 0;
        const int b = p.block_order ? __ldg(p.block_order + blockIdx.x) : (int)blockIdx.x;
        x0 = p.rx0 + (b % p.blocks_x) * kTW;
        y0 = p.ry0 + (b / p.blocks_x) * kTH;
    }
}

__device__ __forceinline__ void local_pixel(int rid, int &dx, int &dy) {
    constexpr int CW = VV_CHUNK_W, CH = 32 / VV_CHUNK_W;
    const int chunk = rid >> 5, l = rid & 31;
    dx = (chunk % (kTW / CW)) * CW + (l % CW);
    dy = (chunk / (kTW / CW)) * CH + (l / CW);
}

__device__ __forceinline__ void cam_write(const CamParams &p, bool inside, long long slot, float r, float g,
                                          float b, float a, float d) {
    if (p.packed) {
        float *o = p.packed + slot * 5;
        o[0] = r; o[1] = g; o[2] = b; o[3] = a; o[4] = d;
        return;
    }
    if (!inside) return;
    if (p.rgb) {
        p.rgb[3 * slot + 0] = r;
        p.rgb[3 * slot + 1] = g;
        p.rgb[3 * slot + 2] = b;
    }
    if (p.alpha) p.alpha[slot] = a;
    if (p.depth) p.depth[slot] = d;
}

// Camera kernel: one thread per pixel; a block renders one 16x8-pixel tile
// (each warp an 8x4-pixel chunk), so the block's warps stay on neighbouring
// pixels (L1 reuse of node rows and slice rows).  Refill-on-finish
// (persistent) variants were measured slower: see DESIGN.md.
constexpr int kWarpsPerTile = kTileRays / 32;

// Lists the warp chunk when a lane deferred its pixel (every lane calls it).
__device__ __forceinline__ bool defer_chunk(const CamParams &p, bool deferred, int tx0, int ty0, int chunk) {
#ifdef VV_VIS_NODEFER
    return false;
#endif
    const unsigned m = __ballot_sync(0xffffffffu, deferred);
    if (!m) return false;
    if ((threadIdx.x & 31) == 0) p.deferred[atomicAdd(p.n_deferred, 1)] = make_int4(tx0, ty0, chunk, (int)m);
    return true;
}

// Visible-set renders, second kernel: the listed pixels walked again from
// the start, decoding per sample -- the segments, sigma and colour
// arithmetic of the sliced walk, so the same bits -- marking the leaves
// they shade for the next frame's slice; each chunk is then counted for its
// band (banded host copies).  A separate launch keeps this walk's registers
// out of the camera kernel (in-kernel it cost 8%).
template <int NMAX, class Entry>
__global__ void __launch_bounds__(kTileRays, kCamMinBlocks) k_camera_rewalk(const __grid_constant__ CamParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ float sA[kMaxC], sB[kMaxC];
    load_rows(p.T, p.frame, sA, sB);
    __syncthreads();
    const FrameCtx F{sA, sB, p.frame, p.early_stop, p.edit_weight, nz_chunks(sA, p.T.C), nz_chunks(sB, p.T.C)};
    pdl_trigger();
    pdl_wait();  // the camera kernel's list is complete
    const int n = *(volatile const int *)p.n_deferred;
    const int lane = threadIdx.x & 31;
    const int nw = (int)gridDim.x * kWarpsPerTile;
    for (int k = (int)blockIdx.x * kWarpsPerTile + (int)(threadIdx.x >> 5); k < n; k += nw) {
        const int4 e = p.deferred[k];
        if (((unsigned)e.w >> lane) & 1u) {
            int dx_, dy_;
            local_pixel(e.z * 32 + lane, dx_, dy_);
            const int ix = e.x + dx_, iy = e.y + dy_;
            const long long slot = (long long)iy * p.cam.width + ix;
            double dx, dy, dz;
            camera_ray(p.cam, ix, iy, dx, dy, dz);
            Ray ray;
            Shader<NMAX, 0, false, false, false, VV_SEG_MIN, 2> sh(p.T, p.S, F, p.K, (float)dx, (float)dy, (float)dz);
            if (ray_setup(p.T, p.cam.ox, p.cam.oy, p.cam.oz, dx, dy, dz, p.tmin, p.tmax, ray))
                traverse<Entry>(p.child_full ? p.child_full : p.T.child, p.T.depth, ray, smem_raw, sh);
            float r, g, b, a, d;
            finalize(sh.acc0, sh.acc1, sh.acc2, sh.aacc, sh.tacc, 1.0, false, p.alpha_floor, p.far_plane, r, g, b, a,
                     d);
            if (p.used) p.used[slot] = sh.used;
            cam_write(p, true, slot, r, g, b, a, d);
        }
        if (p.band_done) {
            __threadfence();
            __syncwarp();
            if (lane == 0) atomicAdd(p.band_done + band_of(p, e.y - p.ry0), 1u);
        }
    }
    if (p.peer) __threadfence_system();
}

// one pixel of the camera kernel (image / region mode) after the slice wait
template <int NMAX, int CACHED, bool EDITS, class Entry, int SEG, int VIS = 0>
__device__ __forceinline__ int camera_pixel(const CamParams &p, const FrameCtx &F, unsigned char *smem, int ix,
                                            int iy, bool &deferred) {
    const long long slot = (long long)iy * p.cam.width + ix;
    const bool inside = ix < p.rx1 && iy < p.ry1;
    float r = 0.f, g = 0.f, b = 0.f, a = 0.f, d = (float)p.far_plane;
    int cost = 0;
    if (inside && (ix < p.cx0 || ix > p.cx1 || iy < p.cy0 || iy > p.cy1 || !covered(p.cov, ix, iy))) {
        // meets no leaf cell: the empty pixel
        if (p.used) p.used[slot] = 0;
    } else if (inside) {
        double dx, dy, dz;
        camera_ray(p.cam, ix, iy, dx, dy, dz);
        Ray ray;
        const bool hit = ray_setup(p.T, p.cam.ox, p.cam.oy, p.cam.oz, dx, dy, dz, p.tmin, p.tmax, ray);
        Shader<NMAX, CACHED, EDITS, false, false, SEG, VIS> sh(p.T, p.S, F, p.K, (float)dx, (float)dy, (float)dz);
        if (hit) traverse<Entry>(p.T.child, p.T.depth, ray, smem, sh);
        deferred = VIS && sh.deferred;  // k_camera_rewalk writes this pixel
        finalize(sh.acc0, sh.acc1, sh.acc2, sh.aacc, sh.tacc, 1.0, false, p.alpha_floor, p.far_plane, r, g, b, a, d);
        if (p.used) p.used[slot] = sh.used;
        cost = sh.used + 1;
    }
    cam_write(p, inside, slot, r, g, b, a, d);
    return cost;
}

template <int NMAX, int CACHED, bool EDITS, class Entry, int SEG = VV_SEG_MIN, int VIS = 0>
__global__ void __launch_bounds__(kTileRays, kCamMinBlocks) k_render_camera(const __grid_constant__ CamParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ float sA[kMaxC], sB[kMaxC];
    // basis rows before griddepcontrol.wait: immutable tree state (the PDL
    // invariant at launch_pdl); after the wait it costs 1.8% (0.7435 vs
    // 0.730 ms at cfg2)
    load_rows(p.T, p.frame, sA, sB);
    __syncthreads();
    if (p.work) {  // persistent warps over the rectangle's warp chunks
        const FrameCtx F{sA, sB, p.frame, p.early_stop, p.edit_weight, nz_chunks(sA, p.T.C), nz_chunks(sB, p.T.C)};
        pdl_trigger();
        pdl_wait();
        const int lane = threadIdx.x & 31;
        while (true) {
            int idx = 0;
            if (lane == 0) idx = atomicAdd(p.work, 1);
            idx = __shfl_sync(0xffffffffu, idx, 0);
            if (idx >= p.n_work) break;
            const int tb = p.block_order ? __ldg(p.block_order + idx / kWarpsPerTile) : idx / kWarpsPerTile;
            int dx_, dy_;
            local_pixel((idx % kWarpsPerTile) * 32 + lane, dx_, dy_);
            bool deferred = false;
            const int cost = camera_pixel<NMAX, CACHED, EDITS, Entry, SEG, VIS>(
                p, F, smem_raw, p.rx0 + (tb % p.blocks_x) * kTW + dx_, p.ry0 + (tb / p.blocks_x) * kTH + dy_, deferred);
            // (the chunk's origin recomputed behind an opaque copy of tb: kept
            // live across the walk it costs the kernel 10%)
            int tbv = tb;
            if (VIS) asm volatile("" : "+r"(tbv));
            if (VIS && defer_chunk(p, deferred, p.rx0 + (tbv % p.blocks_x) * kTW, p.ry0 + (tbv / p.blocks_x) * kTH,
                                   idx % kWarpsPerTile)) {
                // counted for its band by k_camera_rewalk
            } else if (p.band_done) {
                __threadfence();
                __syncwarp();
                if (lane == 0) atomicAdd(p.band_done + band_of(p, (tb / p.blocks_x) * kTH), 1u);
            }
            __syncwarp();
            if (p.block_cost) {
                const unsigned sum = __reduce_add_sync(0xffffffffu, (unsigned)cost);
                if (lane == 0) atomicAdd(p.block_cost + tb, sum);
            }
        }
        if (p.peer) __threadfence_system();
        // the last warp out leaves the counters zeroed for the next launch
        // (camera plans reuse them without a memset between the kernels)
        if (lane == 0 && atomicAdd(p.work + 1, 1) == (int)(gridDim.x * kWarpsPerTile) - 1) {
            p.work[0] = 0;
            p.work[1] = 0;
        }
        return;
    }
    int x0, y0, lx0, ly0;
    long long my_tile;
    block_origin(p, x0, y0, my_tile, lx0, ly0);
    FrameCtx F{sA, sB, p.frame, p.early_stop, p.edit_weight, nz_chunks(sA, p.T.C), nz_chunks(sB, p.T.C)};
    {
        const int rid = (int)threadIdx.x;  // blockDim.x == kTileRays
        int dx_, dy_;
        local_pixel(rid, dx_, dy_);
        const int ix = x0 + dx_, iy = y0 + dy_;
        const long long slot = p.packed ? my_tile * p.tile * p.tile + (long long)(ly0 + dy_) * p.tile + (lx0 + dx_)
                                        : (long long)iy * p.cam.width + ix;
        float r = 0.f, g = 0.f, b = 0.f, a = 0.f, d = (float)p.far_plane;
        const bool inside = p.tile ? (ix < p.cam.width && iy < p.cam.height) : (ix < p.rx1 && iy < p.ry1);
        double dx = 0.0, dy = 0.0, dz = 1.0;
        Ray ray;
        bool hit = false, deferred = false;
        if (inside) {  // pure arithmetic: overlaps the previous kernel's tail
            camera_ray(p.cam, ix, iy, dx, dy, dz);
            hit = ray_setup(p.T, p.cam.ox, p.cam.oy, p.cam.oz, dx, dy, dz, p.tmin, p.tmax, ray);
        }
        pdl_trigger();
        pdl_wait();  // the frame slice (and node mask, coverage) is complete; earlier writers of the outputs are done
        if (inside) {
            Shader<NMAX, CACHED, EDITS, false, false, SEG, VIS> sh(p.T, p.S, F, p.K, (float)dx, (float)dy, (float)dz);
            if (hit && (p.tile || (ix >= p.cx0 && ix <= p.cx1 && iy >= p.cy0 && iy <= p.cy1 && covered(p.cov, ix, iy))))
                traverse<Entry>(p.T.child, p.T.depth, ray, smem_raw, sh);
            deferred = VIS && sh.deferred;
            finalize(sh.acc0, sh.acc1, sh.acc2, sh.aacc, sh.tacc, 1.0, false, p.alpha_floor, p.far_plane, r, g, b,
                     a, d);
            if (p.used) p.used[slot] = sh.used;
        }
        cam_write(p, inside, slot, r, g, b, a, d);
        if (VIS && !p.tile && defer_chunk(p, deferred, x0, y0, (int)(threadIdx.x >> 5))) {
            // counted for its band by k_camera_rewalk
        } else if (p.band_done) {  // this warp's pixels are stored: count it for its band
            __threadfence();
            __syncwarp();
            if ((threadIdx.x & 31) == 0) atomicAdd(p.band_done + band_of(p, y0 - p.ry0), 1u);
        }
    }
    // peer stores: make them visible system-wide before the kernel retires
    // (the caller's stream-ordered barrier then publishes the frame)
    if (p.peer) __threadfence_system();
}

// ------------------------------------------------------------------ scene
struct InstView {
    TreeView T;
    SliceView S;      // per-instance frame slice (sigma == null: decode per sample)
    CamView cam;      // mode 0: pulled-back pose
    double inv[12];   // mode 1: rows of inv(affine)[:3, :4]
    int frame, mode;
    // pixels [rx0, rx1] x [ry0, ry1] (inclusive) whose ray can reach the
    // instance's occupied leaf cells (its tight box projected, one pixel of
    // margin): outside, the instance's layer is exactly (0, alpha 0, far)
    int rx0, ry0, rx1, ry1;
};

struct SceneParams {
    Consts K;
    CamView cam;
    InstView inst[kMaxInst];
    int n_inst;
    double early_stop, edit_weight, tmin, tmax, far_plane, alpha_floor;
    double bg0, bg1, bg2;
    int composite;  // 1: image = composite over bg; 0: image = blended (unpremultiplied) rgb
    float *image, *alpha, *depth;
    int max_depth;  // deepest instance tree (stack sizing)
    // a scene in several launches (> kMaxInst instances, mixed n_max): the
    // per-pixel Algorithm-1 state (I0, I1, I2, D, A; f64) continues from
    // state_in and, except in the last launch, goes to state_out instead of
    // the outputs; total_inst counts every launch's instances
    const double *state_in;
    double *state_out;
    int total_inst;
    // persistent warps (a scene plan): counters [next chunk, warps done],
    // launch order and per-block costs of the 16x8-pixel blocks
    int *work;
    int n_work, blocks_x;
    const int32_t *block_order;
    uint32_t *block_cost;
};

// CACHED 2: per-instance decode decided at run time (some instances sliced);
// CACHED 0 with EDITS false: every instance decoded per sample and no
// edits (the common scene case, k_render_scene_lean).
// One pixel of the scene kernel: every instance through its pulled-back ray,
// finalized, blended by Algorithm 1 in instance order, then unpremultiplied
// and composited (or handed on to the next launch of a chained scene).
// Returns the pixel's walk cost (samples + 1 per reached instance + 1).
template <int NMAX, class Entry, int CACHED, bool EDITS>
__device__ __forceinline__ int scene_pixel(const SceneParams &p, unsigned char *smem_raw, const float (*sA)[kMaxC],
                                           const float (*sB)[kMaxC], const uint32_t (*sM)[2], int ix, int iy) {
    if (ix >= p.cam.width || iy >= p.cam.height) return 0;
    int cost = 1;
    double cdx, cdy, cdz;
    camera_ray(p.cam, ix, iy, cdx, cdy, cdz);
    // blended state (compose.py:386-405): I (3), D, A
    const int64_t pix = (int64_t)iy * p.cam.width + ix;
    double I0 = 0, I1 = 0, I2 = 0, D = 0, A = 0;
    bool have = false;
    if (p.state_in) {  // an earlier launch's instances
        const double *s = p.state_in + 5 * pix;
        I0 = s[0]; I1 = s[1]; I2 = s[2]; D = s[3]; A = s[4];
        have = true;
    }
    for (int i = 0; i < p.n_inst; ++i) {
        const InstView &v = p.inst[i];
        double ox, oy, oz, dx = 0.0, dy = 0.0, dz = 1.0, scale = 1.0;
        bool scaled = false;
        const bool reach = ix >= v.rx0 && ix <= v.rx1 && iy >= v.ry0 && iy <= v.ry1;
        if (!reach) {  // no leaf cell on this ray: the empty layer (no setup, no walk)
            ox = oy = oz = 0.0;
            scaled = v.mode != 0;
        } else if (v.mode == 0) {
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
        FrameCtx F{sA[i], sB[i], v.frame, p.early_stop, p.edit_weight, sM[i][0], sM[i][1]};
        Shader<NMAX, CACHED, EDITS, false> sh(v.T, v.S, F, p.K, (float)dx, (float)dy, (float)dz);
        Ray ray;
        if (reach && ray_setup(v.T, ox, oy, oz, dx, dy, dz, p.tmin, p.tmax, ray))
            traverse<Entry>(v.T.child, v.T.depth, ray, smem_raw, sh);
        cost += reach ? sh.used + 1 : 0;
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
        if (!have) {
            I0 = li0; I1 = li1; I2 = li2; D = ld; A = al;
            have = true;
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
    if (p.state_out) {  // a later launch continues the blend
        double *s = p.state_out + 5 * pix;
        s[0] = I0; s[1] = I1; s[2] = I2; s[3] = D; s[4] = A;
        return cost;
    }
    if (p.total_inst > 1) {  // unpremultiply the blend (compose.py:457-460)
        const double safe = A > 1e-300 ? A : 1e-300;
        if (A > 0.0) {
            I0 = xdiv(I0, safe);
            I1 = xdiv(I1, safe);
            I2 = xdiv(I2, safe);
        } else {
            I0 = I1 = I2 = 0.0;
        }
    }
    if (p.image && p.composite) {
        // composite_background: a * rgb + (1 - a) * bg (render.py:243-251)
        const double om = xsub(1.0, A);
        p.image[3 * pix + 0] = (float)xadd(xmul(A, I0), xmul(om, p.bg0));
        p.image[3 * pix + 1] = (float)xadd(xmul(A, I1), xmul(om, p.bg1));
        p.image[3 * pix + 2] = (float)xadd(xmul(A, I2), xmul(om, p.bg2));
    } else if (p.image) {  // the blended layer, for the lighting passes
        p.image[3 * pix + 0] = (float)I0;
        p.image[3 * pix + 1] = (float)I1;
        p.image[3 * pix + 2] = (float)I2;
    }
    if (p.alpha) p.alpha[pix] = (float)A;
    if (p.depth) p.depth[pix] = (float)D;
    return cost;
}

template <int NMAX, class Entry, int CACHED, bool EDITS>
__device__ __forceinline__ void scene_body(const SceneParams &p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ float sA[kMaxInst][kMaxC], sB[kMaxInst][kMaxC];
    __shared__ uint32_t sM[kMaxInst][2];
    for (int i = 0; i < p.n_inst; ++i) load_rows(p.inst[i].T, p.inst[i].frame, sA[i], sB[i]);
    __syncthreads();
    if ((int)threadIdx.x < p.n_inst) {
        sM[threadIdx.x][0] = nz_chunks(sA[threadIdx.x], p.inst[threadIdx.x].T.C);
        sM[threadIdx.x][1] = nz_chunks(sB[threadIdx.x], p.inst[threadIdx.x].T.C);
    }
    __syncthreads();
    if (p.work) {  // persistent warps over the 16x2-pixel warp chunks, in cost order when planned
        const int lane = threadIdx.x & 31;
        while (true) {
            int idx = 0;
            if (lane == 0) idx = atomicAdd(p.work, 1);
            idx = __shfl_sync(0xffffffffu, idx, 0);
            if (idx >= p.n_work) break;
            const int tb = p.block_order ? __ldg(p.block_order + idx / 4) : idx / 4;
            const int w = idx % 4;
            const int ix = (tb % p.blocks_x) * 16 + (lane & 15), iy = (tb / p.blocks_x) * 8 + w * 2 + (lane >> 4);
            const int cost = scene_pixel<NMAX, Entry, CACHED, EDITS>(p, smem_raw, sA, sB, sM, ix, iy);
            __syncwarp();
            if (p.block_cost) {
                const unsigned sum = __reduce_add_sync(0xffffffffu, (unsigned)cost);
                if (lane == 0) atomicAdd(p.block_cost + tb, sum);
            }
        }
        if (lane == 0 && atomicAdd(p.work + 1, 1) == (int)(gridDim.x * (blockDim.x / 32)) - 1) {
            p.work[0] = 0;
            p.work[1] = 0;
        }
        return;
    }
    int ix, iy;
    block_pixel(blockIdx.x, blockIdx.y, ix, iy);
    scene_pixel<NMAX, Entry, CACHED, EDITS>(p, smem_raw, sA, sB, sM, ix, iy);
}

template <int NMAX, class Entry>
__global__ void __launch_bounds__(kBlock) k_render_scene(const __grid_constant__ SceneParams p) {
    scene_body<NMAX, Entry, 2, true>(p);
}

#ifdef VV_SCENE_LEAN_MINB
#define VV_SCENE_LEAN_BOUNDS __launch_bounds__(kBlock, VV_SCENE_LEAN_MINB)
#else
#define VV_SCENE_LEAN_BOUNDS __launch_bounds__(kBlock)
#endif
template <int NMAX, class Entry>
__global__ void VV_SCENE_LEAN_BOUNDS k_render_scene_lean(const __grid_constant__ SceneParams p) {
    scene_body<NMAX, Entry, 0, false>(p);
}

// ------------------------------------------------------------------ playback, several frames
// k_render_camera for KF frames of one camera in one walk (ShaderMulti):
// per-frame slices (required), images and results identical to KF
// single-frame renders.
struct CamMultiParams {
    TreeView T;
    SliceView S[kMaxMulti];
    int frames[kMaxMulti];
    Consts K;
    CamView cam;
    double early_stop, edit_weight, tmin, tmax, far_plane, alpha_floor;
    float *rgb[kMaxMulti], *alpha[kMaxMulti], *depth[kMaxMulti];
    int blocks_x;
    int cx0, cy0, cx1, cy1;  // pixel rectangle of the tree's occupied box (inclusive)
    CoverView cov;           // pixels that can reach the tree (a plan's cached coverage)
    // persistent warps (a plan): counters, launch order and per-block costs
    int *work;
    int n_work;
    const int32_t *block_order;
    uint32_t *block_cost;
};

#ifndef VV_MULTI_MINB_HI
#define VV_MULTI_MINB_HI kCamMinBlocks  // resident blocks for 3- and 4-frame walks
#endif

// One pixel of the shared-walk playback kernel; returns its walk cost.
template <int NMAX, int KF, bool EDITS, class Entry, int SEG>
__device__ __forceinline__ int multi_pixel(const CamMultiParams &p, unsigned char *smem_raw, int ix, int iy) {
    if (ix >= p.cam.width || iy >= p.cam.height) return 0;
    const bool reach = ix >= p.cx0 && ix <= p.cx1 && iy >= p.cy0 && iy <= p.cy1 && covered(p.cov, ix, iy);
    double dx = 0.0, dy = 0.0, dz = 1.0;
    if (reach) camera_ray(p.cam, ix, iy, dx, dy, dz);
    ShaderMulti<NMAX, KF, EDITS, SEG> sh(p.T, p.S, p.frames, p.K, p.early_stop, p.edit_weight, (float)dx, (float)dy,
                                        (float)dz);
    Ray ray;
    int cost = 1;
    if (reach && ray_setup(p.T, p.cam.ox, p.cam.oy, p.cam.oz, dx, dy, dz, p.tmin, p.tmax, ray)) {
        traverse<Entry>(p.T.child, p.T.depth, ray, smem_raw, sh);
        cost += sh.used;
    }
    const long long slot = (long long)iy * p.cam.width + ix;
#pragma unroll
    for (int k = 0; k < KF; ++k) {
        float r, g, b, a, d;
        finalize(sh.acc0[k], sh.acc1[k], sh.acc2[k], sh.aacc[k], sh.tacc[k], 1.0, false, p.alpha_floor,
                 p.far_plane, r, g, b, a, d);
        if (p.rgb[k]) {
            p.rgb[k][3 * slot + 0] = r;
            p.rgb[k][3 * slot + 1] = g;
            p.rgb[k][3 * slot + 2] = b;
        }
        if (p.alpha[k]) p.alpha[k][slot] = a;
        if (p.depth[k]) p.depth[k][slot] = d;
    }
    return cost;
}

template <int NMAX, int KF, bool EDITS, class Entry, int SEG = VV_SEG_MIN>
__global__ void __launch_bounds__(kTileRays, KF >= 3 ? VV_MULTI_MINB_HI : kCamMinBlocks)
    k_render_camera_multi(const __grid_constant__ CamMultiParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (p.work) {  // persistent warps over the warp chunks, in the plan's cost order
        const int lane = threadIdx.x & 31;
        while (true) {
            int idx = 0;
            if (lane == 0) idx = atomicAdd(p.work, 1);
            idx = __shfl_sync(0xffffffffu, idx, 0);
            if (idx >= p.n_work) break;
            const int tb = p.block_order ? __ldg(p.block_order + idx / kWarpsPerTile) : idx / kWarpsPerTile;
            int dx_, dy_;
            local_pixel((idx % kWarpsPerTile) * 32 + lane, dx_, dy_);
            const int cost = multi_pixel<NMAX, KF, EDITS, Entry, SEG>(p, smem_raw, (tb % p.blocks_x) * kTW + dx_,
                                                                     (tb / p.blocks_x) * kTH + dy_);
            __syncwarp();
            if (p.block_cost) {
                const unsigned sum = __reduce_add_sync(0xffffffffu, (unsigned)cost);
                if (lane == 0) atomicAdd(p.block_cost + tb, sum);
            }
        }
        if (lane == 0 && atomicAdd(p.work + 1, 1) == (int)(gridDim.x * kWarpsPerTile) - 1) {
            p.work[0] = 0;
            p.work[1] = 0;
        }
        return;
    }
    const int bx = blockIdx.x % p.blocks_x, by = blockIdx.x / p.blocks_x;
    int dx_, dy_;
    local_pixel((int)threadIdx.x, dx_, dy_);  // blockDim.x == kTileRays
    multi_pixel<NMAX, KF, EDITS, Entry, SEG>(p, smem_raw, bx * kTW + dx_, by * kTH + dy_);
}

// ------------------------------------------------------------------ slice
struct SliceParams {
    TreeView T;
    Consts K;
    int n_frames;               // 1..kMaxMulti frames sliced from one read of the payload
    int frame[kMaxMulti];
    int64_t n_leaves;
    float4 *rec[kMaxMulti];     // (n_leaves, rec4) slice records per frame
    int rec4;
    uint32_t mS, mG;            // w_sigma / w_gamma chunks the frames need (union of nz_chunks)
    int skip_dark;              // render-internal slice: dark chunks get sigma only (no colour)
    uint8_t *lit;               // optional (n_leaves): bit f set iff frame f's sigma > 0 (node masks)
    // optional: slice only the chunks listed (region renders; written by
    // k_chunk_cull, the previous kernel -- read after griddepcontrol.wait)
    const int32_t *chunk_list;
    const int32_t *n_list;
    // visible-set slices (k_slice_visible): the tree's visible set is the
    // union of two bitmaps over leaf rows (null: every leaf); only leaves in
    // it get their colour, a lit leaf outside it -sigma (SliceView)
    const uint32_t *vis0, *vis1;
    // with a walk table (k_slice_leaves): the set's leaf rows, listed by k_vis_table
    const int32_t *leaf_list;
    const int32_t *n_leaf_list;
    // two-phase lit pass (dark-heavy trees, whole tree): k_slice_lit lists the
    // lit leaves here (lit_n zeroed) for k_slice_leaves; dark_unread: the
    // walks use this slice's node mask, which cuts every dark leaf, so the
    // dark leaves' records are not written
    int32_t *lit_list;
    int32_t *lit_n;
    int dark_unread;
    // a region render: bit c set iff 64-leaf chunk c is in the region's
    // chunk list (k_slice_leaves skips the set's other leaves: the region's
    // rays cannot reach them)
    const uint32_t *chunk_bits;
};

// build_slice_kernel (kernels.py:397-407).  Persistent warps take chunks of
// consecutive leaves (64; 32 for 3- and 4-frame passes), strided over the
// grid so the chunks in flight are neighbours in HBM.  Each warp owns a
// double-buffered shared-memory stage.  One lane issues the chunk's TMA
// bulk copies, completed on an mbarrier: one per w_sigma / w_gamma float4
// chunk the group's A / B rows do not zero out (chunk-major planes, 1 KB
// contiguous each) and one for the w_hh rows.  Meanwhile the warp slices
// the previous chunk, each lane taking leaves lane and lane + 32, from
// shared memory.
//   * Basis chunks that are all zero are never read; their products are
//     +-0 and the sums skip them bit-exactly (nz_chunks).
//   * The records are staged in shared memory and leave as the chunk's
//     contiguous bytes (coalesced stores).
//   * Render-only passes also skip the colour of chunks dark in every frame
//     (see below).
#ifndef VV_SLICE_WARPS
#define VV_SLICE_WARPS 4  // max warps per block (fewer when a warp's stages are large)
#endif
#ifndef VV_SLICE_BPS
#define VV_SLICE_BPS 1  // resident slice blocks per SM (0: as many as fit)
#endif
constexpr int kSliceWarps = VV_SLICE_WARPS;
#ifndef VV_SLICE_RUNS
#define VV_SLICE_RUNS 0  // 1: contiguous runs of chunks per warp instead of strided
#endif
#ifndef VV_SLICE_CHUNK
#define VV_SLICE_CHUNK 64  // leaves per staged chunk (a multiple of 32; lanes loop over their leaves)
#endif
constexpr int kSliceChunk = VV_SLICE_CHUNK;
#ifndef VV_SLICE_CHUNK_MULTI
#define VV_SLICE_CHUNK_MULTI 32  // leaves per staged chunk for 3- and 4-frame passes (measured 6% faster than 64)
#endif
// a KF-frame pass stages KF frames' records per warp: more frames, smaller chunks (more warps)
__host__ __device__ constexpr int slice_chunk(int kf) { return kf >= 3 ? VV_SLICE_CHUNK_MULTI : kSliceChunk; }
static_assert(kSliceChunk % 32 == 0 && VV_SLICE_CHUNK_MULTI % 32 == 0, "slice chunk must be whole warps of leaves");

__host__ __device__ inline size_t slice_stage_floats4(int need, int hh4, int chunk = kSliceChunk) {
    return (size_t)chunk * (need + hh4);  // need = staged w_sigma + w_gamma chunks
}
#ifndef VV_SLICE_STAGE_OUT
#define VV_SLICE_STAGE_OUT 1  // records staged in shared memory, written out coalesced (0: direct per-lane stores)
#endif
// float4 per warp for the staged output records (row stride R4 + 1: no bank conflicts)
__host__ __device__ inline size_t slice_out_floats4(int kf, int r4) {
    return VV_SLICE_STAGE_OUT ? (size_t)kf * slice_chunk(kf) * (r4 + 1) : 0;
}

// KF frames (playback groups) are sliced from ONE read of the payload: a
// staged row's w_sigma / w_gamma entries are read once and feed KF sigma
// (f64) and KF gamma (fp32) accumulators side by side -- each frame keeps
// exactly its single-frame summation order -- and w_hh is loaded once for
// the KF HH->SH slices.
template <int NMAX, int KF>
__global__ void __launch_bounds__(kSliceWarps * 32) k_build_slice(const __grid_constant__ SliceParams p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ float sA[KF][kMaxC], sB[KF][kMaxC];
    __shared__ double dA[KF][kMaxC];  // A rows widened once (the values sigma_pre multiplies)
    constexpr int kChunk = slice_chunk(KF);
    constexpr int kPer = kChunk / 32;  // leaves per lane per chunk
    constexpr int R4 = slice_rec4(Basis<NMAX>::S);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int hh4 = p.T.hh4;
    const uint32_t mS = p.mS, mG = p.mG;  // chunk masks (host: nz_chunks of the group's rows)
    const int nS = __popc(mS), nG = __popc(mG);
    const size_t stage4 = slice_stage_floats4(nS + nG, hh4, kChunk);
    const size_t out4 = slice_out_floats4(KF, R4);
    float4 *wbase = reinterpret_cast<float4 *>(smem_raw) + (size_t)warp * (2 * stage4 + 2 + out4);
    float4 *obuf = wbase + 2 * stage4 + 2;  // (KF, kChunk, R4 + 1) when VV_SLICE_STAGE_OUT
    // bar[0..1]: a stage's staged copies; bar[2..3]: its colour rows fetched late
    uint64_t *bar = reinterpret_cast<uint64_t *>(wbase + 2 * stage4);
    if (lane == 0) {
#pragma unroll
        for (int b = 0; b < 4; ++b) mbar_init(&bar[b], 1);
        mbar_fence_init();
    }
#pragma unroll
    for (int f = 0; f < KF; ++f) load_rows(p.T, p.frame[f], sA[f], sB[f]);
    __syncthreads();
    for (int i = threadIdx.x; i < KF * kMaxC; i += blockDim.x) dA[i / kMaxC][i % kMaxC] = (double)sA[i / kMaxC][i % kMaxC];
    __syncthreads();
    const int C = p.T.C;
    const int64_t ls = p.T.lstride;
    const int64_t n_chunks = (p.n_leaves + kChunk - 1) / kChunk;
    const int nw = blockDim.x >> 5;  // <= kSliceWarps: the launcher fits the stages in shared memory
    const int64_t n_warps = (int64_t)gridDim.x * nw, wid = (int64_t)blockIdx.x * nw + warp;
#if VV_SLICE_RUNS
    // contiguous runs of chunks per warp (the chunk before is a spatial neighbour)
    int64_t c_begin = n_chunks * wid / n_warps, c_end = n_chunks * (wid + 1) / n_warps, c_step = 1;
#else
    // chunks strided over the warps: the chunks in flight at any time are
    // neighbours in HBM
    int64_t c_begin = wid, c_end = n_chunks, c_step = n_warps;
#endif
    // list mode: positions in the chunk list instead of chunk ids
    const bool listed = p.chunk_list != nullptr;
    auto chunk_at = [&](int64_t i) -> int64_t { return listed ? (int64_t)p.chunk_list[i] : i; };
    // stage: [needed w_sigma chunks][kChunk leaves] | [needed w_gamma chunks][kChunk] | [leaves][hh4]
    auto rows_of = [&](int64_t c) { return (int)min((int64_t)kChunk, p.n_leaves - c * kChunk); };
    (void)rows_of;
    auto issue_colour = [&](int64_t c, int stg, uint64_t *b, bool arrive) {
        const int64_t base = c * kChunk;
        const int rows = rows_of(c);
        float4 *dst = wbase + stg * stage4 + (size_t)nS * kChunk;
        const uint32_t cb = (uint32_t)rows * 16, hb = (uint32_t)rows * hh4 * 16;
        if (arrive) mbar_expect_tx(b, (uint32_t)nG * cb + hb);
        for (uint32_t m = mG; m; m &= m - 1, dst += kChunk)
            bulk_g2s(dst, p.T.gam + (__ffs(m) - 1) * ls + base, cb, b);
        bulk_g2s(dst, p.T.hh + base * hh4, hb, b);
    };
    auto issue = [&](int64_t c, int stg, bool colour) {  // lane 0
        const int64_t base = c * kChunk;
        const int rows = rows_of(c);
        float4 *dst = wbase + stg * stage4;
        const uint32_t cb = (uint32_t)rows * 16, hb = (uint32_t)rows * hh4 * 16;
        mbar_expect_tx(&bar[stg], (uint32_t)nS * cb + (colour ? (uint32_t)nG * cb + hb : 0u));
        for (uint32_t m = mS; m; m &= m - 1, dst += kChunk)
            bulk_g2s(dst, p.T.sig + (__ffs(m) - 1) * ls + base, cb, &bar[stg]);
        if (colour) issue_colour(c, stg, &bar[stg], false);
    };
    // colour rows are staged with the sigma chunks while the chunks are
    // bright; a dark chunk (every leaf's sigma 0 in every frame: the shader
    // never reads its colour, kernels.py:556-559) only gets its sigma
    // written, and while chunks stay dark the colour rows are not fetched
    // (render-internal slices of trees without edits: p.skip_dark)
    uint32_t colour_in = 3u;  // bit s: stage s was issued with its colour rows
    // lane 0 stages list position i
    auto stage = [&](int64_t i, int stg, bool colour) { issue(chunk_at(i), stg, colour); };
    // payload reads only: may overlap the previous kernel
    if (lane == 0 && !listed) {
        if (c_begin < c_end) stage(c_begin, 0, true);
        if (c_begin + c_step < c_end) stage(c_begin + c_step, 1, true);
    }
    pdl_trigger();
    pdl_wait();  // no record is written before the previous kernel is complete
    if (listed) {  // the list is the previous kernel's output
        const int64_t nl = (int64_t)*(volatile const int32_t *)p.n_list;
#if VV_SLICE_RUNS
        c_begin = nl * wid / n_warps;
        c_end = nl * (wid + 1) / n_warps;
#else
        c_end = nl;
#endif
        if (lane == 0) {
            if (c_begin < c_end) stage(c_begin, 0, true);
            if (c_begin + c_step < c_end) stage(c_begin + c_step, 1, true);
        }
    }
    uint32_t late_par = 0;  // phase parity of bar[2], bar[3]
    int k = 0;
    for (int64_t ci = c_begin; ci < c_end; ci += c_step, ++k) {
        const int64_t c = chunk_at(ci);
        if (kDebugChecks && (c < 0 || c >= n_chunks)) debug_violation(p.T.dbg, VV_DBG_CHUNK);
        const int stg = k & 1;
        mbar_wait(&bar[stg], (uint32_t)((k >> 1) & 1));
        const int64_t base = c * kChunk;
        const int rows = rows_of(c);
        const float4 *st4 = wbase + stg * stage4;
        // sigma_pre (kernels.py:374-381, f64, sequential), every frame, over
        // the needed chunks in column order
        double sp[kPer][KF];
        bool lit = false;
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int r = lane + 32 * u;
#pragma unroll
            for (int f = 0; f < KF; ++f) sp[u][f] = 0.0;
            if (r < rows) {
                const float4 *sv = st4 + r;
                for (uint32_t m = mS; m; m &= m - 1, sv += kChunk) {
                    const float4 v = ld4<false>(sv);
                    const double w[4] = {(double)v.x, (double)v.y, (double)v.z, (double)v.w};
                    const int cc = 4 * (__ffs(m) - 1);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        if (cc + e < C) {
#pragma unroll
                            for (int f = 0; f < KF; ++f) sp[u][f] = xadd(sp[u][f], xmul(dA[f][cc + e], w[e]));
                        }
                    }
                }
#pragma unroll
                for (int f = 0; f < KF; ++f) lit |= sp[u][f] > 0.0;
            }
        }
        const bool bright = !p.skip_dark || __any_sync(0xffffffffu, lit);
        if (bright && !((colour_in >> stg) & 1u)) {  // mispredicted dark: fetch the colour rows now
            if (lane == 0) {
                fence_proxy_async();  // the colour region was last read through the generic proxy
                issue_colour(c, stg, &bar[2 + stg], true);
            }
            mbar_wait(&bar[2 + stg], (late_par >> stg) & 1u);
            late_par ^= 1u << stg;
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int r = lane + 32 * u;
            if (r >= rows) continue;
            if (p.lit) {  // coalesced byte per leaf: which frames see it lit
                uint32_t bits = 0;
#pragma unroll
                for (int f = 0; f < KF; ++f) bits |= (sp[u][f] > 0.0 ? 1u : 0u) << f;
                p.lit[base + r] = (uint8_t)bits;
            }
            if (!bright) {  // sigma only: the record's last float4 pair (one sector at even R4)
#pragma unroll
                for (int f = 0; f < KF; ++f) {
                    const double sigma = sp[u][f] > 0.0 ? sp[u][f] : 0.0;
                    const unsigned long long sb = (unsigned long long)__double_as_longlong(sigma);
                    float4 *o = p.rec[f] + (base + r) * p.rec4 + (R4 - 1);
                    if (R4 % 2 == 0) o[-1] = make_float4(0.f, 0.f, 0.f, 0.f);
                    *o = make_float4(0.f, 0.f, __uint_as_float((unsigned)(sb & 0xffffffffu)),
                                     __uint_as_float((unsigned)(sb >> 32)));
                }
                continue;
            }
            // the gamma dot (fp32), every frame, over the needed chunks
            float gp[KF];
#pragma unroll
            for (int f = 0; f < KF; ++f) gp[f] = 0.0f;
            const float4 *sv = st4 + (size_t)nS * kChunk + r;
            for (uint32_t m = mG; m; m &= m - 1, sv += kChunk) {
                const float4 g = ld4<false>(sv);
                const float gw[4] = {g.x, g.y, g.z, g.w};
                const int cc = 4 * (__ffs(m) - 1);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if (cc + e < C) {
#pragma unroll
                        for (int f = 0; f < KF; ++f) gp[f] = __fmaf_rn(sB[f][cc + e], gw[e], gp[f]);
                    }
                }
            }
            const float4 *shh = st4 + (size_t)(nS + nG) * kChunk + (size_t)r * hh4;
            float wh[4 * Basis<NMAX>::HH4];
            load_hh<NMAX, false>(shh, wh);
#pragma unroll
            for (int f = 0; f < KF; ++f) {
                float q[4 * R4];
#pragma unroll
                for (int i = 0; i < 4 * R4; ++i) q[i] = 0.0f;
                float R[Basis<NMAX>::NPAIRS];
                radial<NMAX>(sigmoidf_(gp[f]), p.K, R);
#pragma unroll
                for (int l = 0; l <= NMAX; ++l)
#pragma unroll
                    for (int m = -l; m <= l; ++m) {
                        const int j = l * l + l + m;
                        slice_col<NMAX>(R, wh, l, m, q[3 * j + 0], q[3 * j + 1], q[3 * j + 2]);
                    }
                const double sigma = sp[u][f] > 0.0 ? sp[u][f] : 0.0;  // max(0.0, sp)
                const unsigned long long sb = (unsigned long long)__double_as_longlong(sigma);
                q[4 * R4 - 2] = __uint_as_float((unsigned)(sb & 0xffffffffu));
                q[4 * R4 - 1] = __uint_as_float((unsigned)(sb >> 32));
                float4 *o = VV_SLICE_STAGE_OUT ? obuf + ((size_t)f * kChunk + r) * (R4 + 1)
                                               : p.rec[f] + (base + r) * p.rec4;
#pragma unroll
                for (int i = 0; i < R4; ++i) o[i] = make_float4(q[4 * i], q[4 * i + 1], q[4 * i + 2], q[4 * i + 3]);
            }
        }
        __syncwarp();
        if (VV_SLICE_STAGE_OUT && bright) {  // the chunk's records are contiguous: coalesced float4 stores
#pragma unroll
            for (int f = 0; f < KF; ++f) {
                float4 *dst = p.rec[f] + base * R4;
                const float4 *src = obuf + (size_t)f * kChunk * (R4 + 1);
                for (int k = lane; k < rows * R4; k += 32) dst[k] = src[(k / R4) * (R4 + 1) + k % R4];
            }
            __syncwarp();
        }
        // stage consumed: refill it with the chunk two ahead, predicting its
        // colour rows are needed iff this chunk's were
        colour_in = (colour_in & ~(1u << stg)) | ((uint32_t)bright << stg);
        if (lane == 0 && ci + 2 * c_step < c_end) {
            fence_proxy_async();
            stage(ci + 2 * c_step, stg, bright);
        }
    }
}

#ifndef VV_SIGMA_TAIL
#define VV_SIGMA_TAIL 2  // float4 per sigma-only record: 32 B measured best (0.166 ms vs 0.191 with 64 B at cfg2)
#endif
// Visible-set slice in one pass (k_slice_visible): one warp per 64-leaf
// chunk (every chunk, or the region's chunk list); lane 0 reads the chunk's
// visible bits once (no bitmaps: every leaf visible, a tree's first slice).
// Each lane takes leaves lane and lane + 32 straight from global memory:
// sigma_pre (f64, kernels.py:374-381), and for a leaf in the set the colour
// -- gamma_s -> radial -> slice_col, the operations and order of
// k_build_slice and of the per-sample shader, so the same bits -- stored as
// its whole record (one 128-byte line at n_max 2); any other leaf gets its
// sigma pair, negated when lit.  No staging: the set is a fifth of the
// leaves, scattered over a third of the chunks, and a thread per leaf keeps
// ~15 independent loads in flight where the staged pass's two stages per
// warp left it latency-bound (0.41 of HBM peak).
#ifndef VV_VIS_MINB
#define VV_VIS_MINB 10  // min resident 64-thread blocks per SM (91 registers, no spills): 0.1357 vs 0.138 ms; 12 spills (0.142)
#endif
#ifndef VV_VIS_BLOCK
#define VV_VIS_BLOCK 64  // threads per block: 0.138 vs 0.143 ms with 256 (cfg2, more resident warps at 96 registers)
#endif
template <int NMAX>
__global__ void __launch_bounds__(VV_VIS_BLOCK, NMAX >= 3 ? 4 : VV_VIS_MINB)  // n_max 3: no register cap (spills)
    k_slice_visible(const __grid_constant__ SliceParams p) {
    __shared__ float sA[kMaxC], sB[kMaxC];
    load_rows(p.T, p.frame[0], sA, sB);
    __syncthreads();
    constexpr int R4 = slice_rec4(Basis<NMAX>::S);
    constexpr int TAIL = R4 % VV_SIGMA_TAIL == 0 ? VV_SIGMA_TAIL : (R4 % 2 == 0 ? 2 : 1);
    const int lane = threadIdx.x & 31;
    const bool listed = p.chunk_list != nullptr;
    const bool all = p.vis0 == nullptr;
    // no set and skip_dark (a render-only slice without a visible set): the
    // colour of every lit leaf, sigma alone for the dark ones
    const bool lit_only = all && p.skip_dark;
    pdl_trigger();
    pdl_wait();  // the bitmaps and the region list are the previous work's; records written after
    const int64_t n_chunks = (p.n_leaves + 63) / 64;
    const int64_t n_items = listed ? (int64_t)*(volatile const int32_t *)p.n_list : n_chunks;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    // a warp's next 32 chunks: lane j reads the bits of the j-th (one round trip for 32 chunks)
    for (int64_t i0 = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i0 < n_items; i0 += 32 * nw) {
        const int64_t ij = i0 + (int64_t)lane * nw;
        int64_t cj = 0;
        unsigned lo = ~0u, hi = ~0u;
        if (ij < n_items) {
            cj = listed ? (int64_t)p.chunk_list[ij] : ij;
            if (!all) {
                lo = __ldcg(p.vis0 + 2 * cj) | __ldcg(p.vis1 + 2 * cj);
                hi = __ldcg(p.vis0 + 2 * cj + 1) | __ldcg(p.vis1 + 2 * cj + 1);
            }
        }
        const int nj = (int)min((int64_t)32, (n_items - i0 + nw - 1) / nw);
        if (!all && i0 == 0 && lane == 0) {  // the walk table's stand-in row: sigma -1 (deferral)
            const unsigned long long sb = (unsigned long long)__double_as_longlong(-1.0);
            float4 *o = p.rec[0] + (p.n_leaves + 1) * p.rec4 - 1;
            *o = make_float4(0.f, 0.f, __uint_as_float((unsigned)(sb & 0xffffffffu)), __uint_as_float((unsigned)(sb >> 32)));
        }
#pragma unroll 1
        for (int j = 0; j < nj; ++j) {
            const int64_t c = __shfl_sync(0xffffffffu, cj, j);
            const uint64_t vm = ((uint64_t)__shfl_sync(0xffffffffu, hi, j) << 32) | __shfl_sync(0xffffffffu, lo, j);
            const int64_t base = c * 64;
            const int rows = (int)min((int64_t)64, p.n_leaves - base);
            if (!all && !vm) continue;  // no leaf of the set: the walk table hides the chunk's leaves
            double sp[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {  // both leaves' w_sigma loads in flight together
                const int r = lane + 32 * u;
                sp[u] = r < rows && (all || ((vm >> r) & 1ull))
                            ? sigma_pre_batched<2>(p.T.sig + base + r, p.T.lstride, sA, p.T.C, p.mS) : 0.0;
            }
#pragma unroll 1
            for (int u = 0; u < 2; ++u) {
                const int r = lane + 32 * u;
                if (r >= rows) continue;
                const int64_t L = base + r;
                if (p.lit) p.lit[L] = sp[u] > 0.0 ? 1u : 0u;
                if (lit_only ? sp[u] > 0.0 : ((vm >> r) & 1ull)) {
                    float q[4 * R4];
#pragma unroll
                    for (int k = 0; k < 4 * R4; ++k) q[k] = 0.0f;
                    float wh[4 * Basis<NMAX>::HH4];
                    load_hh<NMAX>(p.T.hh + L * p.T.hh4, wh);  // in flight with the gamma chunks
                    const float s = gamma_s_batched<2>(p.T.gam + L, p.T.lstride, sB, p.T.C, p.mG);
                    float R[Basis<NMAX>::NPAIRS];
                    radial<NMAX>(s, p.K, R);
#pragma unroll
                    for (int l = 0; l <= NMAX; ++l)
#pragma unroll
                        for (int m = -l; m <= l; ++m) {
                            const int jj = l * l + l + m;
                            slice_col<NMAX>(R, wh, l, m, q[3 * jj + 0], q[3 * jj + 1], q[3 * jj + 2]);
                        }
                    const double sigma = sp[u] > 0.0 ? sp[u] : 0.0;
                    const unsigned long long sb = (unsigned long long)__double_as_longlong(sigma);
                    q[4 * R4 - 2] = __uint_as_float((unsigned)(sb & 0xffffffffu));
                    q[4 * R4 - 1] = __uint_as_float((unsigned)(sb >> 32));
                    float4 *o = p.rec[0] + L * p.rec4;
#pragma unroll
                    for (int k = 0; k < R4; ++k) o[k] = make_float4(q[4 * k], q[4 * k + 1], q[4 * k + 2], q[4 * k + 3]);
                } else if (all) {  // (outside the set: no record -- the walk table hides the leaf)
                    const double sigma = sp[u] > 0.0 ? -sp[u] : 0.0;
                    const unsigned long long sb = (unsigned long long)__double_as_longlong(sigma);
                    float4 *o = p.rec[0] + (L + 1) * p.rec4 - TAIL;
#pragma unroll
                    for (int k = 0; k < TAIL - 1; ++k) o[k] = make_float4(0.f, 0.f, 0.f, 0.f);
                    o[TAIL - 1] = make_float4(0.f, 0.f, __uint_as_float((unsigned)(sb & 0xffffffffu)),
                                              __uint_as_float((unsigned)(sb >> 32)));
                }
            }
        }
    }
}

// Lit pass, phase 1 (dark-heavy trees): a thread per leaf computes sigma
// (f64, as k_build_slice), writes the node mask's lit byte, lists a lit leaf
// for phase 2 (k_slice_leaves over the list: its whole record) and gives a
// dark leaf its sigma pair (0) unless the walks cannot read it.  Light and
// bandwidth-bound; the colour work, a tenth of the leaves at cfg3, then runs
// with every lane busy.
template <int NMAX>  // (unused: one instantiation per n_max like the other slice kernels)
__global__ void __launch_bounds__(256) k_slice_lit(const __grid_constant__ SliceParams p) {
    __shared__ float sA[kMaxC], sB[kMaxC];
    load_rows(p.T, p.frame[0], sA, sB);
    __syncthreads();
    pdl_trigger();
    pdl_wait();  // records / lit bytes / the list counter / a region's chunk list: earlier work's
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;  // a multiple of 32
    // a region: the leaves of its listed 64-leaf chunks
    const bool listed = p.chunk_list != nullptr;
    const int64_t n_items = listed ? 64 * (int64_t)*(volatile const int32_t *)p.n_list : p.n_leaves;
    for (int64_t b0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); b0 < n_items; b0 += stride) {
        const int64_t it = b0 + lane;
        int64_t L = it;
        if (listed && it < n_items) L = 64 * (int64_t)__ldg(p.chunk_list + (it >> 6)) + (it & 63);
        const bool in = it < n_items && L < p.n_leaves;
        double sp = 0.0;
        if (in) sp = sigma_pre_batched<2>(p.T.sig + L, p.T.lstride, sA, p.T.C, p.mS);
        const bool lit = in && sp > 0.0;
        const unsigned m = __ballot_sync(0xffffffffu, lit);
        int base = 0;
        if (lane == 0 && m) base = atomicAdd(p.lit_n, __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (!in) continue;
        if (p.lit) p.lit[L] = lit ? 1u : 0u;
        if (lit) {
            p.lit_list[base + __popc(m & ((1u << lane) - 1u))] = (int32_t)L;
        } else if (!p.dark_unread) {  // sigma 0 (two float4: the record's last sector)
            float4 *o = p.rec[0] + (L + 1) * p.rec4 - 2;
            o[0] = make_float4(0.f, 0.f, 0.f, 0.f);
            o[1] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
}

// Visible-set slice with a walk table: a thread per leaf of the set (the
// list k_vis_table wrote), its whole record decoded exactly as in
// k_slice_visible; plus the walk table's stand-in row (sigma -1).  Every
// lane works, where a chunk-per-warp pass left the lanes of the set's
// sparse chunks idle.
template <int NMAX>
__global__ void __launch_bounds__(VV_VIS_BLOCK, NMAX >= 3 ? 4 : VV_VIS_MINB)
    k_slice_leaves(const __grid_constant__ SliceParams p) {
    __shared__ float sA[kMaxC], sB[kMaxC];
    load_rows(p.T, p.frame[0], sA, sB);
    __syncthreads();
    constexpr int R4 = slice_rec4(Basis<NMAX>::S);
    pdl_trigger();
    pdl_wait();  // the list is the previous kernel's
    const int64_t n = (int64_t)*(volatile const int32_t *)p.n_leaf_list;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t0 == 0 && !p.lit_list) {  // the walk table's stand-in row (not in the lit pass)
        const unsigned long long sb = (unsigned long long)__double_as_longlong(-1.0);
        float4 *o = p.rec[0] + (p.n_leaves + 1) * p.rec4 - 1;
        *o = make_float4(0.f, 0.f, __uint_as_float((unsigned)(sb & 0xffffffffu)), __uint_as_float((unsigned)(sb >> 32)));
    }
#pragma unroll 1
    for (int64_t i = t0; i < n; i += stride) {
        const int64_t L = __ldg(p.leaf_list + i);
        if (p.chunk_bits && !((__ldg(p.chunk_bits + (L >> 11)) >> ((L >> 6) & 31)) & 1u)) continue;
        float wh[4 * Basis<NMAX>::HH4];
        load_hh<NMAX>(p.T.hh + L * p.T.hh4, wh);  // in flight with the sigma and gamma chunks
        const double sp = sigma_pre_batched<2>(p.T.sig + L, p.T.lstride, sA, p.T.C, p.mS);
        const float s = gamma_s_batched<2>(p.T.gam + L, p.T.lstride, sB, p.T.C, p.mG);
        float q[4 * R4];
#pragma unroll
        for (int k = 0; k < 4 * R4; ++k) q[k] = 0.0f;
        float R[Basis<NMAX>::NPAIRS];
        radial<NMAX>(s, p.K, R);
#pragma unroll
        for (int l = 0; l <= NMAX; ++l)
#pragma unroll
            for (int m = -l; m <= l; ++m) {
                const int jj = l * l + l + m;
                slice_col<NMAX>(R, wh, l, m, q[3 * jj + 0], q[3 * jj + 1], q[3 * jj + 2]);
            }
        const double sigma = sp > 0.0 ? sp : 0.0;
        const unsigned long long sb = (unsigned long long)__double_as_longlong(sigma);
        q[4 * R4 - 2] = __uint_as_float((unsigned)(sb & 0xffffffffu));
        q[4 * R4 - 1] = __uint_as_float((unsigned)(sb >> 32));
        float4 *o = p.rec[0] + L * p.rec4;
#pragma unroll
        for (int k = 0; k < R4; ++k) o[k] = make_float4(q[4 * k], q[4 * k + 1], q[4 * k + 2], q[4 * k + 3]);
    }
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
    Ray ray;
    const bool hit = ray_setup(p.T, p.origins[3 * r], p.origins[3 * r + 1], p.origins[3 * r + 2],
                               p.dirs[3 * r], p.dirs[3 * r + 1], p.dirs[3 * r + 2], p.tmin, p.tmax, ray);
    if (COLLECT) {
        const int64_t b = p.ray_start[r];
        CollectVisitor v{{}, p.T.leaf_ref, p.seg_leaf + b, p.seg_t0 + b, p.seg_t1 + b, 0, p.ray_start[r + 1] - b};
        if (hit) traverse<Entry>(p.T.child, p.T.depth, ray, smem_raw, v);
    } else {
        CountVisitor v;
        if (hit) traverse<Entry>(p.T.child, p.T.depth, ray, smem_raw, v);
        p.count[r] = v.count;
    }
}

// ------------------------------------------------------------------ paint query
// Termination voxel of compose.paint (compose.py:482-532): walk all leaf
// segments of the ray (ray_segments, octree.py:296-326) and return the
// first leaf where accumulated alpha reaches the threshold, else -1.
// sigma = max(0, w_sigma . A[frame]) in f64 (sequential; the reference
// uses numpy's matmul -- equal to within an ulp), delta = (t1 - t0) * |d|
// with |d| from the host (np.linalg.norm, as ray_segments).
struct TermParams {
    TreeView T;
    int frame;
    const double *origins, *dirs, *norms;
    int64_t n;
    double thr;
    int64_t *out_leaf;
};

struct TerminateVisitor : NoChecks {
    static constexpr int kSegMin = VV_SEG_MIN, kSegSlots = VV_SEG_SLOTS;
    static constexpr bool kPops = false;
    const TreeView &T;
    const float *sA;
    double norm, thr;
    uint32_t mA;
    double acc = 0.0, trans = 1.0;
    int64_t hit = -1;
    __device__ __forceinline__ TerminateVisitor(const TreeView &T_, const float *sA_, double norm_, double thr_)
        : T(T_), sA(sA_), norm(norm_), thr(thr_), mA(nz_chunks(sA_, T_.C)) {}
    __device__ __forceinline__ void pop() {}
    __device__ __forceinline__ int pop_count() const { return 0; }
    __device__ __forceinline__ bool batch(const SegBuf &seg, int n) {
        for (int s = 0; s < n; ++s) {
            const uint32_t L = (uint32_t)seg.leaf_at(s);
            const double sp = sigma_pre(T.sig + L, T.lstride, sA, T.C, mA);
            const double sigma = sp > 0.0 ? sp : 0.0;
            const double delta = xmul(xsub(seg.t1_at(s), seg.t0_at(s)), norm);
            const double a = xsub(1.0, exp(xmul(-sigma, delta)));
            acc = xadd(acc, xmul(trans, a));
            trans = xmul(trans, xsub(1.0, a));
            if (acc >= thr) {
                hit = ref_row(T.leaf_ref, L);
                return true;
            }
        }
        return false;
    }
};

template <class Entry>
__global__ void __launch_bounds__(kBlock) k_terminate(const __grid_constant__ TermParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ float sA[kMaxC];
    for (int c = threadIdx.x; c < kMaxC; c += blockDim.x)
        sA[c] = c < p.T.C ? p.T.basis_a[(size_t)p.frame * p.T.C + c] : 0.0f;
    __syncthreads();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= p.n) return;
    Ray ray;
    const bool hit = ray_setup(p.T, p.origins[3 * r], p.origins[3 * r + 1], p.origins[3 * r + 2],
                               p.dirs[3 * r], p.dirs[3 * r + 1], p.dirs[3 * r + 2], 0.0, 1e30, ray);
    TerminateVisitor v(p.T, sA, p.norms[r], p.thr);
    if (hit) traverse<Entry>(p.T.child, p.T.depth, ray, smem_raw, v);
    p.out_leaf[r] = v.hit;
}

// ------------------------------------------------------------------ dispatch helpers
template <class F>
inline int with_nmax(int nmax, F &&f) {
    switch (nmax) {
        case 0: return f(std::integral_constant<int, 0>());
        case 1: return f(std::integral_constant<int, 1>());
        case 2: return f(std::integral_constant<int, 2>());
        case 3: return f(std::integral_constant<int, 3>());
        default: return set_error(VV_E_UNSUPPORTED, "n_max %d not supported on device (max 3)", nmax);
    }
}

// traversal shared memory per block: segment queues + stacks (traverse());
// pops: the visitor queues node-visit counts (k_render_rays)
inline size_t stack_bytes(int depth, bool wide, bool pops = false, int threads = kBlock, int slots = kSegSlots) {
    return (size_t)threads * (seg_bytes_per_thread(pops, slots) +
                              (size_t)stack_cap(depth) * (wide ? EntryW::kBytes : EntryN::kBytes));
}

template <class Kern>
inline int prep_smem(Kern k, size_t smem) {
    // opt in beyond 48 KB per block: the limit covers static + dynamic
    // shared memory (the scene kernel stages 8 KB of basis rows statically)
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k);
    if (e != cudaSuccess) return set_error(VV_E_CUDA, "function attributes: %s", cudaGetErrorString(e));
    if (smem + fa.sharedSizeBytes > 48 * 1024 && (int)smem > fa.maxDynamicSharedSizeBytes) {
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return set_error(VV_E_CUDA, "smem attribute: %s", cudaGetErrorString(e));
    }
    return VV_OK;
}

#ifndef VV_PDL
#define VV_PDL 1  // launch the slice pass and the camera kernel with programmatic serialization
#endif
// kernel<<<grid, block, smem, st>>>(args...), with programmatic stream
// serialization when VV_PDL (the kernel must pdl_wait() before dependent
// accesses).
// Invariant the PDL prologues rely on: a tree's node table, payload planes
// and basis rows are immutable once vv_tree_upload/bind/voct_upload has
// returned, and every in-place writer of tree state (the repack at upload,
// vv_tree_set_edits) ends with cudaDeviceSynchronize -- so the only tree
// reads issued before griddepcontrol.wait (k_build_slice's TMA loads of the
// payload and basis rows, k_render_camera's basis rows) can never race a
// stream-ordered write.  A future stream-ordered tree update must move those
// reads after the wait.  (Per-frame data -- slices, node masks -- is read
// only after it.)
template <class Kern, class... Args>
inline void launch_pdl(Kern k, dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = VV_PDL ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k, args...);
}

inline int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(VV_E_CUDA, "%s launch failed: %s", what, cudaGetErrorString(e));
    return VV_OK;
}

// resident-grid size of a persistent kernel on the current device
template <class Kern>
inline unsigned persistent_grid(Kern k, int block, size_t smem, unsigned max_blocks) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, block, smem) != cudaSuccess || per_sm < 1) {
        cudaGetLastError();
        per_sm = 1;
    }
    const unsigned resident = (unsigned)(sms * per_sm);
    return max_blocks < resident ? max_blocks : resident;
}

// ------------------------------------------------------------------ launchers
// mode: 0 = decode per sample, 1 = frame slice
int launch_rays(int nmax, int mode, bool edits, bool wide, bool visits, const RaysParams &p, unsigned grid,
                size_t smem, cudaStream_t st);
// one block per 32x16 tile (max_blocks = tile count)
int launch_count_dark(const TreeView &T, int frame, uint32_t mS, int64_t n, unsigned long long *count,
                      cudaStream_t st);
// visible-set renders: the walk of the deferred pixels (after launch_camera with vis)
int launch_camera_rewalk(int nmax, bool wide, const CamParams &p, cudaStream_t st);
// vis: the slice is a visible-set slice (p.S.mark set; sliced, no edits)
int launch_camera(int nmax, int mode, bool edits, bool wide, const CamParams &p, unsigned max_blocks, size_t smem,
                  cudaStream_t st, bool long_queue = false, bool vis = false);
int launch_camera_multi(int nmax, int kf, bool edits, bool wide, const CamMultiParams &p, unsigned grid,
                        cudaStream_t st, bool long_queue = false);
int launch_scene(int nmax, bool wide, bool lean, const SceneParams &p, dim3 grid, size_t smem, cudaStream_t st);
// per-sample depth-ordered joint composition (vv_launch_joint.cu)
int launch_scene_joint(int nmax, bool wide, const SceneParams &p, cudaStream_t st);
int launch_slice(int nmax, const SliceParams &p, cudaStream_t st);
// visible-set slice of one frame (k_slice_visible; p.vis0/vis1, or neither:
// every leaf; k_slice_leaves when p.leaf_list is set)
int launch_slice_visible(int nmax, const SliceParams &p, cudaStream_t st);
// per-frame node mask (vv_launch_mask.cu): child table with every child whose
// subtree holds no lit leaf replaced by -1
struct MaskParams {
    const int32_t *child;       // (n_internal, 8) the tree's table
    const int32_t *parent;      // (n_internal) parent node id, -1 at the root
    const int32_t *last;        // last-level internal nodes (children are leaf rows)
    const int32_t *upper;       // the other internal nodes
    int64_t n_last, n_upper, n_internal;
    const uint8_t *lit;         // (n_leaves) from the slice pass
    uint32_t *flag;             // (n_internal) scratch: subtree holds a lit leaf
    int32_t *mask;              // (n_internal, 8) out
};
int launch_node_mask(const MaskParams &p, cudaStream_t st);
// visible-set walk table: the tree's table with every leaf outside the set
// (a snapshot of vis0 | vis1) replaced by the stand-in row, whose slice
// record holds sigma -1 (the walk defers the pixel).  `out` must already
// hold a copy of the table (its upper rows are not rewritten).
struct VisTableParams {
    const int32_t *child;
    const int32_t *last;  // last-level internal nodes
    int64_t n_last;
    const uint32_t *vis0, *vis1;
    int32_t stand_in;
    int32_t *out;
    int32_t *list;     // out: the set's leaf rows (the slice pass's work list), in last-level node order
    int32_t *n_list;   // zeroed before the launch (when the snapshot changed)
    const int32_t *changed;  // nonzero: the snapshot changed (else the table and list stand)
};
int launch_vis_table(const VisTableParams &p, cudaStream_t st);
// out[i] = a[i] | b[i]: the slice's snapshot of the visible set (the table
// and the slice pass both read it, so they agree whatever walks mark meanwhile)
int launch_vis_snapshot(const uint32_t *a, const uint32_t *b, uint32_t *out, int64_t n, cudaStream_t st);
// the same into a kept snapshot: flags[0] = 1 if any word changed (or
// force); the last block then zeroes *n_list for the table pass to refill
int launch_vis_snapshot_diff(const uint32_t *a, const uint32_t *b, uint32_t *snap, int64_t n, bool force,
                             int32_t *flags, int32_t *n_list, cudaStream_t st);
// bits[list[i] / 32] |= 1 << (list[i] % 32) for i < *n (bits zeroed first)
int launch_chunk_bits(const int32_t *list, const int32_t *n, uint32_t *bits, int64_t max_n, cudaStream_t st);
// leaf rows per box of the chunk culling (= the single-frame slice chunk)
constexpr int kRegionChunk = kSliceChunk;
// chunks whose leaf-cell box can project into a pixel rectangle
// (vv_launch_mask.cu): the chunk list of a region render's slice pass
struct CullParams {
    const int4 *box;            // (n_box, 2) inclusive leaf-cell boxes
    int64_t n_box;
    double lo0, lo1, lo2, cell; // tree corner and leaf cell size (world)
    CamView cam;
    double x0, y0, x1, y1;      // pixel-centre extent of the region, margin included
    int32_t *list, *count;
};
int launch_chunk_cull(const CullParams &p, cudaStream_t st);
// coverage of one tree's leaf-chunk boxes as seen by a camera (optionally
// through an instance affine A, 3x4 rows): the CoverView bitmaps
struct CoverParams {
    const int4 *box;
    int64_t n_box;
    double lo0, lo1, lo2, cell;
    CamView cam;
    double A[12];
    int use_A;
    int width, height, words, cw;
    uint32_t *fine;
    uint8_t *coarse;
    int *all;
};
int launch_coverage(const CoverParams &p, cudaStream_t st);
// camera plan (vv_launch_mask.cu): launch order of n blocks, costliest first
// (counting sort on log-scale cost buckets)
int launch_plan_order(uint32_t *cost, int n, int32_t *order, int *counter, cudaStream_t st);
int launch_segments(bool wide, bool collect, const SegParams &p, unsigned grid, size_t smem, cudaStream_t st);
int launch_terminate(bool wide, const TermParams &p, unsigned grid, size_t smem, cudaStream_t st);
int launch_shadow_blur(const float *alpha, int res, const double *weights, int radius, double *tmp, double *out,
                       cudaStream_t st);
struct LightView {  // vv_light (include/voxvid_b200.h)
    double px, py, pz;
    double ga, gb, gc, gd;
    double strength, r0sq, min_scale;
    int cast_shadows, falloff_enabled;
    const double *map;
    int res;
    double w2c[12];
    double fx, fy, cx, cy;
};
int launch_scene_light(const CamView &cam, const float *rgb, const float *alpha, const float *depth, double bg0,
                       double bg1, double bg2, const LightView *lights, int n_lights, float *image, float *lit_rgb,
                       cudaStream_t st);
int launch_repack(const float *src, int64_t rows, int P, int C, int K3, int c4, int hh4, int64_t lstride,
                  int64_t r0, const int32_t *dst_row, float4 *sig, float4 *gam, float4 *hh, cudaStream_t st);
// slice records (device rows) -> sigma (n) f64 / q (n, 3S) f32 in reference row order
int launch_slice_export(const float4 *rec, int rec4, int s3, int64_t n, const int32_t *dev_row, double *sigma,
                        float *q, cudaStream_t st);
int launch_unpack(const float *packed, int width, int height, int tile, int n_shards, int tiles_x, int tiles_total,
                  float *rgb, float *alpha, float *depth, cudaStream_t st);

}  // namespace vvk
