// vv_launch_misc.cu -- slice build, traversal-only, repack and tile-unpack launches.
#include <algorithm>

#include "vv_kernels.cuh"

namespace vvk {

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

// ------------------------------------------------------------------ repack
// leaf rows (source stride P floats: [w_sigma (C) | w_gamma (C) | w_hh (K3)])
// r0 .. r0 + rows - 1 -> chunk-major w_sigma / w_gamma planes (float4 chunk
// j of row g at [j * lstride + g], zero padded past C) and the row-major
// w_hh plane (hh4 float4 per row, zero padded past K3)
// (dst_row: reference row -> device row, walk order; null = identity)
__global__ void k_repack(const float *__restrict__ src, int64_t rows, int P, int C, int K3, int c4, int hh4,
                         int64_t lstride, int64_t r0, const int32_t *__restrict__ dst_row, float4 *sig, float4 *gam,
                         float4 *hh) {
    const int64_t planar = 2 * (int64_t)c4 * rows, total = planar + rows * hh4;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        float v[4];
        if (i < planar) {  // row index fastest: coalesced plane writes
            const int pj = (int)(i / rows);
            const int64_t r = i % rows;
            const int j = pj % c4;
            const float *s = src + r * P + (pj < c4 ? 0 : C);
#pragma unroll
            for (int e = 0; e < 4; ++e) v[e] = 4 * j + e < C ? s[4 * j + e] : 0.0f;
            const int64_t g = dst_row ? (int64_t)dst_row[r0 + r] : r0 + r;
            (pj < c4 ? sig : gam)[(int64_t)j * lstride + g] = make_float4(v[0], v[1], v[2], v[3]);
        } else {
            const int64_t k = i - planar, r = k / hh4;
            const int q = (int)(k % hh4);
            const float *s = src + r * P + 2 * C;
#pragma unroll
            for (int e = 0; e < 4; ++e) v[e] = 4 * q + e < K3 ? s[4 * q + e] : 0.0f;
            const int64_t g = dst_row ? (int64_t)dst_row[r0 + r] : r0 + r;
            hh[g * hh4 + q] = make_float4(v[0], v[1], v[2], v[3]);
        }
    }
}


// leaves whose sigma is 0 at `frame` (the tree's dark fraction, estimated at
// upload from a few frames, picks the camera kernel's queue threshold)
__global__ void k_count_dark(const __grid_constant__ TreeView T, int frame, uint32_t mS, int64_t n,
                             unsigned long long *count) {
    __shared__ float sA[kMaxC];
    for (int c = threadIdx.x; c < kMaxC; c += blockDim.x)
        sA[c] = c < T.C ? T.basis_a[(size_t)frame * T.C + c] : 0.0f;
    __syncthreads();
    unsigned long long dark = 0;
    for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < n; L += (int64_t)gridDim.x * blockDim.x)
        dark += sigma_pre(T.sig + L, T.lstride, sA, T.C, mS) > 0.0 ? 0 : 1;
#pragma unroll
    for (int o = 16; o; o >>= 1) dark += __shfl_down_sync(0xffffffffu, dark, o);
    if ((threadIdx.x & 31) == 0 && dark) atomicAdd(count, dark);
}

int launch_count_dark(const TreeView &T, int frame, uint32_t mS, int64_t n, unsigned long long *count,
                      cudaStream_t st) {
    k_count_dark<<<592, 256, 0, st>>>(T, frame, mS, n, count);
    return check_launch("count_dark");
}

template <int NM, int KF>
static int go_slice(const SliceParams &p, cudaStream_t st) {
    constexpr int kChunk = slice_chunk(KF);
    const size_t per_warp =
        2 * slice_stage_floats4(__builtin_popcount(p.mS) + __builtin_popcount(p.mG), p.T.hh4, kChunk) * 16 + 32 +
        slice_out_floats4(KF, slice_rec4(Basis<NM>::S)) * 16;
    const size_t limit = 227 * 1024 - 4096;  // opt-in maximum less the static arrays
    const int nw = (int)std::min<size_t>(kSliceWarps, limit / per_warp);
    if (nw < 1)
        return set_error(VV_E_UNSUPPORTED, "slice stage of %zu bytes per warp exceeds shared memory", per_warp);
    const size_t smem = (size_t)nw * per_warp;
    auto kern = k_build_slice<NM, KF>;
    int r = prep_smem(kern, smem);
    if (r) return r;
    const int64_t chunks = (p.n_leaves + kChunk - 1) / kChunk;
    const unsigned want = (unsigned)((chunks + nw - 1) / nw);
    unsigned grid = persistent_grid(kern, nw * 32, smem, want);
    if (VV_SLICE_BPS > 0) {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        grid = std::min(grid, (unsigned)(VV_SLICE_BPS * sms));
    }
    launch_pdl(kern, dim3(grid), dim3(nw * 32), smem, st, p);
    return check_launch("build_slice");
}

int launch_slice(int nmax, const SliceParams &p, cudaStream_t st) {
    return with_nmax(nmax, [&](auto N) {
        constexpr int NM = decltype(N)::value;
        switch (p.n_frames) {
            case 1: return go_slice<NM, 1>(p, st);
            case 2: return go_slice<NM, 2>(p, st);
            case 3: return go_slice<NM, 3>(p, st);
            case 4: return go_slice<NM, 4>(p, st);
            default: return set_error(VV_E_UNSUPPORTED, "%d frames per slice pass", p.n_frames);
        }
    });
}

int launch_slice_visible(int nmax, const SliceParams &p, cudaStream_t st) {
    if (p.n_frames != 1 || !p.vis0 != !p.vis1)
        return set_error(VV_E_INVALID, "visible-set slice: one frame and both bitmaps (or neither)");
    return with_nmax(nmax, [&](auto N) {
        constexpr int NM = decltype(N)::value;
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int64_t chunks = (p.n_leaves + 63) / 64;
        if (p.lit_list) {  // two-phase lit pass: sigma for every leaf, then the lit leaves' records
            const unsigned g1 = (unsigned)std::max<int64_t>(1, std::min<int64_t>((p.n_leaves + 255) / 256, sms * 16));
            // (a region's n_list lives on the device: the grid covers the whole tree's leaves)
            launch_pdl(k_slice_lit<NM>, dim3(g1), dim3(256), 0, st, p);
            int r = check_launch("slice_lit");
            if (r) return r;
            SliceParams q = p;
            q.leaf_list = p.lit_list;
            q.n_leaf_list = p.lit_n;
            launch_pdl(k_slice_leaves<NM>, dim3((unsigned)(sms * 16)), dim3(VV_VIS_BLOCK), 0, st, q);
            return check_launch("slice_leaves(lit)");
        }
        if (p.leaf_list) {  // a thread per leaf of the set
            launch_pdl(k_slice_leaves<NM>, dim3((unsigned)(sms * 16)), dim3(VV_VIS_BLOCK), 0, st, p);
            return check_launch("slice_leaves");
        }
        constexpr int wpb = VV_VIS_BLOCK / 32;
        const unsigned grid =
            (unsigned)std::max<int64_t>(1, std::min<int64_t>((chunks + wpb - 1) / wpb, (int64_t)sms * 64 / wpb));
        launch_pdl(k_slice_visible<NM>, dim3(grid), dim3(VV_VIS_BLOCK), 0, st, p);
        return check_launch("slice_visible");
    });
}

template <class Entry, bool COLLECT>
static int go_seg(const SegParams &p, unsigned grid, size_t smem, cudaStream_t st) {
    auto kern = k_segments<Entry, COLLECT>;
    int r = prep_smem(kern, smem);
    if (r) return r;
    kern<<<grid, kBlock, smem, st>>>(p);
    return check_launch("segments");
}

int launch_segments(bool wide, bool collect, const SegParams &p, unsigned grid, size_t smem, cudaStream_t st) {
    if (wide) return collect ? go_seg<EntryW, true>(p, grid, smem, st) : go_seg<EntryW, false>(p, grid, smem, st);
    return collect ? go_seg<EntryN, true>(p, grid, smem, st) : go_seg<EntryN, false>(p, grid, smem, st);
}

template <class Entry>
static int go_term(const TermParams &p, unsigned grid, size_t smem, cudaStream_t st) {
    auto kern = k_terminate<Entry>;
    int r = prep_smem(kern, smem);
    if (r) return r;
    kern<<<grid, kBlock, smem, st>>>(p);
    return check_launch("terminate");
}

int launch_terminate(bool wide, const TermParams &p, unsigned grid, size_t smem, cudaStream_t st) {
    return wide ? go_term<EntryW>(p, grid, smem, st) : go_term<EntryN>(p, grid, smem, st);
}

int launch_repack(const float *src, int64_t rows, int P, int C, int K3, int c4, int hh4, int64_t lstride,
                  int64_t r0, const int32_t *dst_row, float4 *sig, float4 *gam, float4 *hh, cudaStream_t st) {
    k_repack<<<1184, 256, 0, st>>>(src, rows, P, C, K3, c4, hh4, lstride, r0, dst_row, sig, gam, hh);
    return check_launch("repack");
}

// FrameSlice export in the reference's row order (build_frame_cache's
// sigma / q arrays, render.py:170-179): record of device row dev_row[r]
__global__ void k_slice_export(const float4 *__restrict__ rec, int rec4, int s3, int64_t n,
                               const int32_t *__restrict__ dev_row, double *sigma, float *q) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = dev_row ? (int64_t)dev_row[r] : r;
        const float *src = reinterpret_cast<const float *>(rec + g * rec4);
        if (sigma) sigma[r] = *reinterpret_cast<const double *>(src + 4 * rec4 - 2);
        if (q)
            for (int i = 0; i < s3; ++i) q[r * s3 + i] = src[i];
    }
}

int launch_slice_export(const float4 *rec, int rec4, int s3, int64_t n, const int32_t *dev_row, double *sigma,
                        float *q, cudaStream_t st) {
    if (n == 0) return VV_OK;
    k_slice_export<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(rec, rec4, s3, n, dev_row,
                                                                                          sigma, q);
    return check_launch("slice_export");
}

int launch_unpack(const float *packed, int width, int height, int tile, int n_shards, int tiles_x, int tiles_total,
                  float *rgb, float *alpha, float *depth, cudaStream_t st) {
    const int64_t npix = (int64_t)width * height;
    k_unpack_tiles<<<(unsigned)((npix + 255) / 256), 256, 0, st>>>(packed, width, height, tile, n_shards, tiles_x,
                                                                      tiles_total, rgb, alpha, depth);
    return check_launch("unpack_tiles");
}

}  // namespace vvk
