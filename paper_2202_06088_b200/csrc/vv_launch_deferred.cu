// vv_launch_deferred.cu -- deferred-colour camera render (vv_deferred.cuh).
#include "vv_kernels.cuh"

#include "vv_deferred.cuh"

namespace vvk {

// 1. sigma per leaf: max(0, sigma_pre) over the frame's nonzero A chunks
//    (coalesced: thread per leaf, chunk-major planes)
__global__ void k_sigma_slice(const __grid_constant__ TreeView T, int frame, uint32_t mS, int64_t n, double *sig8) {
    __shared__ float sA[kMaxC];
    for (int c = threadIdx.x; c < kMaxC; c += blockDim.x)
        sA[c] = c < T.C ? T.basis_a[(size_t)frame * T.C + c] : 0.0f;
    __syncthreads();
    for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < n; L += (int64_t)gridDim.x * blockDim.x) {
        const double sp = sigma_pre(T.sig + L, T.lstride, sA, T.C, mS);
        sig8[L] = sp > 0.0 ? sp : 0.0;
    }
}

// 2. the walk with the weights (one thread per pixel, camera tiles as in
//    k_render_camera)
template <class Entry>
__global__ void __launch_bounds__(kTileRays, kCamMinBlocks)
    k_walk_deferred(const __grid_constant__ CamParams p, const __grid_constant__ DeferView D) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int x0, y0, lx0, ly0;
    long long my_tile;
    block_origin(p, x0, y0, my_tile, lx0, ly0);
    int dx_, dy_;
    local_pixel((int)threadIdx.x, dx_, dy_);
    const int ix = x0 + dx_, iy = y0 + dy_;
    if (ix >= p.cam.width || iy >= p.cam.height) return;
    const long long slot = (long long)iy * p.cam.width + ix;
    double dx, dy, dz;
    camera_ray(p.cam, ix, iy, dx, dy, dz);
    DeferShader sh(D, p.early_stop, slot);
    Ray ray;
    if (ray_setup(p.T, p.cam.ox, p.cam.oy, p.cam.oz, dx, dy, dz, p.tmin, p.tmax, ray))
        traverse<Entry>(p.T.child, p.T.depth, ray, smem_raw, sh);
    float r, g, b, a, d;
    finalize(0.0, 0.0, 0.0, sh.aacc, sh.tacc, 1.0, false, p.alpha_floor, p.far_plane, r, g, b, a, d);
    if (p.alpha) p.alpha[slot] = a;
    if (p.depth) p.depth[slot] = d;
    D.aacc[slot] = sh.aacc;
    D.count[slot] = sh.shaded;
}

// 3. the stamped leaves, listed (order irrelevant: q is stored per leaf);
//    one atomic per block and round
__global__ void k_list_stamped(const uint32_t *__restrict__ stamp, uint32_t epoch, int64_t n, uint32_t *list,
                               uint32_t *count) {
    __shared__ uint32_t warp_n[32], block_base;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t rounded = (n + stride - 1) / stride * stride;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rounded; i += stride) {
        const bool f = i < n && __ldg(stamp + i) == epoch;
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (lane == 0) warp_n[warp] = (uint32_t)__popc(bal);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t tot = 0;
            for (int w = 0; w < nw; ++w) {
                const uint32_t c = warp_n[w];
                warp_n[w] = tot;
                tot += c;
            }
            block_base = tot ? atomicAdd(count, tot) : 0u;
        }
        __syncthreads();
        if (f) list[block_base + warp_n[warp] + __popc(bal & ((1u << lane) - 1u))] = (uint32_t)i;
        __syncthreads();
    }
}

// 4. q of the listed leaves (k_build_slice's colour half: the same gamma
//    dot, radial profiles and HH->SH slice, in the same order)
template <int NMAX>
__global__ void k_slice_listed(const __grid_constant__ TreeView T, const __grid_constant__ Consts K, int frame,
                               uint32_t mG, const uint32_t *__restrict__ list, const uint32_t *__restrict__ count,
                               float4 *rec, int rec4) {
    __shared__ float sB[kMaxC];
    for (int c = threadIdx.x; c < kMaxC; c += blockDim.x)
        sB[c] = c < T.C ? T.basis_b[(size_t)frame * T.C + c] : 0.0f;
    __syncthreads();
    constexpr int R4 = slice_rec4(Basis<NMAX>::S);
    const uint32_t n = *count;
    const int C = T.C;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t L = __ldg(list + i);
        float gp = 0.0f;
        for (uint32_t m = mG; m; m &= m - 1) {
            const int j = __ffs(m) - 1;
            const float4 g = __ldg(T.gam + (int64_t)j * T.lstride + L);
            const float gw[4] = {g.x, g.y, g.z, g.w};
            const int cc = 4 * j;
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (cc + e < C) gp = __fmaf_rn(sB[cc + e], gw[e], gp);
        }
        float wh[4 * Basis<NMAX>::HH4];
        load_hh<NMAX>(T.hh + (size_t)L * T.hh4, wh);
        float q[4 * R4];
#pragma unroll
        for (int k = 0; k < 4 * R4; ++k) q[k] = 0.0f;
        float R[Basis<NMAX>::NPAIRS];
        radial<NMAX>(sigmoidf_(gp), K, R);
#pragma unroll
        for (int l = 0; l <= NMAX; ++l)
#pragma unroll
            for (int m = -l; m <= l; ++m) {
                const int j = l * l + l + m;
                slice_col<NMAX>(R, wh, l, m, q[3 * j + 0], q[3 * j + 1], q[3 * j + 2]);
            }
        float4 *o = rec + (size_t)L * rec4;
#pragma unroll
        for (int k = 0; k < R4; ++k) o[k] = make_float4(q[4 * k], q[4 * k + 1], q[4 * k + 2], q[4 * k + 3]);
    }
}

// 5. colour: acc += w * sigmoid(y . q) over the ray's recorded samples, in
//    order (Shader::leaf's colour half); rays beyond `cap` are listed for
//    the per-sample fallback
template <int NMAX>
__global__ void k_colour(const __grid_constant__ CamParams p, const __grid_constant__ DeferView D, uint32_t *ovf,
                         uint32_t *n_ovf) {
    const int64_t npix = (int64_t)p.cam.width * p.cam.height;
    const int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pix >= npix) return;
    const int cnt = D.count[pix];
    if (cnt > D.cap) {
        ovf[atomicAdd(n_ovf, 1u)] = (uint32_t)pix;
        return;
    }
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    if (cnt > 0) {
        double dx, dy, dz;
        camera_ray(p.cam, (int)(pix % p.cam.width), (int)(pix / p.cam.width), dx, dy, dz);
        float y[Basis<NMAX>::S];
        sh_basis<NMAX>((float)dx, (float)dy, (float)dz, p.K, y);
        const uint32_t *sl = D.sleaf + pix;
        const double *sw = D.sw + pix;
        constexpr int Q4 = Basis<NMAX>::Q4;
#pragma unroll 1
        for (int i = 0; i < cnt; ++i)  // every record of the ray to L1 first (independent requests)
            prefetch_l1(p.S.row(__ldg(sl + i * D.npix)));
#pragma unroll 1
        for (int i = 0; i < cnt; ++i) {
            const float4 *qr = p.S.row(__ldg(sl + i * D.npix));
            float q[4 * Q4];
#pragma unroll
            for (int k = 0; k < Q4; ++k) {
                const float4 v = __ldg(qr + k);
                q[4 * k + 0] = v.x;
                q[4 * k + 1] = v.y;
                q[4 * k + 2] = v.z;
                q[4 * k + 3] = v.w;
            }
            float c0 = 0.0f, c1 = 0.0f, c2 = 0.0f;
#pragma unroll
            for (int j = 0; j < Basis<NMAX>::S; ++j) {
                c0 = __fmaf_rn(y[j], q[3 * j + 0], c0);
                c1 = __fmaf_rn(y[j], q[3 * j + 1], c1);
                c2 = __fmaf_rn(y[j], q[3 * j + 2], c2);
            }
            const double w = __ldg(sw + i * D.npix);
            acc0 = xadd(acc0, xmul(w, (double)sigmoidf_(c0)));
            acc1 = xadd(acc1, xmul(w, (double)sigmoidf_(c1)));
            acc2 = xadd(acc2, xmul(w, (double)sigmoidf_(c2)));
        }
    }
    float r, g, b, a, d;
    finalize(acc0, acc1, acc2, D.aacc[pix], 0.0, 1.0, false, p.alpha_floor, p.far_plane, r, g, b, a, d);
    if (p.rgb) {
        p.rgb[3 * pix + 0] = r;
        p.rgb[3 * pix + 1] = g;
        p.rgb[3 * pix + 2] = b;
    }
}

// 6. listed pixels through the one-pass per-sample path (rays with more
//    shaded samples than the record holds)
template <int NMAX, class Entry>
__global__ void __launch_bounds__(kBlock) k_render_pixels(const __grid_constant__ CamParams p,
                                                          const uint32_t *__restrict__ list,
                                                          const uint32_t *__restrict__ count) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ float sA[kMaxC], sB[kMaxC];
    load_rows(p.T, p.frame, sA, sB);
    __syncthreads();
    FrameCtx F{sA, sB, p.frame, p.early_stop, p.edit_weight, nz_chunks(sA, p.T.C), nz_chunks(sB, p.T.C)};
    const uint32_t n = *count;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i0 = blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
        const uint32_t i = i0 + threadIdx.x;
        if (i >= n) continue;
        const uint32_t pix = __ldg(list + i);
        const int ix = (int)(pix % (uint32_t)p.cam.width), iy = (int)(pix / (uint32_t)p.cam.width);
        double dx, dy, dz;
        camera_ray(p.cam, ix, iy, dx, dy, dz);
        Shader<NMAX, 0, false, false> sh(p.T, p.S, F, p.K, (float)dx, (float)dy, (float)dz);
        Ray ray;
        if (ray_setup(p.T, p.cam.ox, p.cam.oy, p.cam.oz, dx, dy, dz, p.tmin, p.tmax, ray))
            traverse<Entry>(p.T.child, p.T.depth, ray, smem_raw, sh);
        float r, g, b, a, d;
        finalize(sh.acc0, sh.acc1, sh.acc2, sh.aacc, sh.tacc, 1.0, false, p.alpha_floor, p.far_plane, r, g, b, a, d);
        if (p.rgb) {
            p.rgb[3 * (size_t)pix + 0] = r;
            p.rgb[3 * (size_t)pix + 1] = g;
            p.rgb[3 * (size_t)pix + 2] = b;
        }
        if (p.alpha) p.alpha[pix] = a;
        if (p.depth) p.depth[pix] = d;
    }
}

template <class Entry>
static int go_walk(const CamParams &p, const DeferView &D, unsigned grid, cudaStream_t st) {
    auto kern = k_walk_deferred<Entry>;
    const size_t smem = stack_bytes(p.T.depth, Entry::kBytes == EntryW::kBytes, false, kTileRays);
    int r = prep_smem(kern, smem);
    if (r) return r;
    kern<<<grid, kTileRays, smem, st>>>(p, D);
    return check_launch("walk_deferred");
}

template <int NM, class Entry>
static int go_pixels(const CamParams &p, const uint32_t *list, const uint32_t *count, cudaStream_t st) {
    auto kern = k_render_pixels<NM, Entry>;
    const size_t smem = stack_bytes(p.T.depth, Entry::kBytes == EntryW::kBytes);
    int r = prep_smem(kern, smem);
    if (r) return r;
    kern<<<148, kBlock, smem, st>>>(p, list, count);  // overflow rays are rare: one block per SM loops
    return check_launch("render_pixels");
}

int launch_deferred(int nmax, bool wide, const CamParams &p, const DeferBuffers &B, unsigned cam_grid,
                    cudaStream_t st) {
    const int64_t npix = (int64_t)p.cam.width * p.cam.height;
    k_sigma_slice<<<1184, 256, 0, st>>>(p.T, p.frame, B.mS, B.n_leaves, B.sig8);
    int r = check_launch("sigma_slice");
    if (r) return r;
    r = wide ? go_walk<EntryW>(p, B.D, cam_grid, st) : go_walk<EntryN>(p, B.D, cam_grid, st);
    if (r) return r;
    k_list_stamped<<<1184, 256, 0, st>>>(B.D.stamp, B.D.epoch, B.n_leaves, B.list, B.counters);
    if ((r = check_launch("list_stamped"))) return r;
    r = with_nmax(nmax, [&](auto N) {
        constexpr int NM = decltype(N)::value;
        k_slice_listed<NM><<<1184, 256, 0, st>>>(p.T, p.K, p.frame, B.mG, B.list, B.counters, B.rec, B.rec4);
        int rr = check_launch("slice_listed");
        if (rr) return rr;
        k_colour<NM><<<(unsigned)((npix + 255) / 256), 256, 0, st>>>(p, B.D, B.ovf, B.counters + 1);
        if ((rr = check_launch("colour"))) return rr;
        return wide ? go_pixels<NM, EntryW>(p, B.ovf, B.counters + 1, st)
                    : go_pixels<NM, EntryN>(p, B.ovf, B.counters + 1, st);
    });
    return r;
}

}  // namespace vvk
