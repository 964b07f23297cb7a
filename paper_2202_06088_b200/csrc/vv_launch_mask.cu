// vv_launch_mask.cu -- per-frame node masks: dark subtrees cut from the walk.
//
// A leaf whose sigma is 0 in a frame is visited but contributes nothing: the
// reference `continue`s before any colour or transmittance update
// (kernels.py:556-559), so T, the accumulators and the early-stop test are
// untouched.  An image render may therefore skip every dark leaf, and every
// internal node whose whole subtree is dark, and produce bitwise the same
// pixels.  After the frame's slice pass (which records, per leaf, whether
// sigma > 0), these kernels rewrite the child table for the frame:
//   k_mask_last   last-level nodes: child = leaf row if the leaf is lit,
//                 else -1; a node with a lit leaf marks itself and walks its
//                 ancestors up (atomicOr; stops at the first already-marked
//                 one, whose marker walked on from there);
//   k_mask_upper  other nodes: child = node id if the child is marked.
// Image kernels (k_render_camera / _multi / _scene / k_render_rays without
// stats) then walk the masked table with unchanged code.  The visit/count
// and segment queries keep walking the tree's own table.
#include <algorithm>

#include "vv_kernels.cuh"

namespace vvk {

__global__ void __launch_bounds__(256) k_mask_last(const __grid_constant__ MaskParams p) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.n_last; i += stride) {
        const int32_t n = __ldg(p.last + i);
        const int4 *row = reinterpret_cast<const int4 *>(p.child) + 2 * (int64_t)n;
        int4 a = __ldg(row), b = __ldg(row + 1);
        int c[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        bool any = false;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const bool keep = c[k] >= 0 && __ldg(p.lit + c[k]) != 0;
            c[k] = keep ? c[k] : -1;
            any |= keep;
        }
        int4 *out = reinterpret_cast<int4 *>(p.mask) + 2 * (int64_t)n;
        out[0] = make_int4(c[0], c[1], c[2], c[3]);
        out[1] = make_int4(c[4], c[5], c[6], c[7]);
        if (any) {
            p.flag[n] = 1u;
            for (int32_t q = __ldg(p.parent + n); q >= 0; q = __ldg(p.parent + q))
                if (atomicOr(p.flag + q, 1u)) break;
        }
    }
}

__global__ void __launch_bounds__(256) k_vis_table(const __grid_constant__ VisTableParams p) {
    if (p.changed && !*(volatile const int32_t *)p.changed) return;  // the kept table and list stand
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;  // a multiple of 32: warps stay whole
    const int lane = threadIdx.x & 31;
    for (int64_t b0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); b0 < p.n_last; b0 += stride) {
        const int64_t i = b0 + lane;
        int c[8];
        unsigned keep = 0;
        int32_t n = -1;
        if (i < p.n_last) {
            n = __ldg(p.last + i);
            const int4 *row = reinterpret_cast<const int4 *>(p.child) + 2 * (int64_t)n;
            const int4 a = __ldg(row), b = __ldg(row + 1);
            c[0] = a.x; c[1] = a.y; c[2] = a.z; c[3] = a.w; c[4] = b.x; c[5] = b.y; c[6] = b.z; c[7] = b.w;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (c[k] < 0) continue;
                // the snapshot (written by the previous kernel, read-only here: L1-cached)
                const uint32_t w = p.vis0 == p.vis1 ? __ldg(p.vis0 + (c[k] >> 5))
                                                    : __ldg(p.vis0 + (c[k] >> 5)) | __ldg(p.vis1 + (c[k] >> 5));
                if ((w >> (c[k] & 31)) & 1u) keep |= 1u << k;
            }
        }
        // the kept leaves go to the work list: one atomic per warp
        const int cnt = __popc(keep);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        int wbase = 0;
        if (lane == 31 && incl) wbase = atomicAdd(p.n_list, incl);
        wbase = __shfl_sync(0xffffffffu, wbase, 31);
        if (n < 0) continue;
        int off = wbase + incl - cnt;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (c[k] < 0) continue;
            if ((keep >> k) & 1u) {
                p.list[off++] = c[k];
            } else {
                c[k] = p.stand_in;
            }
        }
        int4 *out = reinterpret_cast<int4 *>(p.out) + 2 * (int64_t)n;
        out[0] = make_int4(c[0], c[1], c[2], c[3]);
        out[1] = make_int4(c[4], c[5], c[6], c[7]);
    }
}

__global__ void __launch_bounds__(256) k_vis_or(const uint32_t *a, const uint32_t *b, uint32_t *out, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = __ldcg(a + i) | __ldcg(b + i);
}

__global__ void __launch_bounds__(256) k_vis_or_diff(const uint32_t *a, const uint32_t *b, uint32_t *snap, int64_t n,
                                                     int force, int32_t *flags, int32_t *n_list) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    bool diff = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t v = __ldcg(a + i) | __ldcg(b + i);
        if (force || v != snap[i]) {
            snap[i] = v;
            diff = true;
        }
    }
    if (__syncthreads_or(diff) && threadIdx.x == 0) atomicOr(flags, 1);
    // the last block out: a changed set refills the list from zero
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(flags + 1, 1) == (int)gridDim.x - 1 && *(volatile int32_t *)flags) *n_list = 0;
    }
}

int launch_vis_snapshot_diff(const uint32_t *a, const uint32_t *b, uint32_t *snap, int64_t n, bool force,
                             int32_t *flags, int32_t *n_list, cudaStream_t st) {
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 4));
    k_vis_or_diff<<<grid, 256, 0, st>>>(a, b, snap, n, force ? 1 : 0, flags, n_list);
    return check_launch("vis_snapshot_diff");
}

int launch_vis_snapshot(const uint32_t *a, const uint32_t *b, uint32_t *out, int64_t n, cudaStream_t st) {
    if (!n) return VV_OK;
    k_vis_or<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 4), 256, 0, st>>>(a, b, out, n);
    return check_launch("vis_snapshot");
}

__global__ void __launch_bounds__(256) k_chunk_bits(const int32_t *list, const int32_t *n, uint32_t *bits) {
    const int64_t m = *n;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
        const int32_t c = list[i];
        atomicOr(bits + (c >> 5), 1u << (c & 31));
    }
}

int launch_chunk_bits(const int32_t *list, const int32_t *n, uint32_t *bits, int64_t max_n, cudaStream_t st) {
    if (max_n <= 0) return VV_OK;
    k_chunk_bits<<<(unsigned)std::min<int64_t>((max_n + 255) / 256, 148 * 4), 256, 0, st>>>(list, n, bits);
    return check_launch("chunk_bits");
}

int launch_vis_table(const VisTableParams &p, cudaStream_t st) {
    if (!p.n_last) return VV_OK;
    const unsigned grid = (unsigned)std::min<int64_t>((p.n_last + 255) / 256, 148 * 8);
    k_vis_table<<<grid, 256, 0, st>>>(p);
    return check_launch("vis_table");
}

__global__ void __launch_bounds__(256) k_mask_upper(const __grid_constant__ MaskParams p) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.n_upper; i += stride) {
        const int32_t n = __ldg(p.upper + i);
        const int4 *row = reinterpret_cast<const int4 *>(p.child) + 2 * (int64_t)n;
        int4 a = __ldg(row), b = __ldg(row + 1);
        int c[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) c[k] = (c[k] >= 0 && p.flag[c[k]]) ? c[k] : -1;
        int4 *out = reinterpret_cast<int4 *>(p.mask) + 2 * (int64_t)n;
        out[0] = make_int4(c[0], c[1], c[2], c[3]);
        out[1] = make_int4(c[4], c[5], c[6], c[7]);
    }
}

int launch_node_mask(const MaskParams &p, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(p.flag, 0, (size_t)p.n_internal * sizeof(uint32_t), st);
    if (e != cudaSuccess) return set_error(VV_E_CUDA, "node mask memset: %s", cudaGetErrorString(e));
    auto blocks = [](int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)); };
    if (p.n_last) k_mask_last<<<blocks(p.n_last), 256, 0, st>>>(p);
    int rc = check_launch("mask_last");
    if (rc) return rc;
    if (p.n_upper) k_mask_upper<<<blocks(p.n_upper), 256, 0, st>>>(p);
    return check_launch("mask_upper");
}

}  // namespace vvk

// ------------------------------------------------------------ chunk culling
// Region renders (vv_render_camera_region): a ray through pixel centre (u, v)
// can reach a leaf only if (u, v) lies in the projection of the leaf's cell,
// hence in the screen rectangle bounding the projected corners of its
// chunk's cell box.  A chunk is listed when that rectangle (one pixel of
// margin for rounding) meets the region, or when a box corner is not in
// front of the eye (then every pixel may reach it).  Unlisted chunks'
// slice records are never read by the region's rays.
namespace vvk {

__global__ void __launch_bounds__(256) k_chunk_cull(const __grid_constant__ CullParams p) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const CamView &c = p.cam;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < p.n_box; base += stride) {
        const int64_t i = base + threadIdx.x;
        bool keep = false;
        if (i < p.n_box) {
            const int4 lo = __ldg(p.box + 2 * i), hi = __ldg(p.box + 2 * i + 1);
            if (lo.x <= hi.x) {
                double u0 = 1e300, u1 = -1e300, v0 = 1e300, v1 = -1e300;
                bool front = true;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const double px = p.lo0 + p.cell * (double)((k & 1) ? hi.x + 1 : lo.x);
                    const double py = p.lo1 + p.cell * (double)((k & 2) ? hi.y + 1 : lo.y);
                    const double pz = p.lo2 + p.cell * (double)((k & 4) ? hi.z + 1 : lo.z);
                    const double dx = px - c.ox, dy = py - c.oy, dz = pz - c.oz;
                    // camera frame: R^T d (R's columns are the camera axes)
                    const double cx = c.r00 * dx + c.r10 * dy + c.r20 * dz;
                    const double cy = c.r01 * dx + c.r11 * dy + c.r21 * dz;
                    const double cz = c.r02 * dx + c.r12 * dy + c.r22 * dz;
                    front &= cz > 1e-9;
                    const double iz = 1.0 / cz;
                    const double u = c.fx * cx * iz + c.cx, v = c.fy * cy * iz + c.cy;
                    u0 = fmin(u0, u);
                    u1 = fmax(u1, u);
                    v0 = fmin(v0, v);
                    v1 = fmax(v1, v);
                }
                keep = !front || (u1 >= p.x0 && u0 <= p.x1 && v1 >= p.y0 && v0 <= p.y1);
            }
        }
        // warp-aggregated append: one atomic per warp
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        const int lane = threadIdx.x & 31;
        int slot = 0;
        if (lane == 0 && m) slot = atomicAdd(p.count, __popc(m));
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if (keep) p.list[slot + __popc(m & ((1u << lane) - 1u))] = (int32_t)i;
    }
}

int launch_chunk_cull(const CullParams &p, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(p.count, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return set_error(VV_E_CUDA, "chunk cull memset: %s", cudaGetErrorString(e));
    if (p.n_box == 0) return VV_OK;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((p.n_box + 255) / 256, 148 * 8));
    k_chunk_cull<<<blocks, 256, 0, st>>>(p);
    return check_launch("chunk_cull");
}

}  // namespace vvk

// ------------------------------------------------------------ camera plans
// Launch order for the next render of a camera (vv_camera_plan): the blocks
// sorted by the walk cost this render measured, costliest first -- a
// counting sort on 128 log-scale buckets (9% apart; order within a bucket
// is arbitrary).  One CTA: the grids are at most tens of thousands of
// blocks.  The order only schedules work; any permutation renders the same
// pixels.
namespace vvk {

constexpr int kPlanBuckets = 128;

__device__ __forceinline__ int plan_bucket(uint32_t c) {
    return min(kPlanBuckets - 1, (int)(8.0f * __log2f((float)c + 1.0f)));
}

// Launched with PDL right after the render: waits for its costs, lets the
// next frame's kernels start early, and leaves the cost array and the chunk
// counter zeroed for the next render (no memsets on the frame path).
__global__ void __launch_bounds__(1024) k_plan_order(uint32_t *cost, int n, int32_t *order, int *counter) {
    // the costs of this thread's blocks, loaded up front (independent loads;
    // a dependent load per loop turn left the sort latency-bound at ~20 us)
    constexpr int kPer = 24;  // 24 K blocks held in registers (1024 threads: 64 registers); more loop below
    __shared__ int hist[kPlanBuckets], off[kPlanBuckets];
    pdl_trigger();
    pdl_wait();
    for (int i = threadIdx.x; i < kPlanBuckets; i += blockDim.x) hist[i] = 0;
    const int lane = threadIdx.x & 31;
    const int stride = blockDim.x;
    const int n_pad = (n + 31) & ~31;
    int bk[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        const int i = threadIdx.x + u * stride;
        bk[u] = i < n ? plan_bucket(cost[i]) : -1;
    }
    __syncthreads();
    // warp-aggregated: the lanes sharing a bucket add once (most blocks fall
    // into a few buckets; per-lane shared atomics serialise on them)
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        if (threadIdx.x + u * stride - lane >= n_pad) break;  // warp-uniform
        const unsigned same = __match_any_sync(0xffffffffu, bk[u]);
        if (bk[u] >= 0 && lane == __ffs(same) - 1) atomicAdd(&hist[bk[u]], __popc(same));
    }
    for (int i = threadIdx.x + kPer * stride; i < n_pad; i += stride) {
        const int b = i < n ? plan_bucket(cost[i]) : -1;
        const unsigned same = __match_any_sync(0xffffffffu, b);
        if (b >= 0 && lane == __ffs(same) - 1) atomicAdd(&hist[b], __popc(same));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int b = kPlanBuckets - 1; b >= 0; --b) {  // costliest bucket first
            off[b] = s;
            s += hist[b];
        }
    }
    __syncthreads();
    auto place = [&](int i, int b) {
        const unsigned same = __match_any_sync(0xffffffffu, b);
        const int leader = __ffs(same) - 1;
        int base = 0;
        if (b >= 0 && lane == leader) base = atomicAdd(&off[b], __popc(same));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (b >= 0) {
            cost[i] = 0u;
            order[base + __popc(same & ((1u << lane) - 1u))] = i;
        }
    };
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        const int i = threadIdx.x + u * stride;
        if (i - lane >= n_pad) break;
        place(i, bk[u]);
    }
    for (int i = threadIdx.x + kPer * stride; i < n_pad; i += stride) place(i, i < n ? plan_bucket(cost[i]) : -1);
    (void)counter;  // the render kernel's last warp resets the chunk counters
}

int launch_plan_order(uint32_t *cost, int n, int32_t *order, int *counter, cudaStream_t st) {
    if (n <= 0) return VV_OK;
    launch_pdl(k_plan_order, dim3(1), dim3(1024), 0, st, cost, n, order, counter);
    return check_launch("plan_order");
}

}  // namespace vvk

// ------------------------------------------------------------ coverage
// k_coverage: each 64-leaf chunk box -> its 8 corners (through the instance
// affine A when given) -> the camera frame -> the pixel rectangle of their
// projection, widened by one pixel; small rectangles set their pixels'
// bits, large ones (> 1024 pixels) their 16x16 tiles; a corner not in front
// of the eye sets `all`.  A ray through a pixel centre outside every
// rectangle meets no leaf cell (the cells lie in the boxes, a box's
// projection in its corners' rectangle).
namespace vvk {

__global__ void __launch_bounds__(256) k_coverage(const __grid_constant__ CoverParams p) {
    pdl_trigger();
    pdl_wait();  // the bitmaps were zeroed, earlier readers are done
    const CamView &c = p.cam;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.n_box; i += stride) {
        const int4 lo = __ldg(p.box + 2 * i), hi = __ldg(p.box + 2 * i + 1);
        if (lo.x > hi.x) continue;
        double u0 = 1e300, u1 = -1e300, v0 = 1e300, v1 = -1e300;
        bool front = true;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            double px = p.lo0 + p.cell * (double)((k & 1) ? hi.x + 1 : lo.x);
            double py = p.lo1 + p.cell * (double)((k & 2) ? hi.y + 1 : lo.y);
            double pz = p.lo2 + p.cell * (double)((k & 4) ? hi.z + 1 : lo.z);
            if (p.use_A) {
                const double *A = p.A;
                const double qx = A[0] * px + A[1] * py + A[2] * pz + A[3];
                const double qy = A[4] * px + A[5] * py + A[6] * pz + A[7];
                const double qz = A[8] * px + A[9] * py + A[10] * pz + A[11];
                px = qx;
                py = qy;
                pz = qz;
            }
            const double dx = px - c.ox, dy = py - c.oy, dz = pz - c.oz;
            const double cx = c.r00 * dx + c.r10 * dy + c.r20 * dz;
            const double cy = c.r01 * dx + c.r11 * dy + c.r21 * dz;
            const double cz = c.r02 * dx + c.r12 * dy + c.r22 * dz;
            front &= cz > 1e-9;
            const double iz = 1.0 / cz;
            const double u = c.fx * cx * iz + c.cx, v = c.fy * cy * iz + c.cy;
            u0 = fmin(u0, u);
            u1 = fmax(u1, u);
            v0 = fmin(v0, v);
            v1 = fmax(v1, v);
        }
        if (!front) {
            *p.all = 1;
            continue;
        }
        // pixel centres ix + 0.5 in [u0 - 1, u1 + 1]
        const int x0 = (int)fmax(0.0, ceil(fmax(u0, -1e9) - 1.5));
        const int x1 = (int)fmin((double)(p.width - 1), floor(fmin(u1, 1e9) + 0.5));
        const int y0 = (int)fmax(0.0, ceil(fmax(v0, -1e9) - 1.5));
        const int y1 = (int)fmin((double)(p.height - 1), floor(fmin(v1, 1e9) + 0.5));
        if (x0 > x1 || y0 > y1) continue;
        if ((int64_t)(x1 - x0 + 1) * (y1 - y0 + 1) > 1024) {
            for (int ty = y0 >> 4; ty <= (y1 >> 4); ++ty)
                for (int tx = x0 >> 4; tx <= (x1 >> 4); ++tx) p.coarse[(size_t)ty * p.cw + tx] = 1;
            continue;
        }
        for (int y = y0; y <= y1; ++y)
            for (int w = x0 >> 5; w <= (x1 >> 5); ++w) {
                const int a = max(x0, 32 * w) - 32 * w, b = min(x1, 32 * w + 31) - 32 * w;  // bits a..b
                const uint32_t m = (b == 31 ? 0xffffffffu : ((1u << (b + 1)) - 1u)) & ~((1u << a) - 1u);
                atomicOr(p.fine + (size_t)y * p.words + w, m);
            }
    }
}

int launch_coverage(const CoverParams &p, cudaStream_t st) {
    if (p.n_box == 0) return VV_OK;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((p.n_box + 255) / 256, 148 * 8));
    launch_pdl(k_coverage, dim3(blocks), dim3(256), 0, st, p);
    return check_launch("coverage");
}

}  // namespace vvk
