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
