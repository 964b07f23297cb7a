// vv_deferred.cuh -- deferred colour for single-frame camera renders.
//
// render_kernel (kernels.py:539-599) composites  acc += w_i * col_i  with
// w_i = T_i (1 - exp(-sigma_i delta_i)): the weights need sigma alone, and
// each colour col_i = sigmoid(y(dir) . q(leaf_i)) enters the sums only
// through that product.  So one frame renders as
//   1. k_sigma_slice    sigma per leaf (f64, the nonzero chunks only)
//   2. k_walk_deferred  the walk with the weights: alpha and depth final,
//                       (leaf, w) of every shaded sample recorded per ray
//                       (up to `cap`), every shaded leaf stamped
//   3. k_list_stamped   the stamped leaves (19% of them at cfg2: the
//                       others are never reached or occluded)
//   4. k_slice_listed   q of the listed leaves only
//   5. k_colour         per ray: acc += w * sigmoid(y . q) in sample order
//   6. overflow rays (more than `cap` shaded samples) re-render through the
//      per-sample path (k_render_pixels)
// Every quantity is computed with the operations and order of the one-pass
// kernels, so the images are bitwise those of render().
#pragma once

namespace vvk {
using namespace vv;

struct DeferView {
    const double *sig8;  // (n_leaves) max(0, sigma_pre) of the frame
    uint32_t *stamp;     // (n_leaves) == epoch: some ray shades the leaf (per-call, zeroed)
    uint32_t epoch;
    uint32_t *sleaf;     // (cap, n_pix) shaded leaves per ray, in order (sample-major: coalesced)
    double *sw;          // (cap, n_pix) their compositing weights
    int64_t npix;
    double *aacc;        // (n_pix) accumulated alpha (f64, for the colour pass)
    int32_t *count;      // (n_pix) shaded samples per ray (may exceed cap)
    int cap;
};

// The weight half of Shader::leaf (same fp64 operations, same order).
struct DeferShader {
    static constexpr int kSegMin = VV_SEG_MIN, kSegSlots = VV_SEG_SLOTS;
    static constexpr bool kPops = false;
    const DeferView &D;
    double early_stop;
    int64_t slot;
    double trans = 1.0, aacc = 0.0, tacc = 0.0;
    int shaded = 0;
    __device__ __forceinline__ DeferShader(const DeferView &D_, double es, int64_t slot_)
        : D(D_), early_stop(es), slot(slot_) {}
    __device__ __forceinline__ void pop() {}
    __device__ __forceinline__ int pop_count() const { return 0; }
    __device__ __forceinline__ bool batch(const SegBuf &seg, int n) {
        uint32_t L = (uint32_t)seg.leaf_at(0);
        double sg = __ldg(D.sig8 + L);
#pragma unroll 1
        for (int s = 0; s < n; ++s) {
            uint32_t Ln = 0;
            double sgn = 0.0;
            if (s + 1 < n) {
                Ln = (uint32_t)seg.leaf_at(s + 1);
                sgn = __ldg(D.sig8 + Ln);
            }
            if (leaf(L, seg.t0_at(s), seg.t1_at(s), sg)) return true;
            L = Ln;
            sg = sgn;
        }
        return false;
    }
    __device__ __forceinline__ bool leaf(uint32_t L, double tin, double tout, double sigma) {
        if (sigma == 0.0) return false;  // zero optical depth (kernels.py:556-559)
        const double delta = xsub(tout, tin);
        const double e = exp(xmul(-sigma, delta));
        const double a = xsub(1.0, e);
        const double w = xmul(trans, a);
        if (shaded < D.cap) {
            D.sleaf[shaded * D.npix + slot] = L;
            D.sw[shaded * D.npix + slot] = w;
        }
        ++shaded;
        D.stamp[L] = D.epoch;  // every writer stores the same value
        aacc = xadd(aacc, w);
        tacc = xadd(tacc, xmul(xmul(w, 0.5), xadd(tin, tout)));
        trans = xmul(trans, e);
        return trans < early_stop;
    }
};

// Per-call buffers (stream-ordered pool allocations, vv_api.cu) and the
// launch sequence (vv_launch_deferred.cu).
struct DeferBuffers {
    DeferView D;
    double *sig8;         // = D.sig8, written by k_sigma_slice
    uint32_t mS, mG;      // nz_chunks of the frame's A / B rows
    int64_t n_leaves;
    uint32_t *list;       // (n_leaves) stamped leaves
    uint32_t *counters;   // [0] listed leaves, [1] overflow rays (zeroed before the launch)
    uint32_t *ovf;        // (n_pix) overflow rays
    float4 *rec;          // (n_leaves, rec4) q of the listed leaves (record layout)
    int rec4;
};

int launch_deferred(int nmax, bool wide, const CamParams &p, const DeferBuffers &B, unsigned cam_grid,
                    cudaStream_t st);

}  // namespace vvk
