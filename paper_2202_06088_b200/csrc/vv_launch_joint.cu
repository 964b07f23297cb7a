// vv_launch_joint.cu -- per-sample depth-ordered joint composition of
// several VOctree instances (north-star kernel 4; render_scene(mode="joint")).
//
// Algorithm 1 (compose.py:373-406, k_render_scene) renders every instance
// to its own layer and blends the layers per pixel by their expected
// depths; that equals joint volume rendering only when the instances'
// volumes do not interleave along a ray.  This kernel renders
// the instances jointly, per sample: every instance walks its own tree
// along its pulled-back ray (render_instance, compose.py:418-440), the
// walks' leaf segments are merged by world depth (t_enter / |d_raw|, ties
// to the earlier instance -- a stable sort of the instances' ordered
// segment lists) and composited once, front to back:
//   tau = sigma * (t1 - t0)  (tree-space length: sigma is per tree unit),
//   a = 1 - exp(-tau), C += T a c, A += T a, T *= exp(-tau),
// which is the reference's own joint oracle (pkg/tests/util.py:205-245,
// joint_segments_oracle); early termination when T < early_stop (0: none,
// as the oracle).  Output: image = C + (1 - A) bg (or C / A unpremultiplied
// for the lighting passes), alpha A, depth = expected world t.
//
// Structure: one warp per block (32 pixels, an 8x4 tile); each lane keeps,
// per instance, a resumable walk (Trav, its own shared-memory stack and a
// 4-slot segment queue filled one last-level node at a time) and merges the
// heads.  Opt-in: the per-lane state of up to kMaxJoint walks lives in local
// memory.
#include "vv_kernels.cuh"

namespace vvk {

constexpr int kMaxJoint = 8;  // instances per joint render

// Visitor of one instance's walk: stop after every last-level node (the
// merge needs only each walk's next segments), no counters.
struct JointVisitor : NoChecks {
    static constexpr int kSegMin = 1, kSegSlots = 4;
    static constexpr bool kPops = false;
    __device__ __forceinline__ void pop() {}
    __device__ __forceinline__ int pop_count() const { return 0; }
};

// sigma (f64) and colour (fp32 -> f64) of leaf L of one instance, as
// Shader::leaf decodes them (kernels.py:539-587), per-sample or sliced
template <int NMAX>
__device__ __forceinline__ double joint_leaf(const InstView &v, const FrameCtx &F, const Consts &K, const float *y,
                                             uint32_t L, double &c0, double &c1, double &c2) {
    constexpr int Q4 = Basis<NMAX>::Q4;
    const TreeView &T = v.T;
    double sigma;
    if (v.S.rec) {
        sigma = v.S.sigma(L);
    } else {
        const double sp = sigma_pre(T.sig + L, T.lstride, F.sA, T.C, F.mA);
        sigma = sp > 0.0 ? sp : 0.0;
    }
    bool edited = false;
    float4 erg = make_float4(0.f, 0.f, 0.f, 0.f);
    if (T.edit_t != nullptr) {
        const int2 et = __ldg(T.edit_t + L);
        if (et.x <= F.frame && F.frame <= et.y) {
            edited = true;
            erg = __ldg(T.edit_rgb + L);
            if ((double)erg.w >= 0.0) sigma = (double)erg.w;
        }
    }
    if (sigma == 0.0) return 0.0;
    float q0 = 0.f, q1 = 0.f, q2 = 0.f;
    if (v.S.rec) {
        float q[4 * Q4];
        const float4 *qr = v.S.row(L);
#pragma unroll
        for (int i = 0; i < Q4; ++i) {
            const float4 x = __ldg(qr + i);
            q[4 * i] = x.x;
            q[4 * i + 1] = x.y;
            q[4 * i + 2] = x.z;
            q[4 * i + 3] = x.w;
        }
#pragma unroll
        for (int j = 0; j < Basis<NMAX>::S; ++j) {
            q0 = __fmaf_rn(y[j], q[3 * j], q0);
            q1 = __fmaf_rn(y[j], q[3 * j + 1], q1);
            q2 = __fmaf_rn(y[j], q[3 * j + 2], q2);
        }
    } else {
        const float s = gamma_s(T.gam + L, T.lstride, F.sB, T.C, F.mB);
        float R[Basis<NMAX>::NPAIRS];
        radial<NMAX>(s, K, R);
        float wh[4 * Basis<NMAX>::HH4];
        load_hh<NMAX>(T.hh + (size_t)L * T.hh4, wh);
#pragma unroll
        for (int l = 0; l <= NMAX; ++l)
#pragma unroll
            for (int m = -l; m <= l; ++m) {
                const int j = l * l + l + m;
                float a0, a1, a2;
                slice_col<NMAX>(R, wh, l, m, a0, a1, a2);
                q0 = __fmaf_rn(y[j], a0, q0);
                q1 = __fmaf_rn(y[j], a1, q1);
                q2 = __fmaf_rn(y[j], a2, q2);
            }
    }
    c0 = (double)sigmoidf_(q0);
    c1 = (double)sigmoidf_(q1);
    c2 = (double)sigmoidf_(q2);
    if (edited) {  // kernels.py:584-587
        const double ew = F.edit_weight, om = xsub(1.0, ew);
        c0 = xadd(xmul(ew, (double)erg.x), xmul(om, c0));
        c1 = xadd(xmul(ew, (double)erg.y), xmul(om, c1));
        c2 = xadd(xmul(ew, (double)erg.z), xmul(om, c2));
    }
    return sigma;
}

template <int NMAX, class Entry>
__global__ void __launch_bounds__(32) k_render_scene_joint(const __grid_constant__ SceneParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ float sA[kMaxJoint][kMaxC], sB[kMaxJoint][kMaxC];
    __shared__ uint32_t sM[kMaxJoint][2];
    for (int i = 0; i < p.n_inst; ++i) load_rows(p.inst[i].T, p.inst[i].frame, sA[i], sB[i]);
    __syncwarp();
    if ((int)threadIdx.x < p.n_inst) {
        sM[threadIdx.x][0] = nz_chunks(sA[threadIdx.x], p.inst[threadIdx.x].T.C);
        sM[threadIdx.x][1] = nz_chunks(sB[threadIdx.x], p.inst[threadIdx.x].T.C);
    }
    __syncwarp();
    const int lane = threadIdx.x;
    const int ix = blockIdx.x * 8 + (lane & 7), iy = blockIdx.y * 4 + (lane >> 3);
    const bool inside = ix < p.cam.width && iy < p.cam.height;
    double cdx = 0, cdy = 0, cdz = 1;
    if (inside) camera_ray(p.cam, ix, iy, cdx, cdy, cdz);

    // per-instance walk state (local memory: indexed by the merge)
    Trav<Entry> tv[kMaxJoint];
    Ray rays[kMaxJoint];
    SegBuf seg[kMaxJoint];
    float dirs[kMaxJoint][3];
    double scale[kMaxJoint];  // world t per tree-space t (1 / |d_raw|)
    int head[kMaxJoint], cnt[kMaxJoint];
    bool live[kMaxJoint];
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t seg_b = 32u * seg_bytes_per_thread(false, JointVisitor::kSegSlots);
    const uint32_t stack_b = 32u * (uint32_t)stack_cap(p.max_depth) * Entry::kBytes;
    JointVisitor vis;
    for (int i = 0; i < p.n_inst; ++i) {
        const InstView &v = p.inst[i];
        const uint32_t base = sbase + (uint32_t)i * (seg_b + stack_b);
        seg[i].init(base, 32, lane, JointVisitor::kSegSlots);
        double ox, oy, oz, dx, dy, dz, sc = 1.0;
        if (v.mode == 0) {
            camera_ray(v.cam, ix, iy, dx, dy, dz);
            ox = v.cam.ox;
            oy = v.cam.oy;
            oz = v.cam.oz;
        } else {
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
            sc = xdiv(1.0, nrm);
        }
        scale[i] = sc;
        dirs[i][0] = (float)dx;
        dirs[i][1] = (float)dy;
        dirs[i][2] = (float)dz;
        live[i] = inside && ray_setup(v.T, ox, oy, oz, dx, dy, dz, p.tmin, p.tmax, rays[i]);
        if (live[i]) tv[i].init(rays[i], base + seg_b + (uint32_t)lane * Entry::kBytes);
        head[i] = cnt[i] = 0;
    }
    const uint32_t stride = 32u * Entry::kBytes;
    float y[kMaxJoint][16];
    bool y_ready[kMaxJoint];
    for (int i = 0; i < p.n_inst; ++i) y_ready[i] = false;
    double trans = 1.0, acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, aacc = 0.0, tacc = 0.0;
    while (true) {
        // refill drained queues; pick the nearest head (ties: lower instance)
        int best = -1;
        double bt = 0.0;
        for (int i = 0; i < p.n_inst; ++i) {
            if (!live[i]) continue;
            if (head[i] == cnt[i]) {
                const InstView &v = p.inst[i];
                const uint32_t stack_base = sbase + (uint32_t)i * (seg_b + stack_b) + seg_b + (uint32_t)lane * Entry::kBytes;
                cnt[i] = trav_next(tv[i], v.T.child, v.T.depth, rays[i], stack_base, stride, vis, seg[i]);
                head[i] = 0;
                if (cnt[i] == 0) {
                    live[i] = false;
                    continue;
                }
            }
            const double tw = xmul(seg[i].t0_at(head[i]), scale[i]);
            if (best < 0 || tw < bt) {
                best = i;
                bt = tw;
            }
        }
        if (best < 0) break;
        const int k = best;
        const InstView &v = p.inst[k];
        const uint32_t L = (uint32_t)seg[k].leaf_at(head[k]);
        const double t0 = seg[k].t0_at(head[k]), t1 = seg[k].t1_at(head[k]);
        ++head[k];
        if (!y_ready[k]) {
            sh_basis<NMAX>(dirs[k][0], dirs[k][1], dirs[k][2], p.K, y[k]);
            y_ready[k] = true;
        }
        const FrameCtx F{sA[k], sB[k], v.frame, p.early_stop, p.edit_weight, sM[k][0], sM[k][1]};
        double c0, c1, c2;
        const double sigma = joint_leaf<NMAX>(v, F, p.K, y[k], L, c0, c1, c2);
        if (sigma == 0.0) continue;
        const double e = exp(xmul(-sigma, xsub(t1, t0)));
        const double w = xmul(trans, xsub(1.0, e));
        acc0 = xadd(acc0, xmul(w, c0));
        acc1 = xadd(acc1, xmul(w, c1));
        acc2 = xadd(acc2, xmul(w, c2));
        aacc = xadd(aacc, w);
        tacc = xadd(tacc, xmul(xmul(w, 0.5), xmul(xadd(t0, t1), scale[k])));
        trans = xmul(trans, e);
        if (trans < p.early_stop) break;
    }
    if (!inside) return;
    const int64_t pix = (int64_t)iy * p.cam.width + ix;
    const double safe = aacc > 1e-300 ? aacc : 1e-300;
    if (p.image && p.composite) {  // C + (1 - A) bg (premultiplied joint colour)
        const double om = xsub(1.0, aacc);
        p.image[3 * pix + 0] = (float)xadd(acc0, xmul(om, p.bg0));
        p.image[3 * pix + 1] = (float)xadd(acc1, xmul(om, p.bg1));
        p.image[3 * pix + 2] = (float)xadd(acc2, xmul(om, p.bg2));
    } else if (p.image) {  // unpremultiplied, for the lighting passes
        p.image[3 * pix + 0] = aacc > 0.0 ? (float)xdiv(acc0, safe) : 0.0f;
        p.image[3 * pix + 1] = aacc > 0.0 ? (float)xdiv(acc1, safe) : 0.0f;
        p.image[3 * pix + 2] = aacc > 0.0 ? (float)xdiv(acc2, safe) : 0.0f;
    }
    if (p.alpha) p.alpha[pix] = (float)aacc;
    if (p.depth) p.depth[pix] = (float)(aacc >= p.alpha_floor ? xdiv(tacc, safe) : p.far_plane);
}

template <int NM, class Entry>
static int go_joint(const SceneParams &p, cudaStream_t st) {
    auto kern = k_render_scene_joint<NM, Entry>;
    const size_t smem = (size_t)p.n_inst * 32 *
                        (seg_bytes_per_thread(false, JointVisitor::kSegSlots) + stack_cap(p.max_depth) * Entry::kBytes);
    int r = prep_smem(kern, smem);
    if (r) return r;
    dim3 grid((unsigned)((p.cam.width + 7) / 8), (unsigned)((p.cam.height + 3) / 4));
    kern<<<grid, 32, smem, st>>>(p);
    return check_launch("render_scene_joint");
}

int launch_scene_joint(int nmax, bool wide, const SceneParams &p, cudaStream_t st) {
    if (p.n_inst > kMaxJoint)
        return set_error(VV_E_UNSUPPORTED, "at most %d instances per joint render", kMaxJoint);
    return with_nmax(nmax, [&](auto N) {
        constexpr int NM = decltype(N)::value;
        return wide ? go_joint<NM, EntryW>(p, st) : go_joint<NM, EntryN>(p, st);
    });
}

}  // namespace vvk
