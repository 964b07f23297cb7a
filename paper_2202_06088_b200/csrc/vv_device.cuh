// vv_device.cuh -- device-side building blocks of the B200 VOctree renderer.
//
// One CUDA thread owns one ray.  The ray walks the BFS node table with the
// reference's parametric near-to-far descent (kernels.py:171-310, 600-647)
// and shades leaf segments as they are reached (kernels.py:539-599), so the
// early-termination test also ends the tree walk.
//
// Numerics:
//   * ray normalisation, plane crossings, sigma decode, transmittance, alpha
//     and tbar are float64 with explicit round-to-nearest intrinsics (no FMA
//     contraction) in the reference's operation order -> visited leaves,
//     segment t values, sample counts and alpha are bit-exact with
//     voxvid.kernels.render_kernel (modulo 1-ulp exp() differences);
//   * the hyper-angle decode, HH radial profiles, SH basis, HH->SH slice and
//     colour sigmoid run in fp32 (tolerance 1e-4 in the contract).
//
// Differences in mechanism (not in results) from the reference:
//   * the stack holds only (node id, level, cell coords) -- 8 bytes -- in
//     shared memory; a popped cell's [t_in, t_out] is recomputed from its six
//     boundary planes.  Every boundary plane of a cell is a mid plane of an
//     ancestor (or a root face), so the recomputed crossings are the very
//     values the reference carried on its stack (proof sketch in DESIGN.md);
//   * the nearest child continues in registers instead of push+pop, and the
//     <= 4 leaves of a last-level node are shaded straight from registers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace vv {

constexpr int kMaxC = 64;       // max temporal basis count C supported on device
constexpr int kMaxNmax = 3;     // HH truncation supported on device
constexpr int kMaxDepth = 20;   // leaf depth supported on device
constexpr int kNarrowDepth = 9; // depth <= 9 packs a stack entry in 8 bytes

template <int NMAX> struct Basis {
    static constexpr int S = (NMAX + 1) * (NMAX + 1);            // SH count
    static constexpr int K = (NMAX + 1) * (NMAX + 2) * (2 * NMAX + 3) / 6;  // HH count
    static constexpr int NPAIRS = (NMAX + 1) * (NMAX + 2) / 2;
    static constexpr int HH4 = (3 * K + 3) / 4;                  // float4 per w_hh
    static constexpr int Q4 = (3 * S + 3) / 4;                   // float4 per sliced q
};

// Constants of kernels.basis_tables (A_nl, SH prefactors), fp32.
struct Consts {
    float pair_norm[16];
    float sh_pref[16];
};

// Device-side bounds checks of the debug build (the pool forbids
// compute-sanitizer): a failed check counts a violation instead of trapping.
#ifdef VV_DEBUG_CHECKS
constexpr bool kDebugChecks = true;
#else
constexpr bool kDebugChecks = false;
#endif
enum : unsigned { VV_DBG_NODE = 1, VV_DBG_STACK = 2, VV_DBG_LEAF = 3, VV_DBG_QUEUE = 4, VV_DBG_CHUNK = 5 };
__device__ __forceinline__ void debug_violation(unsigned *dbg, unsigned code) {
    if (dbg) {
        atomicAdd(dbg, 1u);
        atomicCAS(dbg + 1, 0u, code);
    }
}

// Device view of one uploaded tree.
struct TreeView;
__device__ __forceinline__ int64_t ref_row(const int32_t *leaf_ref, uint32_t L) {
    return leaf_ref ? (int64_t)__ldg(leaf_ref + L) : (int64_t)L;
}
struct TreeView {
    const int32_t *child;    // (n_internal, 8)
    // w_sigma / w_gamma chunk-major: float4 chunk j (columns 4j..4j+3, zero
    // padded) of leaf L at [j * lstride + L] -- a frame whose A (B) row is
    // zero over a chunk never reads it, and the chunks it does read are
    // contiguous over consecutive leaves
    const float4 *sig;       // (c4, lstride)
    const float4 *gam;       // (c4, lstride)
    const float4 *hh;        // (n_leaves, hh4): w_hh padded, row-major
    const float4 *edit_rgb;  // (n_leaves) or null
    const int2 *edit_t;      // (n_leaves) or null
    const float *basis_a;    // (T, C)
    const float *basis_b;    // (T, C)
    // Leaf rows on the device are in walk (BFS = Morton) order, not the
    // reference's row order: leaf_ref maps a device row back to the
    // reference row id wherever one leaves the device (visit lists, segment
    // lists, termination leaves); null = identity (tables that are not trees)
    const int32_t *leaf_ref;
    int64_t n_leaves, n_internal;
    // bounds-checked builds (VV_DEBUG_CHECKS, `make debug`): violations
    // counted at dbg[0], first violation's code at dbg[1]; null otherwise
    unsigned *dbg;
    double lo0, lo1, lo2, side;
    // side a power of two: v / side == v * (1 / side) exactly (both are the
    // correctly rounded v * 2^-k), so ray setup multiplies instead of
    // dividing -- 6 of the ray's 14 fp64 divisions
    double inv_side;
    int side_pow2;
    int64_t lstride;         // leaf rows per chunk plane (>= n_leaves)
    int depth, C, c4, hh4, frames, nmax;
};

// Bit j set when the basis row (fp32, C columns) has a nonzero entry among
// columns 4j..4j+3.  The sigma / gamma sums skip the other chunks: their
// products are +-0, and adding +-0 to an accumulator that starts at +0 and
// so is never -0 leaves it bit-identical (finite payloads).
__device__ __forceinline__ uint32_t nz_chunks(const float *row, int C) {
    uint32_t m = 0;
    for (int c = 0; c < C; ++c)
        if (row[c] != 0.0f) m |= 1u << (c >> 2);
    return m;
}

// Per-frame slice: one record per leaf, [q (3S fp32) | pad | sigma (f64)],
// rec4 float4 long -- 128 bytes (one cache line) at n_max = 2.
struct SliceView {
    const float4 *rec;  // (n_leaves, rec4) or null (decode per sample)
    int rec4;           // float4 per record = ceil((3S + 2) / 4)
    // visible-set slices (VIS kernels): records only for the tree's visible
    // set, walked through a table whose other leaves point at a stand-in
    // record with sigma -1 (vv_api.cu, vis_prepare).  A walk that meets a
    // negative sigma stops and the pixel is walked again per sample
    // (k_camera_rewalk), marking the leaves it visits in `mark`; a census
    // walk (VIS 3) marks every leaf it visits.
    int census;
    uint32_t *mark;
    __device__ __forceinline__ const float4 *row(uint32_t L) const { return rec + (size_t)L * rec4; }
    __device__ __forceinline__ double sigma(uint32_t L) const {
        return __ldg(reinterpret_cast<const double *>(rec + (size_t)(L + 1) * rec4) - 1);
    }
};
__host__ __device__ constexpr int slice_rec4(int S) { return (3 * S + 2 + 3) / 4; }

// ------------------------------------------------------------ fp64 helpers
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xdiv(double a, double b) { return __ddiv_rn(a, b); }
// Python builtin max/min of two floats (first argument wins ties)
__device__ __forceinline__ double pmax(double a, double b) { return (b > a) ? b : a; }
__device__ __forceinline__ double pmin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ void prefetch_l1(const void *p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
// ---- programmatic dependent launch: a kernel launched with the
// programmatic-serialization attribute may start while the previous kernel
// on the stream finishes; it does its read-only prologue, then pdl_wait()s
// (the previous grid complete and its memory visible) before touching
// anything that grid or an earlier one produces or may still use.  Both are
// no-ops for a kernel launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }
// ---- TMA bulk copies (cp.async.bulk) completed on an mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        "VV_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra VV_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// exact 2^-k for 0 <= k <= 1022
__device__ __forceinline__ double pow2neg(int k) {
    return __longlong_as_double((long long)(1023 - k) << 52);
}

// ------------------------------------------------------------ ray setup
// kernels.py:482-532 (== _collect_segments 180-236)
struct Ray {
    double o0, o1, o2, i0, i1, i2;
    double rt_in, rt_out;
    int mirror;
};

__device__ __forceinline__ bool ray_setup(const TreeView &T, double ox, double oy, double oz,
                                          double dx, double dy, double dz, double tmin,
                                          double tmax, Ray &r) {
    auto scale = [&](double v) { return T.side_pow2 ? xmul(v, T.inv_side) : xdiv(v, T.side); };
    double o0 = scale(xsub(ox, T.lo0));
    double o1 = scale(xsub(oy, T.lo1));
    double o2 = scale(xsub(oz, T.lo2));
    double d0 = scale(dx);
    double d1 = scale(dy);
    double d2 = scale(dz);
    int mirror = 0;
    if (d0 < 0.0) { o0 = xsub(1.0, o0); d0 = -d0; mirror |= 1; }
    if (d1 < 0.0) { o1 = xsub(1.0, o1); d1 = -d1; mirror |= 2; }
    if (d2 < 0.0) { o2 = xsub(1.0, o2); d2 = -d2; mirror |= 4; }
    bool ok = true;
    double i0, i1, i2;
    if (d0 < 1e-300) { if (o0 < 0.0 || o0 >= 1.0) ok = false; i0 = 1e300; } else i0 = xdiv(1.0, d0);
    if (d1 < 1e-300) { if (o1 < 0.0 || o1 >= 1.0) ok = false; i1 = 1e300; } else i1 = xdiv(1.0, d1);
    if (d2 < 1e-300) { if (o2 < 0.0 || o2 >= 1.0) ok = false; i2 = 1e300; } else i2 = xdiv(1.0, d2);
    r.o0 = o0; r.o1 = o1; r.o2 = o2;
    r.i0 = i0; r.i1 = i1; r.i2 = i2;
    r.mirror = mirror;
    if (!ok) return false;
    r.rt_in = pmax(pmax(xmul(xsub(0.0, o0), i0), xmul(xsub(0.0, o1), i1)),
                   pmax(xmul(xsub(0.0, o2), i2), tmin));
    r.rt_out = pmin(pmin(xmul(xsub(1.0, o0), i0), xmul(xsub(1.0, o1), i1)),
                    pmin(xmul(xsub(1.0, o2), i2), tmax));
    return r.rt_in < r.rt_out;
}

// ------------------------------------------------------------ stack entries
// A cell is identified by its level L and packed coordinates pc.  Packing
// keeps each axis in its own bit field so a child's code is
// (pc << 1) | spread(child bits); the fields never carry into each other.
// narrow (depth <= 9): 8-byte entry {ptr, pc | L << 27}, 9 bits per axis
struct EntryN {
    using Code = uint32_t;
    static constexpr int kShift = 9;
    static constexpr Code kMask = 511u;
    static constexpr uint32_t kBytes = 8;
    __device__ __forceinline__ static Code spread(int b) {
        return (Code)(b & 1) | ((Code)(b & 2) << 8) | ((Code)(b & 4) << 16);
    }
    __device__ __forceinline__ static void store(uint32_t addr, uint32_t ptr, int L, Code pc) {
        asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(ptr), "r"(pc | ((uint32_t)L << 27)));
    }
    __device__ __forceinline__ static void load(uint32_t addr, uint32_t &ptr, int &L, Code &pc) {
        uint32_t c;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(ptr), "=r"(c) : "r"(addr));
        L = (int)(c >> 27);
        pc = c & 0x7FFFFFFu;
    }
};
// wide (depth <= 20): 16-byte entry {ptr, L, pc (64-bit)}, 21 bits per axis
struct EntryW {
    using Code = unsigned long long;
    static constexpr int kShift = 21;
    static constexpr Code kMask = (1ull << 21) - 1;
    static constexpr uint32_t kBytes = 16;
    __device__ __forceinline__ static Code spread(int b) {
        return (Code)(b & 1) | ((Code)(b & 2) << 20) | ((Code)(b & 4) << 40);
    }
    __device__ __forceinline__ static void store(uint32_t addr, uint32_t ptr, int L, Code pc) {
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(ptr), "r"((uint32_t)L),
                     "r"((uint32_t)pc), "r"((uint32_t)(pc >> 32)));
    }
    __device__ __forceinline__ static void load(uint32_t addr, uint32_t &ptr, int &L, Code &pc) {
        uint32_t l, lo, hi;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(ptr), "=r"(l), "=r"(lo), "=r"(hi) : "r"(addr));
        L = (int)l;
        pc = ((Code)hi << 32) | lo;
    }
};

// slots per thread: a level-L node (L <= depth-2; last-level nodes queue
// segments, they do not push) holds <= 3L entries and writes slots up to
// 3L+2, so 3(depth-1) slots suffice.  One slot (8 B/thread) less than the
// looser 3(depth-1)+1 lets four 128-thread camera blocks fit the 196 KB
// shared-memory carveout at depth 9, leaving 60 KB of L1 instead of 28 KB.
__host__ __device__ constexpr int stack_cap(int depth) { return depth <= 1 ? 1 : 3 * (depth - 1); }

// ------------------------------------------------------------ traversal
// Visitor interface:
//   void pop()                                   one internal-node pop
//   int pop_count()                              pops so far (stats)
//   bool batch(const SegBuf &seg, int n)
//        the next n queued leaf segments, near to far: leaf row
//        seg.leaf_at(s) over [seg.t0_at(s), seg.t1_at(s)]; returns true to
//        stop the ray (early termination).
//
// Structure (queued "while-while", see traverse()): a lane walks internal
// nodes, queueing the kept leaves of the last-level nodes it passes, until
// it holds >= kSegMin segments; then the warp shades in lock step.
//
// Node step (kernels.py:600-647 restated): the reference walks the pierced
// children by repeatedly taking the smallest not-yet-crossed mid-plane
// crossing (ties x, y, z) until it reaches the node's exit.  That is a
// stable sort of the (up to three) uncrossed crossings, done here as a rank
// sort with independent comparisons, which yields the same order and the
// same boundary values st[k] = min(k-th crossing, t_out); step k exists
// iff st[k] < t_out, which the 'st[k+1] > st[k]' segment test already
// implies.  Node corners are tracked as exact doubles so crossings need no
// int->double conversion: p_mid = x_lo + h/2 is the same double as the
// reference's (2c+1) * 2^-(L+1).

// Resumable traversal state of one ray.  The stack lives in shared memory
// at a 32-bit shared-window address (one slot per level of pending
// siblings, `stride` bytes between a thread's consecutive slots).
template <class Entry>
struct Trav {
    uint32_t ptr;
    typename Entry::Code pc;  // packed cell coordinates of the current node
    int L;
    uint32_t sp;              // shared address of the next free stack slot
    double xl, yl, zl, h;     // node low corner and size (exact)
    double tin, tout;
    bool need_pop;
    __device__ __forceinline__ void init(const Ray &r, uint32_t stack_base) {
        ptr = 0;
        pc = 0;
        L = 0;
        sp = stack_base;
        xl = yl = zl = 0.0;
        h = 1.0;
        tin = r.rt_in;
        tout = r.rt_out;
        need_pop = false;
    }
};

// Leaf segments queued for shading live in shared memory, structure of
// arrays per slot (consecutive threads -> consecutive words, conflict-free):
// t0, t1, leaf rows, node-visit counts.  A walk queues >= kSegMin segments
// (one last-level node adds up to 4) before the warp shades; the walk may
// so run ahead of an early termination, and the visit count queued with
// each segment restores the reference's count at the terminating one.
#ifndef VV_SEG_MIN
#define VV_SEG_MIN 6
#endif
#ifndef VV_SEG_SLOTS
#define VV_SEG_SLOTS (VV_SEG_MIN + 3)
#endif
constexpr int kSegMin = VV_SEG_MIN;
constexpr int kSegSlots = VV_SEG_SLOTS;
static_assert(kSegSlots >= kSegMin + 3, "a last-level node queues up to 4 segments");
// every visitor declares the queue geometry it walks with (kSegMin,
// kSegSlots); Shader takes it as a parameter: long, mostly dark walks prefer
// a longer queue
// (the visit counts only for visitors that report them, kPops)
__host__ __device__ constexpr uint32_t seg_bytes_per_thread(bool pops, int slots = kSegSlots) {
    return (uint32_t)slots * (pops ? 24u : 20u);
}
struct SegBuf {
    uint32_t t0, t1, leaf, pops;  // shared addresses of this thread's slot 0
    uint32_t sl, sd;              // slot strides (bytes) of the int and double arrays
    __device__ __forceinline__ void init(uint32_t base, int nthreads, int tid, int slots) {
        sl = 4u * nthreads;
        sd = 8u * nthreads;
        t0 = base + 8u * tid;
        t1 = t0 + slots * sd;
        leaf = base + 2 * slots * sd + 4u * tid;
        pops = leaf + slots * sl;
    }
    template <bool POPS>
    __device__ __forceinline__ void put(int s, int32_t L, double a, double b, int np) const {
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(leaf + s * sl), "r"(L));
        asm volatile("st.shared.f64 [%0], %1;" ::"r"(t0 + s * sd), "d"(a));
        asm volatile("st.shared.f64 [%0], %1;" ::"r"(t1 + s * sd), "d"(b));
        if (POPS) asm volatile("st.shared.u32 [%0], %1;" ::"r"(pops + s * sl), "r"(np));
    }
    __device__ __forceinline__ int pops_at(int s) const {
        int v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(pops + s * sl));
        return v;
    }
    __device__ __forceinline__ int32_t leaf_at(int s) const {
        int32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(leaf + s * sl));
        return v;
    }
    __device__ __forceinline__ double t0_at(int s) const {
        double v;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(t0 + s * sd));
        return v;
    }
    __device__ __forceinline__ double t1_at(int s) const {
        double v;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(t1 + s * sd));
        return v;
    }
};

// Advance the walk, queueing the kept leaves of the last-level nodes it
// passes, until >= kSegMin segments are queued or the tree is exhausted;
// returns the number queued (0: done).
template <class Entry, class Visitor>
__device__ __forceinline__ int trav_next(Trav<Entry> &t, const int32_t *__restrict__ child, int depth, const Ray &r,
                                         uint32_t stack_base, uint32_t stride, Visitor &vis, const SegBuf &seg) {
    int n = 0;
    int32_t cp[4];
    double st[5];
    const double o0 = r.o0, o1 = r.o1, o2 = r.o2, i0 = r.i0, i1 = r.i1, i2 = r.i2;
    const int mirror = r.mirror;
    while (true) {
        if (t.need_pop) {
            if (t.sp == stack_base) return n;
            t.sp -= stride;
            Entry::load(t.sp, t.ptr, t.L, t.pc);
            // recompute the popped cell's interval from its six faces
            t.h = pow2neg(t.L);
            t.xl = xmul((double)(uint32_t)(t.pc & Entry::kMask), t.h);
            t.yl = xmul((double)(uint32_t)((t.pc >> Entry::kShift) & Entry::kMask), t.h);
            t.zl = xmul((double)(uint32_t)((t.pc >> (2 * Entry::kShift)) & Entry::kMask), t.h);
            const double xh = xadd(t.xl, t.h), yh = xadd(t.yl, t.h), zh = xadd(t.zl, t.h);
            t.tin = pmax(pmax(r.rt_in, xmul(xsub(t.xl, o0), i0)),
                         pmax(xmul(xsub(t.yl, o1), i1), xmul(xsub(t.zl, o2), i2)));
            t.tout = pmin(pmin(r.rt_out, xmul(xsub(xh, o0), i0)),
                          pmin(xmul(xsub(yh, o1), i1), xmul(xsub(zh, o2), i2)));
            t.need_pop = false;
        }
        vis.pop();
        if (kDebugChecks) vis.check_node(t.ptr, (t.sp - stack_base) / stride);
        const double tin = t.tin, tout = t.tout;
        const double hh = xmul(t.h, 0.5);
        const double txm = xmul(xsub(xadd(t.xl, hh), o0), i0);
        const double tym = xmul(xsub(xadd(t.yl, hh), o1), i1);
        const double tzm = xmul(xsub(xadd(t.zl, hh), o2), i2);
        const bool bx = txm < tin, by = tym < tin, bz = tzm < tin;
        const int b0 = (bx ? 1 : 0) | (by ? 2 : 0) | (bz ? 4 : 0);
        double k0 = bx ? 1e301 : txm, k1 = by ? 1e301 : tym, k2 = bz ? 1e301 : tzm;
        // stable rank sort: the three comparisons are independent (the
        // network below chains them); rank_i = #{j: k_j < k_i} + #{j < i:
        // k_j == k_i} -- the same order, ties to the earlier axis
        const bool l10 = k1 < k0, l20 = k2 < k0, l21 = k2 < k1;
        const int r0 = (int)l10 + (int)l20, r1 = (int)!l10 + (int)l21;
        const double s0 = r0 == 0 ? k0 : (r1 == 0 ? k1 : k2);
        const double s1 = r0 == 1 ? k0 : (r1 == 1 ? k1 : k2);
        const double s2 = r0 == 2 ? k0 : (r1 == 2 ? k1 : k2);
        const int a0 = r0 == 0 ? 1 : (r1 == 0 ? 2 : 4);
        const int a1 = r0 == 1 ? 1 : (r1 == 1 ? 2 : 4);
        k0 = s0;
        k1 = s1;
        k2 = s2;
        const int c0 = b0, c1 = c0 | a0, c2 = c1 | a1, c3 = 7;  // every axis crossed
        st[0] = tin;
        st[1] = pmin(k0, tout);
        st[2] = pmin(k1, tout);
        st[3] = pmin(k2, tout);
        st[4] = tout;
        // child pointers: four independent loads from the same 32-byte row
        const int32_t *row = child + (size_t)t.ptr * 8u;
        cp[0] = __ldg(row + (c0 ^ mirror));
        cp[1] = __ldg(row + (c1 ^ mirror));
        cp[2] = __ldg(row + (c2 ^ mirror));
        cp[3] = __ldg(row + (c3 ^ mirror));
        int keep = 0;
#pragma unroll
        for (int s = 0; s < 4; ++s)
            if (cp[s] >= 0 && st[s + 1] > st[s]) keep |= 1 << s;
        if (t.L + 1 == depth) {
            t.need_pop = true;
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                // branch-free: write slot n, keep it only for a kept leaf
                // (n < kSegMin before this node, so n + 3 < kSegSlots)
                seg.put<Visitor::kPops>(n, cp[s], st[s], st[s + 1], vis.pop_count());
                n += (keep >> s) & 1;
            }
            if (kDebugChecks) vis.check_queue(n, Visitor::kSegSlots);
            if (n >= Visitor::kSegMin) return n;
            continue;
        }
        if (!keep) {
            t.need_pop = true;
            continue;
        }
        // push the farther kept children far -> near (kernels.py:639-647),
        // predicated, then continue with the nearest kept child in registers
        const int cb[4] = {c0, c1, c2, c3};
        const typename Entry::Code pc2 = t.pc << 1;
#pragma unroll
        for (int s = 3; s >= 1; --s) {
            // branch-free: the entry always goes to the top slot and the top
            // moves only for a real push (a slot above the top is scratch;
            // at a level-L node the stack holds <= 3L entries, so the slot
            // is <= 3(depth-2)+2 < stack_cap = 3(depth-1))
            const bool push = ((keep >> s) & 1) && (keep & ((1 << s) - 1));
            Entry::store(t.sp, (uint32_t)cp[s], t.L + 1, pc2 | Entry::spread(cb[s]));
            t.sp += push ? stride : 0u;
        }
        uint32_t nptr = 0;
        int nb = 0;
        double ntin = 0.0, ntout = 0.0;
#pragma unroll
        for (int s = 3; s >= 0; --s) {
            if ((keep >> s) & 1) {
                nptr = (uint32_t)cp[s];
                nb = cb[s];
                ntin = st[s];
                ntout = st[s + 1];
            }
        }
        t.ptr = nptr;
        t.pc = pc2 | Entry::spread(nb);
        if (nb & 1) t.xl = xadd(t.xl, hh);
        if (nb & 2) t.yl = xadd(t.yl, hh);
        if (nb & 4) t.zl = xadd(t.zl, hh);
        t.h = hh;
        ++t.L;
        t.tin = ntin;
        t.tout = ntout;
    }
}

// Whole-ray traversal: walk -> shade queue -> walk ... until exhausted or
// stopped.  `smem` is the block's dynamic shared memory: the segment
// queues (seg_bytes_per_thread per thread), then the stacks (one slot per
// pending sibling, consecutive slots blockDim.x entries apart).
//
// Warp-synchronous while-while: the lanes that entered together walk and
// shade in lock step (finished lanes idle), so every shading round runs
// converged; queueing >= kSegMin segments per round keeps the walks of the
// lanes similar in length.  (One last-level node per round shaded in
// lock step wasted the walkers' time; letting the compiler interleave walk
// and shade per lane shaded in partial warps -- both measured slower.)
template <class Entry, class Visitor>
__device__ __forceinline__ void traverse(const int32_t *__restrict__ child, int depth, const Ray &r,
                                         unsigned char *smem, Visitor &vis) {
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
    const int nt = blockDim.x, tid = threadIdx.x;
    SegBuf seg;
    seg.init(sbase, nt, tid, Visitor::kSegSlots);
    const uint32_t base =
        sbase + seg_bytes_per_thread(Visitor::kPops, Visitor::kSegSlots) * nt + (uint32_t)tid * Entry::kBytes;
    const uint32_t stride = (uint32_t)nt * Entry::kBytes;
    Trav<Entry> t;
    t.init(r, base);
    const unsigned mask = __activemask();
    bool alive = true;
    while (true) {
        int n = 0;
        if (alive) {
            n = trav_next(t, child, depth, r, base, stride, vis, seg);
            alive = n >= Visitor::kSegMin;  // fewer: the walk is exhausted
        }
        __syncwarp(mask);
        if (n && vis.batch(seg, n)) alive = false;
        if (!__any_sync(mask, alive)) break;
    }
}

// ------------------------------------------------------------ fp32 basis
__device__ __forceinline__ float frcp_fast(float x) { return __fdividef(1.0f, x); }
// fp32 logistic; MUFU exp + fast reciprocal (abs error ~1e-7, well inside
// the 1e-4 colour tolerance).  exp(-x) overflowing to inf gives exactly 0.
__device__ __forceinline__ float sigmoidf_(float x) {
    return frcp_fast(1.0f + __expf(-x));
}

// Real SH stack at a unit direction, kernels.py:127-164 (fp32)
template <int NMAX>
__device__ __forceinline__ void sh_basis(float dx, float dy, float dz, const Consts &K, float *out) {
    const float rxy = sqrtf(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)));
    float cphi = 1.0f, sphi = 0.0f;
    if (rxy > 0.0f) {
        const float ir = frcp_fast(rxy);
        cphi = dx * ir;
        sphi = dy * ir;
    }
    const float z = dz;
    float cm = 1.0f, sm = 0.0f, pmm = 1.0f;
#pragma unroll
    for (int mu = 0; mu <= NMAX; ++mu) {
        if (mu > 0) {
            const float ncm = cm * cphi - sm * sphi;
            const float nsm = sm * cphi + cm * sphi;
            cm = ncm;
            sm = nsm;
            pmm = pmm * (2.0f * mu - 1.0f) * rxy;
        }
        float p_prev = 0.0f, p = pmm;
#pragma unroll
        for (int l = mu; l <= NMAX; ++l) {
            if (l == mu) {
                p = pmm;
            } else if (l == mu + 1) {
                p_prev = p;
                p = z * (2.0f * mu + 1.0f) * pmm;
            } else {
                const float np_ = (z * (float)(2 * l - 1) * p - (float)(l + mu - 1) * p_prev) / (float)(l - mu);
                p_prev = p;
                p = np_;
            }
            const int base = l * l + l;
            if (mu == 0) {
                out[base] = K.sh_pref[base] * p;
            } else {
                out[base + mu] = K.sh_pref[base + mu] * p * cm;
                out[base - mu] = K.sh_pref[base - mu] * p * sm;
            }
        }
    }
}

// Radial profiles A_nl sin^l(g) C^{l+1}_{n-l}(cos g), kernels.py:106-124 (fp32).
// s = sigmoid(gamma_pre), gamma = pi * s, so sin/cos come from sincospi(s).
template <int NMAX>
__device__ __forceinline__ void radial(float s, const Consts &K, float *R) {
    float sg, cg;
    sincospif(s, &sg, &cg);
    int p = 0;
#pragma unroll
    for (int n = 0; n <= NMAX; ++n) {
#pragma unroll
        for (int l = 0; l <= n; ++l) {
            const int d = n - l;
            const float alpha = (float)(l + 1);
            float c = 1.0f;
            if (d >= 1) {
                float c_prev = 1.0f;
                c = 2.0f * alpha * cg;
#pragma unroll
                for (int dd = 2; dd <= d; ++dd) {
                    const float nc = (2.0f * cg * (float)(dd + l) * c - (float)(dd + 2 * l) * c_prev) / (float)dd;
                    c_prev = c;
                    c = nc;
                }
            }
            float sl = 1.0f;
#pragma unroll
            for (int i = 0; i < l; ++i) sl *= sg;
            R[p] = K.pair_norm[p] * sl * c;
            ++p;
        }
    }
}

// HH->SH slice for one SH column j = (l, m): q_j,ch = sum_{n=l..NMAX}
// R(n,l) * w_hh[k(n,l,m), ch]  (kernels.py:384-394, reordered per column;
// pinned fp32 ops so cached and uncached renders agree bitwise).
template <int NMAX>
__device__ __forceinline__ void slice_col(const float *R, const float *wh, int l, int m, float &q0,
                                          float &q1, float &q2) {
    q0 = 0.0f;
    q1 = 0.0f;
    q2 = 0.0f;
#pragma unroll
    for (int n = 0; n <= NMAX; ++n) {
        if (n >= l) {
            const int kbase = n * (n + 1) * (2 * n + 1) / 6;  // sum_{n'<n} (n'+1)^2
            const int k = kbase + l * l + (m + l);
            const float rp = R[n * (n + 1) / 2 + l];
            q0 = __fmaf_rn(rp, wh[3 * k + 0], q0);
            q1 = __fmaf_rn(rp, wh[3 * k + 1], q1);
            q2 = __fmaf_rn(rp, wh[3 * k + 2], q2);
        }
    }
}

// row loads: read-only global path (__ldg) or the shared-memory staging
// (ld.shared at a 32-bit shared address; volatile keeps it after the
// mbarrier wait that published the TMA data)
template <bool G>
__device__ __forceinline__ float4 ld4(const float4 *p) {
    if (G) return __ldg(p);
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return v;
}

// Decoded fp32 hyper-angle sigmoid s = sigmoid(B[t] . w_gamma) (fp32 dot)
// over the chunks in `mask` (nz_chunks of B[t]); chunk i at g[i * cs].
template <bool G = true>
__device__ __forceinline__ float gamma_s(const float4 *__restrict__ g, int64_t cs, const float *sB, int C,
                                         uint32_t mask) {
    float gp = 0.0f;
    for (uint32_t m = mask; m; m &= m - 1) {
        const int i = __ffs(m) - 1;
        const float4 v = ld4<G>(g + i * cs);
        const int c = 4 * i;
        gp = __fmaf_rn(sB[c], v.x, gp);
        if (c + 1 < C) gp = __fmaf_rn(sB[c + 1], v.y, gp);
        if (c + 2 < C) gp = __fmaf_rn(sB[c + 2], v.z, gp);
        if (c + 3 < C) gp = __fmaf_rn(sB[c + 3], v.w, gp);
    }
    return sigmoidf_(gp);
}

// sigma_pre = sum_c A[t,c] * w_sigma[c], float64, sequential (kernels.py:374-381),
// over the chunks in `mask` (nz_chunks of A[t]); chunk i at w[i * cs].
template <bool G = true>
__device__ __forceinline__ double sigma_pre(const float4 *__restrict__ w, int64_t cs, const float *sA, int C,
                                            uint32_t mask) {
    double sp = 0.0;
    for (uint32_t m = mask; m; m &= m - 1) {
        const int i = __ffs(m) - 1;
        const float4 v = ld4<G>(w + i * cs);
        const int c = 4 * i;
        sp = xadd(sp, xmul((double)sA[c], (double)v.x));
        if (c + 1 < C) sp = xadd(sp, xmul((double)sA[c + 1], (double)v.y));
        if (c + 2 < C) sp = xadd(sp, xmul((double)sA[c + 2], (double)v.z));
        if (c + 3 < C) sp = xadd(sp, xmul((double)sA[c + 3], (double)v.w));
    }
    return sp;
}

// sigma_pre / the gamma dot with the first P chunk loads issued together
// (independent loads in flight; the sums keep the same order, so the same
// bits as sigma_pre / gamma_s)
template <int P>
__device__ __forceinline__ double sigma_pre_batched(const float4 *__restrict__ w, int64_t cs, const float *sA, int C,
                                                    uint32_t mask) {
    float4 v[P];
    int at[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
        at[k] = -1;
        if (mask) {
            at[k] = __ffs(mask) - 1;
            mask &= mask - 1;
            v[k] = __ldg(w + at[k] * cs);
        }
    }
    double sp = 0.0;
#pragma unroll
    for (int k = 0; k < P; ++k) {
        if (at[k] < 0) break;
        const int c = 4 * at[k];
        sp = xadd(sp, xmul((double)sA[c], (double)v[k].x));
        if (c + 1 < C) sp = xadd(sp, xmul((double)sA[c + 1], (double)v[k].y));
        if (c + 2 < C) sp = xadd(sp, xmul((double)sA[c + 2], (double)v[k].z));
        if (c + 3 < C) sp = xadd(sp, xmul((double)sA[c + 3], (double)v[k].w));
    }
    for (uint32_t m = mask; m; m &= m - 1) {  // chunks beyond the first P
        const int i = __ffs(m) - 1;
        const float4 x = __ldg(w + i * cs);
        const int c = 4 * i;
        sp = xadd(sp, xmul((double)sA[c], (double)x.x));
        if (c + 1 < C) sp = xadd(sp, xmul((double)sA[c + 1], (double)x.y));
        if (c + 2 < C) sp = xadd(sp, xmul((double)sA[c + 2], (double)x.z));
        if (c + 3 < C) sp = xadd(sp, xmul((double)sA[c + 3], (double)x.w));
    }
    return sp;
}

template <int P>
__device__ __forceinline__ float gamma_s_batched(const float4 *__restrict__ g, int64_t cs, const float *sB, int C,
                                                 uint32_t mask) {
    float4 v[P];
    int at[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
        at[k] = -1;
        if (mask) {
            at[k] = __ffs(mask) - 1;
            mask &= mask - 1;
            v[k] = __ldg(g + at[k] * cs);
        }
    }
    float gp = 0.0f;
#pragma unroll
    for (int k = 0; k < P; ++k) {
        if (at[k] < 0) break;
        const int c = 4 * at[k];
        gp = __fmaf_rn(sB[c], v[k].x, gp);
        if (c + 1 < C) gp = __fmaf_rn(sB[c + 1], v[k].y, gp);
        if (c + 2 < C) gp = __fmaf_rn(sB[c + 2], v[k].z, gp);
        if (c + 3 < C) gp = __fmaf_rn(sB[c + 3], v[k].w, gp);
    }
    for (uint32_t m = mask; m; m &= m - 1) {
        const int i = __ffs(m) - 1;
        const float4 x = __ldg(g + i * cs);
        const int c = 4 * i;
        gp = __fmaf_rn(sB[c], x.x, gp);
        if (c + 1 < C) gp = __fmaf_rn(sB[c + 1], x.y, gp);
        if (c + 2 < C) gp = __fmaf_rn(sB[c + 2], x.z, gp);
        if (c + 3 < C) gp = __fmaf_rn(sB[c + 3], x.w, gp);
    }
    return sigmoidf_(gp);
}

template <int NMAX, bool G = true>
__device__ __forceinline__ void load_hh(const float4 *__restrict__ hh_row, float *wh) {
    constexpr int H4 = Basis<NMAX>::HH4;
#pragma unroll
    for (int i = 0; i < H4; ++i) {
        const float4 v = ld4<G>(hh_row + i);
        wh[4 * i + 0] = v.x;
        wh[4 * i + 1] = v.y;
        wh[4 * i + 2] = v.z;
        wh[4 * i + 3] = v.w;
    }
}

// visible-set bit of leaf row L (fire-and-forget reduction)
__device__ __forceinline__ void vis_mark(uint32_t *m, uint32_t L) { atomicOr(m + (L >> 5), 1u << (L & 31)); }

// ------------------------------------------------------------ shading visitor
struct FrameCtx {
    const float *sA;   // A[t] row in shared memory
    const float *sB;   // B[t] row in shared memory
    int frame;
    double early_stop;
    double edit_weight;
    uint32_t mA, mB;   // nz_chunks of the two rows
};

// CACHED: 0 = decode per sample, 1 = read the frame slice, 2 = decided at
// run time by S.rec != nullptr (scene kernel, per-instance slices).
// VIS (camera kernel, visible-set slices): 1 = sliced walk that stops at a
// leaf outside the slice's visible set (record sigma < 0; `deferred`: the
// pixel is walked again per sample); 3 = the same in a census frame, also
// marking every leaf it visits; 2 = the per-sample walk of a deferred
// pixel, marking every leaf it visits.
template <int NMAX, int CACHED, bool EDITS, bool VISITS, bool POPS = false, int SEG = VV_SEG_MIN, int VIS = 0>
struct Shader {
    static constexpr bool kPops = POPS;  // exact node-pop counts (stats)
    static constexpr int kSegMin = SEG, kSegSlots = SEG + 3;
    const TreeView &T;
    const SliceView &S;
    const FrameCtx &F;
    const Consts &K;
    float dx, dy, dz;
    double trans, acc0, acc1, acc2, aacc, tacc;
    int used, pops, shaded;
    bool y_ready;
    bool deferred = false;  // VIS 1: met a leaf outside the visible set
    float y[Basis<NMAX>::S];
    int64_t *visit;  // VISITS: this ray's slice of the CSR

    __device__ __forceinline__ Shader(const TreeView &T_, const SliceView &S_, const FrameCtx &F_,
                                      const Consts &K_, float dx_, float dy_, float dz_)
        : T(T_), S(S_), F(F_), K(K_), dx(dx_), dy(dy_), dz(dz_), trans(1.0), acc0(0.0), acc1(0.0),
          acc2(0.0), aacc(0.0), tacc(0.0), used(0), pops(0), shaded(0), y_ready(false), visit(nullptr) {}

    __device__ __forceinline__ void pop() { ++pops; }
    __device__ __forceinline__ int pop_count() const { return pops; }
    // bounds checks (debug build): node row, stack slots in use, queue fill
    __device__ __forceinline__ void check_node(uint32_t ptr, uint32_t slots) const {
        if (ptr >= (uint64_t)T.n_internal) debug_violation(T.dbg, VV_DBG_NODE);
        if (slots > (uint32_t)stack_cap(T.depth)) debug_violation(T.dbg, VV_DBG_STACK);
        if (T.dbg) atomicMax(T.dbg + 2, slots);  // stack high-water mark
    }
    __device__ __forceinline__ void check_queue(int n, int slots) const {
        if (n > slots) debug_violation(T.dbg, VV_DBG_QUEUE);
    }

    __device__ __forceinline__ void reset(float dx_, float dy_, float dz_) {
        dx = dx_;
        dy = dy_;
        dz = dz_;
        trans = 1.0;
        acc0 = acc1 = acc2 = aacc = tacc = 0.0;
        used = pops = shaded = 0;
        y_ready = false;
    }

    __device__ __forceinline__ bool is_cached() const { return CACHED == 1 || (CACHED == 2 && S.rec != nullptr); }

    // one round of queued segments: warm L1 with every queued record first
    // (independent prefetches; one 128-byte line per record at n_max 2,
    // sigma in its last 8 bytes), then composite them in order
    __device__ __forceinline__ bool batch(const SegBuf &seg, int n) {
        if (is_cached()) {
#pragma unroll 1
            for (int s = 0; s < n; ++s) {
                const char *q = reinterpret_cast<const char *>(S.row((uint32_t)seg.leaf_at(s)));
                prefetch_l1(q);
                if (16 * S.rec4 > 128) prefetch_l1(q + 16 * S.rec4 - 1);
            }
        }
        // software-pipelined: the next segment's sigma is requested before
        // the current one shades
        uint32_t L = (uint32_t)seg.leaf_at(0);
        double sg = is_cached() ? S.sigma(L) : 0.0;
#pragma unroll 1
        for (int s = 0; s < n; ++s) {
            uint32_t Ln = 0;
            double sgn = 0.0;
            if (s + 1 < n) {
                Ln = (uint32_t)seg.leaf_at(s + 1);
                if (is_cached()) sgn = S.sigma(Ln);
            }
            if (leaf(L, seg.t0_at(s), seg.t1_at(s), sg)) {
                if (POPS) pops = seg.pops_at(s);  // the walk may have run ahead
                return true;
            }
            L = Ln;
            sg = sgn;
        }
        return false;
    }

    __device__ __forceinline__ bool leaf(uint32_t L, double tin, double tout, double sigma_cached) {
        if (kDebugChecks && L >= (uint64_t)T.n_leaves) debug_violation(T.dbg, VV_DBG_LEAF);
        if (VISITS) visit[used] = ref_row(T.leaf_ref, L);
        ++used;
        constexpr int Q4 = Basis<NMAX>::Q4;
        // sliced coefficients: from the frame slice record, or decoded now
        // from the payload (render_kernel's uncached branch)
        const bool from_rec = is_cached();
        double sigma;
        // visible-set walks: a deferred pixel's walk (VIS 2) and a census
        // (VIS 3) put every leaf they visit in the set
        if (VIS == 2) vis_mark(S.mark, L);
        if (from_rec) {
            sigma = sigma_cached;
            // outside the slice's set (a negative sigma, or the walk table's
            // stand-in row): the pixel is walked again per sample
            if ((VIS == 1 || VIS == 3) && sigma < 0.0) {
                deferred = true;
                return true;
            }
            if (VIS == 3) vis_mark(S.mark, L);
        } else {
            const double sp = sigma_pre(T.sig + L, T.lstride, F.sA, T.C, F.mA);
            sigma = sp > 0.0 ? sp : 0.0;
        }
        bool edited = false;
        float4 erg = make_float4(0.f, 0.f, 0.f, 0.f);
        if (EDITS && T.edit_t != nullptr) {
            const int2 et = __ldg(T.edit_t + L);
            if (et.x <= F.frame && F.frame <= et.y) {
                edited = true;
                erg = __ldg(T.edit_rgb + L);
                const double sd = (double)erg.w;
                if (sd >= 0.0) sigma = sd;
            }
        }
        if (sigma == 0.0) return false;  // zero optical depth (kernels.py:556-559)
        ++shaded;
        if (!y_ready) {
            sh_basis<NMAX>(dx, dy, dz, K, y);
            y_ready = true;
        }
        // colour: c_ch = sigmoid(sum_j y_j q_j,ch)
        float c0 = 0.0f, c1 = 0.0f, c2 = 0.0f;
        if (from_rec) {
            float q[4 * Q4];
            const float4 *qr = S.row(L);
#pragma unroll
            for (int i = 0; i < Q4; ++i) {
                const float4 v = __ldg(qr + i);
                q[4 * i + 0] = v.x;
                q[4 * i + 1] = v.y;
                q[4 * i + 2] = v.z;
                q[4 * i + 3] = v.w;
            }
#pragma unroll
            for (int j = 0; j < Basis<NMAX>::S; ++j) {
                c0 = __fmaf_rn(y[j], q[3 * j + 0], c0);
                c1 = __fmaf_rn(y[j], q[3 * j + 1], c1);
                c2 = __fmaf_rn(y[j], q[3 * j + 2], c2);
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
                    float q0, q1, q2;
                    slice_col<NMAX>(R, wh, l, m, q0, q1, q2);
                    c0 = __fmaf_rn(y[j], q0, c0);
                    c1 = __fmaf_rn(y[j], q1, c1);
                    c2 = __fmaf_rn(y[j], q2, c2);
                }
        }
        double col0 = (double)sigmoidf_(c0);
        double col1 = (double)sigmoidf_(c1);
        double col2 = (double)sigmoidf_(c2);
        if (EDITS && edited) {  // kernels.py:584-587
            const double ew = F.edit_weight, om = xsub(1.0, ew);
            col0 = xadd(xmul(ew, (double)erg.x), xmul(om, col0));
            col1 = xadd(xmul(ew, (double)erg.y), xmul(om, col1));
            col2 = xadd(xmul(ew, (double)erg.z), xmul(om, col2));
        }
        // front-to-back compositing, float64 (kernels.py:588-598)
        const double delta = xsub(tout, tin);
        const double e = exp(xmul(-sigma, delta));
        const double a = xsub(1.0, e);
        const double w = xmul(trans, a);
        acc0 = xadd(acc0, xmul(w, col0));
        acc1 = xadd(acc1, xmul(w, col1));
        acc2 = xadd(acc2, xmul(w, col2));
        aacc = xadd(aacc, w);
        tacc = xadd(tacc, xmul(xmul(w, 0.5), xadd(tin, tout)));
        trans = xmul(trans, e);
        return trans < F.early_stop;
    }
};

// Several frames of one camera in one walk (playback): the rays, and so the
// traversal and the segment list, do not depend on the frame; every frame
// keeps its own slice, accumulators and early termination, and sees the
// same segments in the same order as a single-frame render -- identical
// results.  The walk ends when every frame has terminated.
constexpr int kMaxMulti = 4;
template <int NMAX, int KF, bool EDITS, int SEG = VV_SEG_MIN>
struct ShaderMulti {
    static constexpr int kSegMin = SEG, kSegSlots = SEG + 3;
    static constexpr bool kPops = false;
    const TreeView &T;
    const SliceView *S;  // KF frame slices
    const int *frames;
    const Consts &K;
    double early_stop, edit_weight;
    float dx, dy, dz;
    double trans[KF], acc0[KF], acc1[KF], acc2[KF], aacc[KF], tacc[KF];
    unsigned alive;
    int used = 0;  // segments consumed by the shared walk (a plan's cost)
    bool y_ready;
    float y[Basis<NMAX>::S];

    __device__ __forceinline__ ShaderMulti(const TreeView &T_, const SliceView *S_, const int *frames_, const Consts &K_,
                                           double es, double ew, float dx_, float dy_, float dz_)
        : T(T_), S(S_), frames(frames_), K(K_), early_stop(es), edit_weight(ew), dx(dx_), dy(dy_), dz(dz_),
          alive((1u << KF) - 1u), y_ready(false) {
#pragma unroll
        for (int k = 0; k < KF; ++k) {
            trans[k] = 1.0;
            acc0[k] = acc1[k] = acc2[k] = aacc[k] = tacc[k] = 0.0;
        }
    }
    __device__ __forceinline__ void pop() {}
    __device__ __forceinline__ int pop_count() const { return 0; }
    __device__ __forceinline__ void check_node(uint32_t ptr, uint32_t slots) const {
        if (ptr >= (uint64_t)T.n_internal) debug_violation(T.dbg, VV_DBG_NODE);
        if (slots > (uint32_t)stack_cap(T.depth)) debug_violation(T.dbg, VV_DBG_STACK);
        if (T.dbg) atomicMax(T.dbg + 2, slots);  // stack high-water mark
    }
    __device__ __forceinline__ void check_queue(int n, int slots) const {
        if (n > slots) debug_violation(T.dbg, VV_DBG_QUEUE);
    }

    __device__ __forceinline__ bool batch(const SegBuf &seg, int n) {
#pragma unroll 1
        for (int s = 0; s < n; ++s) {  // records of the live frames to L1
            const uint32_t L = (uint32_t)seg.leaf_at(s);
#pragma unroll
            for (int k = 0; k < KF; ++k)
                if ((alive >> k) & 1u) prefetch_l1(S[k].row(L));
        }
#pragma unroll 1
        for (int s = 0; s < n; ++s) {
            const uint32_t L = (uint32_t)seg.leaf_at(s);
            const double tin = seg.t0_at(s), tout = seg.t1_at(s);
            ++used;
            double sg[KF];  // every live frame's sigma requested at once (independent loads)
#pragma unroll
            for (int k = 0; k < KF; ++k) sg[k] = ((alive >> k) & 1u) ? S[k].sigma(L) : 0.0;
#pragma unroll
            for (int k = 0; k < KF; ++k)
                if (((alive >> k) & 1u) && leaf(k, L, tin, tout, sg[k])) alive &= ~(1u << k);
            if (!alive) return true;
        }
        return false;
    }

    // Shader::leaf (kernels.py:539-599) for frame k (a constant after
    // unrolling: the per-frame arrays stay in registers), sliced path
    __device__ __forceinline__ bool leaf(int k, uint32_t L, double tin, double tout, double sigma) {
        constexpr int Q4 = Basis<NMAX>::Q4;
        if (kDebugChecks && L >= (uint64_t)T.n_leaves) debug_violation(T.dbg, VV_DBG_LEAF);
        bool edited = false;
        float4 erg = make_float4(0.f, 0.f, 0.f, 0.f);
        if (EDITS && T.edit_t != nullptr) {
            const int2 et = __ldg(T.edit_t + L);
            if (et.x <= frames[k] && frames[k] <= et.y) {
                edited = true;
                erg = __ldg(T.edit_rgb + L);
                const double sd = (double)erg.w;
                if (sd >= 0.0) sigma = sd;
            }
        }
        if (sigma == 0.0) return false;
        if (!y_ready) {
            sh_basis<NMAX>(dx, dy, dz, K, y);
            y_ready = true;
        }
        float c0 = 0.0f, c1 = 0.0f, c2 = 0.0f;
        {
            float q[4 * Q4];
            const float4 *qr = S[k].row(L);
#pragma unroll
            for (int i = 0; i < Q4; ++i) {
                const float4 v = __ldg(qr + i);
                q[4 * i + 0] = v.x;
                q[4 * i + 1] = v.y;
                q[4 * i + 2] = v.z;
                q[4 * i + 3] = v.w;
            }
#pragma unroll
            for (int j = 0; j < Basis<NMAX>::S; ++j) {
                c0 = __fmaf_rn(y[j], q[3 * j + 0], c0);
                c1 = __fmaf_rn(y[j], q[3 * j + 1], c1);
                c2 = __fmaf_rn(y[j], q[3 * j + 2], c2);
            }
        }
        double col0 = (double)sigmoidf_(c0);
        double col1 = (double)sigmoidf_(c1);
        double col2 = (double)sigmoidf_(c2);
        if (EDITS && edited) {
            const double ew = edit_weight, om = xsub(1.0, ew);
            col0 = xadd(xmul(ew, (double)erg.x), xmul(om, col0));
            col1 = xadd(xmul(ew, (double)erg.y), xmul(om, col1));
            col2 = xadd(xmul(ew, (double)erg.z), xmul(om, col2));
        }
        const double delta = xsub(tout, tin);
        const double e = exp(xmul(-sigma, delta));
        const double a = xsub(1.0, e);
        const double w = xmul(trans[k], a);
        acc0[k] = xadd(acc0[k], xmul(w, col0));
        acc1[k] = xadd(acc1[k], xmul(w, col1));
        acc2[k] = xadd(acc2[k], xmul(w, col2));
        aacc[k] = xadd(aacc[k], w);
        tacc[k] = xadd(tacc[k], xmul(xmul(w, 0.5), xadd(tin, tout)));
        trans[k] = xmul(trans[k], e);
        return trans[k] < early_stop;
    }
};

// Traversal-only visitors (count / collect, kernels.py:313-367)
struct NoChecks {  // visitors without a tree view: no bounds checks
    __device__ __forceinline__ void check_node(uint32_t, uint32_t) const {}
    __device__ __forceinline__ void check_queue(int, int) const {}
};
struct CountVisitor : NoChecks {
    static constexpr int kSegMin = VV_SEG_MIN, kSegSlots = VV_SEG_SLOTS;
    static constexpr bool kPops = false;
    int64_t count = 0;
    __device__ __forceinline__ void pop() {}
    __device__ __forceinline__ int pop_count() const { return 0; }
    __device__ __forceinline__ bool batch(const SegBuf &, int n) {
        count += n;
        return false;
    }
};
struct CollectVisitor : NoChecks {
    static constexpr int kSegMin = VV_SEG_MIN, kSegSlots = VV_SEG_SLOTS;
    static constexpr bool kPops = false;
    const int32_t *leaf_ref;
    int64_t *leaf_out;
    double *t0_out, *t1_out;
    int64_t count, cap;
    __device__ __forceinline__ void pop() {}
    __device__ __forceinline__ int pop_count() const { return 0; }
    __device__ __forceinline__ bool batch(const SegBuf &seg, int n) {
        for (int s = 0; s < n; ++s) {
            if (count < cap) {
                leaf_out[count] = ref_row(leaf_ref, (uint32_t)seg.leaf_at(s));
                t0_out[count] = seg.t0_at(s);
                t1_out[count] = seg.t1_at(s);
            }
            ++count;
        }
        return false;
    }
};

// ------------------------------------------------------------ camera rays
// Camera.rays (render.py:74-83): pixel centre, d_cam = (x, y, 1),
// d_world = R d_cam, normalised.  fp64.  The BLAS product of the reference
// is not reproducible bit for bit across CPUs; parity for bit-exact visit
// lists is therefore checked with host-generated rays (render_rays).
struct CamView {
    int width, height;
    double fx, fy, cx, cy;
    double r00, r01, r02, r10, r11, r12, r20, r21, r22;
    double ox, oy, oz;
};

__device__ __forceinline__ void camera_ray(const CamView &c, int ix, int iy, double &dx, double &dy,
                                           double &dz) {
    const double x = xdiv(xsub(xadd((double)ix, 0.5), c.cx), c.fx);
    const double y = xdiv(xsub(xadd((double)iy, 0.5), c.cy), c.fy);
    const double w0 = __fma_rn(1.0, c.r02, __fma_rn(y, c.r01, xmul(x, c.r00)));
    const double w1 = __fma_rn(1.0, c.r12, __fma_rn(y, c.r11, xmul(x, c.r10)));
    const double w2 = __fma_rn(1.0, c.r22, __fma_rn(y, c.r21, xmul(x, c.r20)));
    const double nrm = sqrt(xadd(xadd(xmul(w0, w0), xmul(w1, w1)), xmul(w2, w2)));
    dx = xdiv(w0, nrm);
    dy = xdiv(w1, nrm);
    dz = xdiv(w2, nrm);
}

// finalize_layer (render.py:218-233) for one ray, fp64 -> fp32 outputs
__device__ __forceinline__ void finalize(double p0, double p1, double p2, double alpha, double tbar,
                                         double depth_scale, bool scaled, double alpha_floor,
                                         double far_plane, float &r, float &g, float &b, float &a,
                                         float &d) {
    const double safe = alpha > 1e-300 ? alpha : 1e-300;
    if (alpha > 0.0) {
        r = (float)xdiv(p0, safe);
        g = (float)xdiv(p1, safe);
        b = (float)xdiv(p2, safe);
    } else {
        r = g = b = 0.0f;
    }
    double t = xdiv(tbar, safe);
    if (scaled) t = xmul(t, depth_scale);
    d = (float)(alpha >= alpha_floor ? t : far_plane);
    a = (float)alpha;
}

}  // namespace vv
