// vv_api.cu -- the C ABI (include/voxvid_b200.h): tree replicas, slices and
// the render entry points.  Kernels: vv_kernels.cuh / vv_launch_*.cu.
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
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <memory>
#include <deque>
#include <mutex>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/voxvid_b200.h"
#include "vv_kernels.cuh"

// NVTX ranges around the host-side phases of every entry point (slice pass,
// node mask, chunk culling, render, band copies, scene, gather): they group
// the launches in an Nsight Systems / ncu timeline.  Header-only NVTX v3;
// no-ops unless a tool is attached.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
};

using namespace vv;
using namespace vvk;

struct vv_tree {
    int device;
    TreeView view;
    int64_t n_leaves, n_internal;
    int32_t frames, C, K, S, n_max, depth;
    bool has_edits;
    int64_t bytes;
    // owned device allocations
    int32_t *d_child;
    float4 *d_sig, *d_gam, *d_hh, *d_edit_rgb;
    int2 *d_edit_t;
    float *d_a, *d_b;
    std::vector<float> h_a, h_b;  // host copies of the basis rows (slice-pass chunk masks)
    float dark_frac = 0.0f;       // share of leaves with sigma 0, over a few frames (queue threshold)
    // node-mask tables (vv_launch_mask.cu), set when the table is a tree
    // (one parent per node, every leaf row at the last level)
    int32_t *d_parent, *d_last, *d_upper;
    int64_t n_last, n_upper;
    bool mask_ok;
    // leaf-cell boxes of every kRegionChunk consecutive leaf rows (cell
    // units at the leaf depth: x0 y0 z0 0 x1 y1 z1 0, inclusive), for
    // region renders that slice only the chunks their pixels can reach
    int4 *d_box;
    int64_t n_box;
    // walk-order leaf layout (analyze_tree): device row -> reference row and
    // back (null: identity); the host copy permutes edit uploads
    int32_t *d_leaf_ref, *d_dev_row;
    std::vector<int32_t> h_perm;
    uint64_t serial;  // unique per upload (caches keyed on a tree never see a reused address)
    double occ_lo[3], occ_hi[3];  // world box of the occupied leaf cells (empty: lo > hi)
    // visible set (vis_begin): two bitmaps over leaf rows, filled by the
    // camera walks; render-internal slices decode colour only for leaves in
    // their union.  State advances per visible-set slice; races between
    // streams only cost misses (the records, not the bitmaps, tell the walk
    // which colours are present).
    mutable std::mutex vis_mu;
    mutable uint32_t *d_vis = nullptr;
    mutable int64_t vis_words = 0;
    mutable int vis_cur = 0, vis_slices = 0;
    mutable bool vis_ready = false;
    mutable uint64_t vis_view = 0;  // the camera the set is being built for (view_hash)
    mutable int vis_static = 0;     // slices since that camera last changed
};

// Per-frame (or per frame group) node mask: the slice pass's lit bits, the
// marker scratch and the masked child table, in one stream-ordered block
// shared by the slices of a group.
struct NodeMask {
    void *mem = nullptr;
    cudaStream_t st = nullptr;
    uint8_t *lit = nullptr;
    uint32_t *flag = nullptr;
    int32_t *mask = nullptr;
    NodeMask() = default;
    NodeMask(const NodeMask &) = delete;
    ~NodeMask() {
        if (mem) cudaFreeAsync(mem, st);
    }
};

// float4 chunks of the frame's fp32 A (which = 0) or B (1) row holding a
// nonzero entry -- the same test as the device's nz_chunks
static uint32_t host_nz_chunks(const vv_tree *t, int frame, int which) {
    const float *row = (which ? t->h_b.data() : t->h_a.data()) + (size_t)frame * t->C;
    uint32_t m = 0;
    for (int c = 0; c < t->C; ++c)
        if (row[c] != 0.0f) m |= 1u << (c >> 2);
    return m;
}

static void set_slice_masks(const vv_tree *t, SliceParams &p) {
    p.mS = p.mG = 0;
    for (int f = 0; f < p.n_frames; ++f) {
        p.mS |= host_nz_chunks(t, p.frame[f], 0);
        p.mG |= host_nz_chunks(t, p.frame[f], 1);
    }
}

struct vv_slice {
    const vv_tree *tree;
    int device;
    int32_t frame;
    float4 *d_rec;  // (n_leaves, rec4) records [q | pad | sigma]
    int rec4;
    bool render_only;  // colour omitted where sigma is 0 (VV_SLICE_RENDER_ONLY): not exportable
    bool visible = false;  // VV_SLICE_VISIBLE: colour only in the visible set (-sigma elsewhere)
    uint32_t *vis_mark = nullptr;  // the set its walks mark
    int vis_census = 0;
    void *d_vis_mem = nullptr;               // its walk table + set snapshot (vis_prepare)
    const int32_t *vis_table = nullptr;
    int64_t n_leaves;
    cudaStream_t stream;  // stream-ordered allocation: freed on this stream
    std::shared_ptr<NodeMask> nmask;  // dark subtrees cut (image renders), or null
};

// Launch plan of one camera stream (vv_camera_plan_create): the camera
// kernel runs persistent warps that take the frame's warp chunks from a
// counter in the order of the previous render's measured block costs
// (costliest first), and records this render's costs for the next.  Used
// from one stream at a time (like a library handle); the mutex guards the
// host state against concurrent calls.
struct vv_camera_plan {
    int device = 0;
    int blocks_x = 0, n_blocks = 0;  // the grid the buffers are sized for
    int32_t *order = nullptr;        // (n_blocks) launch order
    uint32_t *cost = nullptr;        // (n_blocks) costs of the last render
    int *counter = nullptr;
    bool valid = false;              // order holds a permutation for this grid
    int renders = 0;                 // renders since the last re-sort
    // coverage of the last (tree, camera) rendered through the plan: built
    // once per view, reused by every frame of it
    void *cov_mem = nullptr;
    size_t cov_cap = 0;
    uint64_t cov_tree = 0;  // serial of the tree the coverage belongs to
    vv_camera cov_cam;
    bool cov_valid = false;
    CoverView cov{};
    // visible-set walk table of the last tree rendered through the plan
    // (vis_prepare): kept across frames and rebuilt on the device only when
    // the set's snapshot changes (a held view's set settles after a frame)
    void *vis_mem = nullptr;
    size_t vis_cap = 0;
    uint64_t vis_tree = 0;
    bool vis_fresh = false;  // buffers (re)made: the next snapshot counts as changed
    std::mutex mu;
};

#define VV_CUDA(call)                                                                          \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess)                                                                 \
            return set_error(VV_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));      \
    } while (0)

// Benchmark split point (vv_profile_split_event): recorded by the calling
// thread's next camera render between its slice pass and its camera kernel.
static thread_local cudaEvent_t split_event = nullptr;

namespace {

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
    o.frame_slice = VV_SLICE_AUTO;
    o.reserved = 0;
    return o;
}

SliceView slice_view(const vv_slice *c) {
    SliceView s{nullptr, 0, 0, nullptr};
    if (c) {
        s.rec = c->d_rec;
        s.rec4 = c->rec4;
        s.census = c->vis_census;
        s.mark = c->vis_mark;
    }
    return s;
}

// ---- visible set (render-internal camera slices of trees without edits)
// A render's walks only reach a fraction of the leaves (cfg2: 19%, in 31% of
// the 64-leaf chunks), yet a slice decodes every lit leaf.  With a set in
// use, the slice decodes only the leaves in the tree's visible set and the
// camera kernel walks a walk table (vis_prepare) in which every other leaf
// points at a stand-in row whose record holds sigma -1: a walk that meets one
// defers its pixel to k_camera_rewalk, which walks it per sample on the
// tree's own table (bitwise the same) and marks what it visits.  Two
// bitmaps: the slice decodes a snapshot of their union; walks mark into the
// current one.  Every kVisEpoch slices the older one is cleared and becomes
// current, and that slice's walks mark every leaf they visit (a census), so
// the set follows the view and leaves drop out within two epochs of last
// being seen.  The set is built per camera (vis_begin's view rule).
// VV_VISIBLE=0 turns the set off (A/B).
constexpr int kVisEpoch = 16;  // cfg2: 2,651 vs 2,637 Mrays/s with 8, 2,648 with 32 (VV_VIS_EPOCH overrides)

struct VisTicket {
    const uint32_t *d0 = nullptr, *d1 = nullptr;  // decode set (null: every lit leaf)
    uint32_t *mark = nullptr;
    int census = 0;
    const int32_t *table = nullptr;  // the walk table (vis_prepare), with a set in use
    const int32_t *list = nullptr, *n_list = nullptr;  // the set's leaf rows (the slice's work list)
};

static bool mask_wanted(const vv_tree *t);
// On for trees without node masks.  Dark-heavy trees (node masks: lit
// leaves move from frame to frame, cfg3) defer too many pixels to the
// per-sample walk: measured cfg3 0.94 vs 0.48 ms per frame with the set, cfg2
// 0.831 vs 0.859, cfg5 1.811 vs 1.816 (profiles/r02_visible_set_ab.json).
// VV_VISIBLE=0 / 1 forces it off / on.
static bool vis_wanted(const vv_tree *t) {
    if (t->has_edits || t->n_leaves == 0 || !t->mask_ok) return false;  // the walk table needs the last-level list
    if (const char *e = getenv("VV_VISIBLE")) {
        if (e[0] == '0') return false;
        if (e[0] == '1') return true;
    }
    return !mask_wanted(t);
}

// A camera's identity for the visible set (its fields, not its padding).
static uint64_t view_hash(const vv_camera &c) {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&h](const void *p, size_t n) {
        const unsigned char *b = static_cast<const unsigned char *>(p);
        for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    };
    mix(&c.width, sizeof(c.width));
    mix(&c.height, sizeof(c.height));
    mix(&c.fx, 4 * sizeof(double));
    mix(c.c2w, sizeof(c.c2w));
    return h ? h : 1;
}

// view: the rendering camera's view_hash (0: unknown -- a VV_SLICE_VISIBLE
// cache, whose caller vouches for a steady view).  The set only pays for
// a camera that holds still: a moving view meets leaves outside it on every
// frame and re-walks those pixels (cfg2 tree orbited 1 deg / 5 deg per frame:
// 1.31 / 2.25 ms per frame with the set, 0.92 without;
// profiles/r02_moving_camera_probe.log).  So a slice for a camera other than
// the last one is a plain slice; the second slice of the same camera
// rebuilds the set for it (every lit leaf decoded, a census); from the
// third on the set is used.
// Whether vis_begin may hand a slice for this view a set (no state change;
// a race only leaves a deferred-chunk list unused).
static bool vis_may_use(const vv_tree *t, uint64_t view) {
    if (!vis_wanted(t)) return false;
    std::lock_guard<std::mutex> lk(t->vis_mu);
    return !view || view == t->vis_view;
}

// allow: the caller can run a visible-set render (else only the view is noted)
static int vis_begin(const vv_tree *t, cudaStream_t st, VisTicket &vt, uint64_t view = 0, bool allow = true) {
    vt = VisTicket();
    if (!vis_wanted(t)) return VV_OK;
    std::lock_guard<std::mutex> lk(t->vis_mu);
    if (view) {
        if (view == t->vis_view) {
            if (t->vis_static < 2) ++t->vis_static;
        } else {
            t->vis_view = view;
            t->vis_static = 0;
        }
        if (t->vis_static == 0 || !allow) return VV_OK;  // a new view: the plain slice
        if (t->vis_static == 1) t->vis_ready = false;    // the view held: rebuild the set for it
    } else if (!allow) {
        return VV_OK;
    }
    if (!t->d_vis) {
        const int64_t words = ((t->n_leaves + 63) / 64) * 2;  // whole 64-leaf slice chunks
        if (cudaMalloc(&t->d_vis, 2 * (size_t)words * sizeof(uint32_t)) != cudaSuccess) {
            cudaGetLastError();
            t->d_vis = nullptr;
            return VV_OK;  // no set: slices decode every lit leaf
        }
        VV_CUDA(cudaMemsetAsync(t->d_vis, 0, 2 * (size_t)words * sizeof(uint32_t), st));
        t->vis_words = words;
    }
    uint32_t *b[2] = {t->d_vis, t->d_vis + t->vis_words};
    if (!t->vis_ready) {  // a first slice, or a new view: every lit leaf decoded, the set started afresh
        VV_CUDA(cudaMemsetAsync(t->d_vis, 0, 2 * (size_t)t->vis_words * sizeof(uint32_t), st));
        t->vis_ready = true;
        t->vis_slices = 0;
        vt.mark = b[t->vis_cur];
        vt.census = 1;
        return VV_OK;
    }
    static const int epoch = [] {
        const char *e = getenv("VV_VIS_EPOCH");  // A/B runs
        const int v = e ? atoi(e) : 0;
        return v > 0 ? v : kVisEpoch;
    }();
    if (++t->vis_slices % epoch == 0) {
        t->vis_cur ^= 1;
        VV_CUDA(cudaMemsetAsync(b[t->vis_cur], 0, (size_t)t->vis_words * sizeof(uint32_t), st));
        vt.census = 1;
    }
    vt.d0 = b[0];
    vt.d1 = b[1];
    vt.mark = b[t->vis_cur];
    return VV_OK;
}

// The slice pass p describes: a visible-set slice (k_slice_visible) when
// the ticket has a set to fill, else the plain pass.
static int launch_slice_vis(const vv_tree *t, SliceParams &p, const VisTicket *vt, cudaStream_t st) {
    if (!vt || !vt->mark) {
        // a single-frame render-only slice of a dark-heavy tree: the
        // thread-per-leaf pass, colour of the lit leaves only (cfg3 0.166 vs
        // 0.191 ms; on mostly-lit trees the staged pass wins, 0.225 vs 0.276
        // at cfg2).  VV_LIT_PASS=0 / 1 forces it off / on.
        const char *e = getenv("VV_LIT_PASS");
        const bool lit_pass = e && (e[0] == '0' || e[0] == '1') ? e[0] == '1' : t->dark_frac >= 0.25f;
        if (!(p.n_frames == 1 && p.skip_dark && lit_pass)) return launch_slice(t->n_max, p, st);
        // sigma for every leaf (of a region: of its chunks) and the lit list, then the lit leaves' records
        void *m = nullptr;
        if (cudaMallocAsync(&m, (size_t)t->n_leaves * sizeof(int32_t) + 256, st) != cudaSuccess) {
            cudaGetLastError();
            return set_error(VV_E_NOMEM, "lit-leaf list allocation failed");
        }
        p.lit_list = static_cast<int32_t *>(m);
        p.lit_n = reinterpret_cast<int32_t *>(static_cast<char *>(m) + (((size_t)t->n_leaves * 4 + 255) & ~(size_t)255));
        int rc = VV_OK;
        if (cudaMemsetAsync(p.lit_n, 0, sizeof(int32_t), st) != cudaSuccess)
            rc = set_error(VV_E_CUDA, "lit-list counter memset failed");
        if (!rc) rc = launch_slice_visible(t->n_max, p, st);
        cudaFreeAsync(m, st);
        return rc;
    }
    p.vis0 = vt->d0;  // null: every leaf visible (a tree's first slice)
    p.vis1 = vt->d1;
    p.leaf_list = vt->list;  // with a walk table: a thread per leaf of the set
    p.n_leaf_list = vt->n_list;
    return launch_slice_visible(t->n_max, p, st);
}

// With a set in use: one stream-ordered block (*mem, the caller frees it)
// holding the set's snapshot (d0 | d1) and the walk table -- the tree's
// table with every leaf outside the snapshot replaced by the stand-in row
// n_leaves, whose record the slice writes with sigma -1.  The slice then
// decodes from the same snapshot (vt.d0 = vt.d1 = snapshot) and writes
// records for the set's chunks only: a leaf outside the set is never read
// through the walk table, and any walk that reaches its stand-in re-walks
// the pixel on the tree's own table.
// With a camera plan (the caller holds its lock) the table, snapshot and
// list live in the plan and are rebuilt only when the snapshot changes
// (k_vis_or flags it; k_vis_table then returns at once): a held view's set
// settles after its census, so steady frames skip the table pass.
static int vis_prepare(const vv_tree *t, VisTicket &vt, cudaStream_t st, void **mem, vv_camera_plan *plan = nullptr) {
    *mem = nullptr;
    if (!vt.mark || !vt.d0) return VV_OK;
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t b_table = al((size_t)t->n_internal * 8 * sizeof(int32_t));
    const size_t b_snap = al((size_t)t->vis_words * sizeof(uint32_t));
    const size_t b_list = al((size_t)t->n_leaves * sizeof(int32_t));
    const size_t total = b_table + b_snap + b_list + 256;
    char *base = nullptr;
    bool fresh = true;
    if (plan) {
        if (!plan->vis_mem || plan->vis_cap < total || plan->vis_tree != t->serial) {
            // stream-ordered: frames already queued on this stream keep reading the old table
            if (plan->vis_mem) {
                cudaFreeAsync(plan->vis_mem, st);
                plan->vis_mem = nullptr;
                plan->vis_cap = 0;
            }
            if (cudaMallocAsync(&plan->vis_mem, total, st) != cudaSuccess) {
                cudaGetLastError();
                plan->vis_mem = nullptr;
                return set_error(VV_E_NOMEM, "visible-set walk table (%zu bytes) failed", total);
            }
            plan->vis_cap = total;
            plan->vis_tree = t->serial;
            plan->vis_fresh = true;
        }
        base = static_cast<char *>(plan->vis_mem);
        fresh = plan->vis_fresh;
        plan->vis_fresh = false;
    } else {
        if (cudaMallocAsync(mem, total, st) != cudaSuccess) {
            cudaGetLastError();
            *mem = nullptr;
            return set_error(VV_E_NOMEM, "visible-set walk table (%zu bytes) failed", total);
        }
        base = static_cast<char *>(*mem);
    }
    int32_t *table = reinterpret_cast<int32_t *>(base);
    uint32_t *snap = reinterpret_cast<uint32_t *>(base + b_table);
    int32_t *list = reinterpret_cast<int32_t *>(base + b_table + b_snap);
    int32_t *n_list = reinterpret_cast<int32_t *>(base + b_table + b_snap + b_list);
    int32_t *flags = n_list + 1;  // [changed, blocks done]
    if (fresh)  // the upper rows, once; every snapshot word then counts as changed
        VV_CUDA(cudaMemcpyAsync(table, t->d_child, (size_t)t->n_internal * 8 * sizeof(int32_t),
                                cudaMemcpyDeviceToDevice, st));
    int rc;
    if (plan) {
        VV_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int32_t), st));
        rc = launch_vis_snapshot_diff(vt.d0, vt.d1, snap, t->vis_words, fresh, flags, n_list, st);
    } else {
        VV_CUDA(cudaMemsetAsync(n_list, 0, sizeof(int32_t), st));
        rc = launch_vis_snapshot(vt.d0, vt.d1, snap, t->vis_words, st);
    }
    if (rc) return rc;
    VisTableParams q;
    q.child = t->d_child;
    q.last = t->d_last;
    q.n_last = t->n_last;
    q.vis0 = snap;
    q.vis1 = snap;
    q.stand_in = (int32_t)t->n_leaves;
    q.out = table;
    q.list = list;
    q.n_list = n_list;
    q.changed = plan ? flags : nullptr;
    if ((rc = launch_vis_table(q, st))) return rc;
    vt.d0 = vt.d1 = snap;
    vt.table = table;
    vt.list = list;
    vt.n_list = n_list;
    return VV_OK;
}

int launch_build_slice(const vv_tree *t, int frame, float4 *rec, int rec4, cudaStream_t st, bool render_only,
                       uint8_t *lit = nullptr, const VisTicket *vt = nullptr, bool dark_unread = false) {
    if (t->n_leaves == 0) return VV_OK;
    SliceParams p;
    memset(&p, 0, sizeof(p));
    p.T = t->view;
    p.K = make_consts(t->n_max);
    p.n_frames = 1;
    p.frame[0] = frame;
    p.n_leaves = t->n_leaves;
    p.rec[0] = rec;
    p.rec4 = rec4;
    p.skip_dark = render_only && !t->has_edits;
    p.lit = lit;
    p.dark_unread = dark_unread && lit != nullptr;  // the node mask (built from lit) cuts the dark leaves
    set_slice_masks(t, p);
    return launch_slice_vis(t, p, vt, st);
}

// Transient per-frame slice in the device's stream-ordered pool; freed
// (stream-ordered) when the render call returns.
struct Transient {
    void *mem = nullptr, *vis_mem = nullptr;
    cudaStream_t st = nullptr;
    std::shared_ptr<NodeMask> nmask;
    const int32_t *vis_table = nullptr;  // visible-set walk table (in vis_mem)
    Transient() = default;
    Transient(const Transient &) = delete;
    ~Transient() {
        if (mem) cudaFreeAsync(mem, st);
        if (vis_mem) cudaFreeAsync(vis_mem, st);
    }
};

void pool_setup(int device) {
    static std::once_flag flags[64];
    std::call_once(flags[device & 63], [device] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;  // keep freed slices cached in the pool
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    });
}

// Node masks pay off when a frame leaves large subtrees dark (cfg3: ~90% of
// leaves); they are skipped for trees with edits (an edit can give a dark
// leaf density).  VV_NODE_MASK=0 / 1 forces them off / on (A/B and tests).
static bool mask_wanted(const vv_tree *t) {
    if (!t->mask_ok || t->has_edits || t->n_leaves == 0) return false;
    if (const char *e = getenv("VV_NODE_MASK")) {
        if (e[0] == '0') return false;
        if (e[0] == '1') return true;
    }
    return t->dark_frac >= 0.25f;
}

int alloc_mask(const vv_tree *t, cudaStream_t st, std::shared_ptr<NodeMask> &out) {
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t b_lit = al((size_t)t->n_leaves), b_flag = al((size_t)t->n_internal * 4);
    const size_t total = b_lit + b_flag + (size_t)t->n_internal * 8 * sizeof(int32_t);
    auto m = std::make_shared<NodeMask>();
    if (cudaMallocAsync(&m->mem, total, st) != cudaSuccess) {
        cudaGetLastError();
        m->mem = nullptr;
        return set_error(VV_E_NOMEM, "node mask allocation (%zu bytes) failed", total);
    }
    m->st = st;
    char *b = static_cast<char *>(m->mem);
    m->lit = reinterpret_cast<uint8_t *>(b);
    m->flag = reinterpret_cast<uint32_t *>(b + b_lit);
    m->mask = reinterpret_cast<int32_t *>(b + b_lit + b_flag);
    out = std::move(m);
    return VV_OK;
}

int build_mask(const vv_tree *t, const NodeMask &m, cudaStream_t st) {
    NvtxRange nv("vv:node_mask");
    MaskParams p;
    p.child = t->d_child;
    p.parent = t->d_parent;
    p.last = t->d_last;
    p.upper = t->d_upper;
    p.n_last = t->n_last;
    p.n_upper = t->n_upper;
    p.n_internal = t->n_internal;
    p.lit = m.lit;
    p.flag = m.flag;
    p.mask = m.mask;
    return launch_node_mask(p, st);
}

// Host analysis of the child table at upload (tree_alloc_common).  For a
// proper tree (no node reached twice, leaf rows only below last-level
// nodes) it yields
//   * the node-mask tables: parent of every node, last-level and upper nodes;
//   * the walk-order leaf layout: leaves numbered in BFS order of their
//     last-level parents and child bit (b = x | y<<1 | z<<2), i.e. Morton
//     order -- the device stores payload planes, slice records and lit bytes
//     in this order, rewrites the table's leaf entries to it, and maps rows
//     back to reference ids wherever one leaves the device (leaf_ref);
//   * per kRegionChunk consecutive device rows, the box of their leaf cells
//     (compact in walk order: region renders cull chunks by it).
// Anything else keeps the identity layout and no masks.
struct TreeLayout {
    bool tree = false;
    std::vector<int32_t> parent, last, upper;
    std::vector<int32_t> perm, iperm;  // device row -> reference row, and back
    std::vector<int32_t> child;        // the table with leaf entries in device rows
    std::vector<int4> box;             // (n_box, 2)
};

static void analyze_tree(int depth, int64_t ni, int64_t nl, const int32_t *child, TreeLayout &out) {
    out = TreeLayout();
    std::vector<int32_t> parent((size_t)ni, -2), last, upper;
    std::vector<int32_t> cur{0}, next;
    std::vector<int32_t> cell{0, 0, 0}, ncell;  // cell coordinates of the nodes in cur
    parent[0] = -1;
    for (int L = 0; L < depth && !cur.empty(); ++L) {
        const bool at_last = L + 1 == depth;
        if (at_last) {
            last = cur;
            break;
        }
        next.clear();
        ncell.clear();
        for (size_t i = 0; i < cur.size(); ++i) {
            const int32_t n = cur[i];
            upper.push_back(n);
            for (int b = 0; b < 8; ++b) {
                const int32_t c = child[(size_t)n * 8 + b];
                if (c < 0) continue;
                if (c >= ni || parent[c] != -2) return;  // not a tree
                parent[c] = n;
                next.push_back(c);
                ncell.push_back(2 * cell[3 * i] + (b & 1));
                ncell.push_back(2 * cell[3 * i + 1] + ((b >> 1) & 1));
                ncell.push_back(2 * cell[3 * i + 2] + ((b >> 2) & 1));
            }
        }
        cur.swap(next);
        cell.swap(ncell);
    }
    std::vector<int32_t> iperm((size_t)nl, -1), perm;
    perm.reserve((size_t)nl);
    for (int32_t n : last)
        for (int b = 0; b < 8; ++b) {
            const int32_t r = child[(size_t)n * 8 + b];
            if (r < 0) continue;
            if (r >= nl || iperm[r] >= 0) return;  // out of range or a leaf reached twice: not a tree
            iperm[r] = (int32_t)perm.size();
            perm.push_back(r);
        }
    for (int64_t r = 0; r < nl; ++r)  // rows no node reaches: after the walked ones
        if (iperm[r] < 0) {
            iperm[r] = (int32_t)perm.size();
            perm.push_back((int32_t)r);
        }
    out.child.assign(child, child + (size_t)ni * 8);
    const int64_t nb = (nl + kRegionChunk - 1) / kRegionChunk;
    out.box.resize((size_t)2 * nb);
    for (int64_t k = 0; k < nb; ++k) {
        out.box[2 * k] = make_int4(INT32_MAX, INT32_MAX, INT32_MAX, 0);
        out.box[2 * k + 1] = make_int4(INT32_MIN, INT32_MIN, INT32_MIN, 0);
    }
    for (size_t i = 0; i < last.size(); ++i) {
        const int32_t n = last[i];
        for (int b = 0; b < 8; ++b) {
            int32_t &e = out.child[(size_t)n * 8 + b];
            if (e < 0) continue;
            e = iperm[e];
            const int32_t x = 2 * cell[3 * i] + (b & 1), y = 2 * cell[3 * i + 1] + ((b >> 1) & 1),
                          z = 2 * cell[3 * i + 2] + ((b >> 2) & 1);
            int4 &lo = out.box[2 * (e / kRegionChunk)], &hi = out.box[2 * (e / kRegionChunk) + 1];
            lo.x = std::min(lo.x, x); lo.y = std::min(lo.y, y); lo.z = std::min(lo.z, z);
            hi.x = std::max(hi.x, x); hi.y = std::max(hi.y, y); hi.z = std::max(hi.z, z);
        }
    }
    for (auto &v : parent) v = v == -2 ? -1 : v;
    out.parent.swap(parent);
    out.last.swap(last);
    out.upper.swap(upper);
    out.perm.swap(perm);
    out.iperm.swap(iperm);
    out.tree = true;
}

// Device copies of the layout's tables (mask tables, boxes, leaf_ref).
static int upload_layout(vv_tree *t, const TreeLayout &lay) {
    auto up = [&](void **d, const void *h, size_t bytes) -> int {
        if (!bytes) return VV_OK;
        if (cudaMalloc(d, bytes) != cudaSuccess) {
            cudaGetLastError();
            return set_error(VV_E_NOMEM, "tree layout table allocation failed");
        }
        t->bytes += (int64_t)bytes;
        if (cudaMemcpy(*d, h, bytes, cudaMemcpyHostToDevice) != cudaSuccess)
            return set_error(VV_E_CUDA, "tree layout table copy failed");
        return VV_OK;
    };
    int rc;
    if ((rc = up((void **)&t->d_parent, lay.parent.data(), lay.parent.size() * 4)) ||
        (rc = up((void **)&t->d_last, lay.last.data(), lay.last.size() * 4)) ||
        (rc = up((void **)&t->d_upper, lay.upper.data(), lay.upper.size() * 4)) ||
        (rc = up((void **)&t->d_box, lay.box.data(), lay.box.size() * sizeof(int4))) ||
        (rc = up((void **)&t->d_leaf_ref, lay.perm.data(), lay.perm.size() * 4)) ||
        (rc = up((void **)&t->d_dev_row, lay.iperm.data(), lay.iperm.size() * 4)))
        return rc;
    t->n_last = (int64_t)lay.last.size();
    t->n_upper = (int64_t)lay.upper.size();
    t->n_box = (int64_t)lay.box.size() / 2;
    t->mask_ok = lay.tree && t->n_last > 0;
    return VV_OK;
}

// Leaf-decode mode for a call without a user cache: 0 = per sample (inside
// the render kernel), 1 = per-frame slice pre-pass.  VV_SLICE_AUTO takes the
// pre-pass when the rays that can reach the tree are numerous enough that
// every leaf is likely decoded several times per frame anyway: n_leaves <=
// 4 x rays (measured on tile shares of cfg2 / cfg3 at leaves/rays 3.4: the
// slice pass wins, 0.64 vs 0.66 ms and 1.27 vs 1.41 ms; at 5.1 the shell
// tree decodes faster per sample; the cfg4 performers at 12.7, 2x faster
// per sample).  (Decoding lazily on first visit inside the
// render kernel was measured slower: the claim atomics, release fences and
// sub-warp decode bursts cost more than the skipped decodes.)
int decode_mode(const vv_tree *t, double n_rays, int policy) {
    if (t->n_leaves == 0 || policy == VV_SLICE_PER_SAMPLE) return 0;
    if (policy == VV_SLICE_PER_FRAME) return 1;
    return (double)t->n_leaves <= 4.0 * n_rays ? 1 : 0;
}

// Rays of `cam` that can reach a tree: the screen rectangle bounding its
// cube (corners lo + side {0,1}^3, mapped by the 3x4 affine A when given)
// projected through the camera; every pixel when a corner is not in front
// of the eye.
double cube_footprint(const vv_camera &cam, const double lo[3], double side, const double *A) {
    const double npix = (double)cam.width * cam.height;
    const double *m = cam.c2w;  // row-major 4x4: columns 0..2 = camera axes
    double x0 = 1e300, x1 = -1e300, y0 = 1e300, y1 = -1e300;
    for (int c = 0; c < 8; ++c) {
        double p[3] = {lo[0] + ((c & 1) ? side : 0.0), lo[1] + ((c & 2) ? side : 0.0), lo[2] + ((c & 4) ? side : 0.0)};
        if (A) {
            double q[3];
            for (int r = 0; r < 3; ++r) q[r] = A[4 * r] * p[0] + A[4 * r + 1] * p[1] + A[4 * r + 2] * p[2] + A[4 * r + 3];
            p[0] = q[0];
            p[1] = q[1];
            p[2] = q[2];
        }
        const double d[3] = {p[0] - m[3], p[1] - m[7], p[2] - m[11]};
        double cc[3];
        for (int k = 0; k < 3; ++k) cc[k] = m[k] * d[0] + m[4 + k] * d[1] + m[8 + k] * d[2];  // R^T d
        if (!(cc[2] > 1e-9)) return npix;
        const double px = cam.fx * cc[0] / cc[2] + cam.cx, py = cam.fy * cc[1] / cc[2] + cam.cy;
        x0 = std::min(x0, px);
        x1 = std::max(x1, px);
        y0 = std::min(y0, py);
        y1 = std::max(y1, py);
    }
    const double w = std::max(0.0, std::min(x1, (double)cam.width) - std::max(x0, 0.0));
    const double h = std::max(0.0, std::min(y1, (double)cam.height) - std::max(y0, 0.0));
    return std::min(npix, w * h);
}

// Affine A (3x4) from its inverse's 3x4 rows (scene instances in mode 1).
void affine_from_inverse(const double *inv, double *A) {
    const double a = inv[0], b = inv[1], c = inv[2], d = inv[4], e = inv[5], f = inv[6], g = inv[8], h = inv[9],
                 i = inv[10];
    const double det = a * (e * i - f * h) - b * (d * i - f * g) + c * (d * h - e * g);
    const double M[9] = {(e * i - f * h) / det, (c * h - b * i) / det, (b * f - c * e) / det,
                         (f * g - d * i) / det, (a * i - c * g) / det, (c * d - a * f) / det,
                         (d * h - e * g) / det, (b * g - a * h) / det, (a * e - b * d) / det};
    for (int r = 0; r < 3; ++r) {
        for (int k = 0; k < 3; ++k) A[4 * r + k] = M[3 * r + k];
        A[4 * r + 3] = -(M[3 * r] * inv[3] + M[3 * r + 1] * inv[7] + M[3 * r + 2] * inv[11]);
    }
}

// Transient per-call slice from the stream-ordered pool (freed, stream
// ordered, when the call returns).
// dark_unread: every walk of this slice uses its node mask (image renders,
// no sample counts), so the dark leaves' records need not be written
int build_transient(const vv_tree *t, int frame, cudaStream_t st, SliceView &sv, Transient &tr, bool vis = false,
                    uint64_t view = 0, vv_camera_plan *plan = nullptr, bool dark_unread = false) {
    NvtxRange nv("vv:slice(transient)");
    pool_setup(t->device);
    const int rec4 = slice_rec4(t->S);
    const size_t bytes = (size_t)(t->n_leaves + 1) * rec4 * sizeof(float4);  // + the walk table's stand-in row
    cudaError_t e = cudaMallocAsync(&tr.mem, bytes, st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        tr.mem = nullptr;
        return set_error(VV_E_NOMEM, "transient slice allocation (%zu bytes) failed: %s", bytes,
                         cudaGetErrorString(e));
    }
    tr.st = st;
    sv.rec = reinterpret_cast<float4 *>(tr.mem);
    sv.rec4 = rec4;
    int rc;
    VisTicket vt;
    if (vis_wanted(t) && (rc = vis_begin(t, st, vt, view, vis))) return rc;
    if ((rc = vis_prepare(t, vt, st, &tr.vis_mem, plan))) return rc;
    tr.vis_table = vt.table;
    sv.mark = vt.mark;
    sv.census = vt.census;
    if (mask_wanted(t) && (rc = alloc_mask(t, st, tr.nmask))) return rc;
    rc = launch_build_slice(t, frame, reinterpret_cast<float4 *>(tr.mem), rec4, st, true,
                            tr.nmask ? tr.nmask->lit : nullptr, &vt, dark_unread);
    if (rc || !tr.nmask) return rc;
    return build_mask(t, *tr.nmask, st);
}

// Transient slice for a pixel region: only the leaf chunks whose cell boxes
// can project into the region are sliced (k_chunk_cull -> chunk list ->
// k_build_slice in list mode); the node mask then treats the other leaves as
// dark (their lit bytes are zeroed), which only cuts subtrees the region's
// rays cannot reach.  Trees without chunk boxes slice every chunk.
int build_transient_region(const vv_tree *t, int frame, cudaStream_t st, const vv_camera &cam, int rx0, int ry0,
                           int rx1, int ry1, SliceView &sv, Transient &tr, bool vis = false) {
    NvtxRange nv("vv:slice(region, culled)");
    if (!t->d_box || t->n_leaves == 0) return build_transient(t, frame, st, sv, tr, vis, view_hash(cam));
    pool_setup(t->device);
    const int rec4 = slice_rec4(t->S);
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t b_rec = al((size_t)(t->n_leaves + 1) * rec4 * sizeof(float4));  // + the stand-in row
    const size_t b_bits = al((size_t)((t->n_box + 31) / 32) * 4);  // the list's chunks as bits (visible-set slices)
    const size_t bytes = b_rec + al((size_t)t->n_box * 4) + 256 + b_bits;
    cudaError_t e = cudaMallocAsync(&tr.mem, bytes, st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        tr.mem = nullptr;
        return set_error(VV_E_NOMEM, "transient region slice allocation (%zu bytes) failed", bytes);
    }
    tr.st = st;
    char *m = static_cast<char *>(tr.mem);
    sv.rec = reinterpret_cast<float4 *>(m);
    sv.rec4 = rec4;
    int32_t *list = reinterpret_cast<int32_t *>(m + b_rec);
    int32_t *count = reinterpret_cast<int32_t *>(m + b_rec + al((size_t)t->n_box * 4));
    CullParams c;
    c.box = t->d_box;
    c.n_box = t->n_box;
    c.lo0 = t->view.lo0;
    c.lo1 = t->view.lo1;
    c.lo2 = t->view.lo2;
    c.cell = t->view.side / (double)(1ll << t->depth);
    c.cam = make_cam(cam);
    c.x0 = rx0 + 0.5 - 1.0;  // pixel centres of the region, one pixel of margin
    c.y0 = ry0 + 0.5 - 1.0;
    c.x1 = rx1 - 0.5 + 1.0;
    c.y1 = ry1 - 0.5 + 1.0;
    c.list = list;
    c.count = count;
    int rc = launch_chunk_cull(c, st);
    if (rc) return rc;
    if (mask_wanted(t)) {
        if ((rc = alloc_mask(t, st, tr.nmask))) return rc;
        e = cudaMemsetAsync(tr.nmask->lit, 0, (size_t)t->n_leaves, st);
        if (e != cudaSuccess) return set_error(VV_E_CUDA, "lit memset: %s", cudaGetErrorString(e));
    }
    SliceParams p;
    memset(&p, 0, sizeof(p));
    p.T = t->view;
    p.K = make_consts(t->n_max);
    p.n_frames = 1;
    p.frame[0] = frame;
    p.n_leaves = t->n_leaves;
    p.rec[0] = sv.rec ? const_cast<float4 *>(sv.rec) : nullptr;
    p.rec4 = rec4;
    p.skip_dark = !t->has_edits;
    p.lit = tr.nmask ? tr.nmask->lit : nullptr;
    p.chunk_list = list;
    p.n_list = count;
    VisTicket vt;
    if (vis_wanted(t) && (rc = vis_begin(t, st, vt, view_hash(cam), vis))) return rc;
    if ((rc = vis_prepare(t, vt, st, &tr.vis_mem))) return rc;
    if (vt.list) {  // the set's leaves of this region's chunks only
        uint32_t *bits = reinterpret_cast<uint32_t *>(m + b_rec + al((size_t)t->n_box * 4) + 256);
        VV_CUDA(cudaMemsetAsync(bits, 0, b_bits, st));
        if ((rc = launch_chunk_bits(list, count, bits, t->n_box, st))) return rc;
        p.chunk_bits = bits;
    }
    tr.vis_table = vt.table;
    sv.mark = vt.mark;
    sv.census = vt.census;
    set_slice_masks(t, p);
    if ((rc = launch_slice_vis(t, p, &vt, st))) return rc;
    return tr.nmask ? build_mask(t, *tr.nmask, st) : VV_OK;
}

// Coverage of the tree's leaf chunks for one camera (k_coverage): pixels
// outside it skip their walk (exactly the empty pixel).  VV_COVERAGE=0
// turns it off (A/B runs).  A = instance affine (3x4 rows) or null.
bool coverage_wanted(const vv_tree *t) {
    if (!t->d_box || t->n_box == 0) return false;
    const char *e = getenv("VV_COVERAGE");
    return !(e && e[0] == '0');
}

static size_t coverage_bytes(int width, int height) {
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const int words = (width + 31) / 32, cw = (width + 15) / 16, ch = (height + 15) / 16;
    return 256 + al((size_t)cw * ch) + (size_t)height * words * 4;
}

// mem: coverage_bytes(width, height) of device memory
int build_coverage_into(const vv_tree *t, const CamView &cam, int width, int height, const double *A,
                        cudaStream_t st, char *m, CoverView &cv) {
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const int words = (width + 31) / 32, cw = (width + 15) / 16, ch = (height + 15) / 16;
    const size_t b_hdr = 256, b_coarse = al((size_t)cw * ch), b_fine = (size_t)height * words * 4;
    VV_CUDA(cudaMemsetAsync(m, 0, b_hdr + b_coarse + b_fine, st));
    CoverParams p;
    memset(&p, 0, sizeof(p));
    p.box = t->d_box;
    p.n_box = t->n_box;
    p.lo0 = t->view.lo0;
    p.lo1 = t->view.lo1;
    p.lo2 = t->view.lo2;
    p.cell = t->view.side / (double)(1ll << t->depth);
    p.cam = cam;
    if (A) {
        memcpy(p.A, A, sizeof(p.A));
        p.use_A = 1;
    }
    p.width = width;
    p.height = height;
    p.words = words;
    p.cw = cw;
    p.all = reinterpret_cast<int *>(m);
    p.coarse = reinterpret_cast<uint8_t *>(m + b_hdr);
    p.fine = reinterpret_cast<uint32_t *>(m + b_hdr + b_coarse);
    int rc = launch_coverage(p, st);
    if (rc) return rc;
    cv.fine = p.fine;
    cv.coarse = p.coarse;
    cv.all = p.all;
    cv.words = words;
    cv.cw = cw;
    return VV_OK;
}

int build_coverage(const vv_tree *t, const CamView &cam, int width, int height, const double *A, cudaStream_t st,
                   Transient &tr, CoverView &cv) {
    const size_t bytes = coverage_bytes(width, height);
    pool_setup(t->device);
    if (cudaMallocAsync(&tr.mem, bytes, st) != cudaSuccess) {
        cudaGetLastError();
        tr.mem = nullptr;
        return set_error(VV_E_NOMEM, "coverage allocation failed");
    }
    tr.st = st;
    return build_coverage_into(t, cam, width, height, A, st, static_cast<char *>(tr.mem), cv);
}

// Long segment queue for mostly dark trees (the cfg3 motion tree).  Measured
// at cfg3 with node masks: 0.493 vs 0.502 ms per frame (without masks 2.02
// vs 2.18); VV_LONG_QUEUE=0 / 1 forces the choice (A/B runs).
bool long_queue(const vv_tree *t, const NodeMask *) {
    if (const char *e = getenv("VV_LONG_QUEUE")) return e[0] == '1';
    return t->dark_frac > 0.5f;
}

// Plan buffers for a grid of n_blocks blocks (blocks_x per row): order,
// costs and the two chunk counters, reallocated when the grid changes.
int plan_prepare(vv_camera_plan *plan, int n_blocks, int blocks_x, cudaStream_t st) {
    if (plan->n_blocks == n_blocks && plan->blocks_x == blocks_x) return VV_OK;
    cudaFree(plan->order);
    plan->order = nullptr;
    plan->valid = false;
    const size_t n = (size_t)n_blocks;
    if (cudaMalloc(&plan->order, n * 8 + 256) != cudaSuccess) {
        cudaGetLastError();
        plan->order = nullptr;
        plan->n_blocks = 0;
        return set_error(VV_E_NOMEM, "camera plan allocation failed");
    }
    plan->cost = reinterpret_cast<uint32_t *>(plan->order + n);
    plan->counter = reinterpret_cast<int *>(plan->cost + n);
    plan->n_blocks = n_blocks;
    plan->blocks_x = blocks_x;
    plan->renders = 0;
    // zero once; afterwards the kernel's last warp re-zeroes the counters
    // and k_plan_order the costs it consumes
    VV_CUDA(cudaMemsetAsync(plan->cost, 0, n * 4 + 256, st));
    return VV_OK;
}

// The plan's coverage for (tree, camera): built once per view, reused by
// every frame of it (plan->cov stays empty -- everything covered -- for
// trees without chunk boxes or with VV_COVERAGE=0).
int plan_coverage(vv_camera_plan *plan, const vv_tree *t, const vv_camera &cam, const CamView &cv, cudaStream_t st) {
    if (!coverage_wanted(t)) {
        plan->cov = CoverView{};
        plan->cov_valid = false;
        return VV_OK;
    }
    if (plan->cov_valid && plan->cov_tree == t->serial && memcmp(&plan->cov_cam, &cam, sizeof(cam)) == 0)
        return VV_OK;
    const size_t bytes = coverage_bytes(cam.width, cam.height);
    if (plan->cov_cap < bytes) {
        cudaFree(plan->cov_mem);
        plan->cov_mem = nullptr;
        plan->cov_cap = 0;
        if (cudaMalloc(&plan->cov_mem, bytes) != cudaSuccess) {
            cudaGetLastError();
            plan->cov_mem = nullptr;
            return set_error(VV_E_NOMEM, "coverage allocation failed");
        }
        plan->cov_cap = bytes;
    }
    plan->cov_valid = false;
    int r = build_coverage_into(t, cv, cam.width, cam.height, nullptr, st, static_cast<char *>(plan->cov_mem),
                                plan->cov);
    if (r) return r;
    plan->cov_tree = t->serial;
    plan->cov_cam = cam;
    plan->cov_valid = true;
    return VV_OK;
}

// After a planned launch: the launch order is re-sorted from the costs
// accumulated over the last kPlanResort renders (the first render sorts at
// once) -- a view's block costs change slowly and the sort (one CTA, ~15
// us) is amortised.
// moving: the content's costs move from frame to frame (dark-heavy trees:
// cfg3's kernel 0.283 ms re-sorting every 4th render, 0.301 every 16th);
// otherwise costs summed over more frames order the blocks better (cfg2
// 0.6277 vs 0.6325 ms).  VV_PLAN_RESORT overrides (A/B).
int plan_finish(vv_camera_plan *plan, cudaStream_t st, bool moving = false) {
    static const int env_resort = [] {
        const char *e = getenv("VV_PLAN_RESORT");
        return e ? atoi(e) : 0;
    }();
    const int kPlanResort = env_resort > 0 ? env_resort : (moving ? 4 : 16);
    if (!plan->valid || ++plan->renders >= kPlanResort) {
        int rc = launch_plan_order(plan->cost, plan->n_blocks, plan->order, plan->counter, st);
        if (rc) return rc;
        plan->valid = true;
        plan->renders = 0;
    }
    return VV_OK;
}

// Persistent warp-chunk queue for the camera kernel (k_render_camera, p.work):
// VV_CAM_QUEUE=0 / 1 forces it off / on; by default only region renders
// with a launch order use it.
bool warp_queue(bool ordered) {
    if (const char *e = getenv("VV_CAM_QUEUE")) return e[0] == '1';
    return ordered;
}

// The child table an image render walks: the frame's node mask when one was
// built (dark subtrees cut; bitwise the same pixels), else the tree's own.
const int32_t *image_child(const vv_tree *t, const NodeMask *m) { return m ? m->mask : t->d_child; }

// Bounds-check counter of the debug build (VV_DEBUG_CHECKS), one per device:
// [violations, first violation code, stack high-water slots]; null in
// release builds.
static unsigned *debug_counter(int device) {
    if (!kDebugChecks) return nullptr;
    static std::mutex mu;
    static unsigned *ctr[64] = {};
    std::lock_guard<std::mutex> lk(mu);
    unsigned *&c = ctr[device & 63];
    if (!c && cudaMalloc(&c, 3 * sizeof(unsigned)) == cudaSuccess) cudaMemset(c, 0, 3 * sizeof(unsigned));
    cudaGetLastError();
    return c;
}

// The occupied cells' world box (union of the chunk boxes); the whole cube
// when the table has no walk-order layout.
static void set_occupied_box(vv_tree *t, const TreeLayout &lay) {
    int64_t mn[3] = {INT64_MAX, INT64_MAX, INT64_MAX}, mx[3] = {INT64_MIN, INT64_MIN, INT64_MIN};
    for (size_t k = 0; k + 1 < lay.box.size(); k += 2) {
        const int4 lo = lay.box[k], hi = lay.box[k + 1];
        if (lo.x > hi.x) continue;
        mn[0] = std::min<int64_t>(mn[0], lo.x); mn[1] = std::min<int64_t>(mn[1], lo.y); mn[2] = std::min<int64_t>(mn[2], lo.z);
        mx[0] = std::max<int64_t>(mx[0], hi.x); mx[1] = std::max<int64_t>(mx[1], hi.y); mx[2] = std::max<int64_t>(mx[2], hi.z);
    }
    const double lo[3] = {t->view.lo0, t->view.lo1, t->view.lo2};
    if (!lay.tree) {
        for (int a = 0; a < 3; ++a) {
            t->occ_lo[a] = lo[a];
            t->occ_hi[a] = lo[a] + t->view.side;
        }
        return;
    }
    t->occ_lo[0] = 1.0;  // no occupied cell: empty box
    t->occ_hi[0] = 0.0;
    if (mn[0] > mx[0]) return;
    const double cell = t->view.side / (double)(1ll << t->depth);
    for (int a = 0; a < 3; ++a) {
        t->occ_lo[a] = lo[a] + cell * (double)mn[a];
        t->occ_hi[a] = lo[a] + cell * (double)(mx[a] + 1);
    }
}

// Inclusive pixel rectangle {x0, y0, x1, y1} of the pixels whose ray (from
// `cam`, or from the scene camera through the instance affine A) can reach
// the tree's occupied box: its 8 corners projected, one pixel of margin; the
// whole image when a corner is not in front of the eye; x0 > x1 when empty.
static void occupied_rect(const vv_tree *t, const CamView &c, const double *A, int w, int h, int r[4]) {
    r[0] = 0; r[1] = 0; r[2] = w - 1; r[3] = h - 1;
    if (t->occ_lo[0] > t->occ_hi[0]) {
        r[0] = 1; r[2] = 0;  // nothing to reach
        return;
    }
    double u0 = 1e300, u1 = -1e300, v0 = 1e300, v1 = -1e300;
    for (int k = 0; k < 8; ++k) {
        double p[3] = {(k & 1) ? t->occ_hi[0] : t->occ_lo[0], (k & 2) ? t->occ_hi[1] : t->occ_lo[1],
                       (k & 4) ? t->occ_hi[2] : t->occ_lo[2]};
        if (A) {
            double q[3];
            for (int i = 0; i < 3; ++i) q[i] = A[4 * i] * p[0] + A[4 * i + 1] * p[1] + A[4 * i + 2] * p[2] + A[4 * i + 3];
            p[0] = q[0]; p[1] = q[1]; p[2] = q[2];
        }
        const double dx = p[0] - c.ox, dy = p[1] - c.oy, dz = p[2] - c.oz;
        const double cx = c.r00 * dx + c.r10 * dy + c.r20 * dz;
        const double cy = c.r01 * dx + c.r11 * dy + c.r21 * dz;
        const double cz = c.r02 * dx + c.r12 * dy + c.r22 * dz;
        if (!(cz > 1e-9)) return;  // whole image
        const double u = c.fx * cx / cz + c.cx, v = c.fy * cy / cz + c.cy;
        u0 = std::min(u0, u); u1 = std::max(u1, u); v0 = std::min(v0, v); v1 = std::max(v1, v);
    }
    auto clampd = [](double x) { return std::max(-1e9, std::min(1e9, x)); };
    r[0] = (int)std::max(0.0, std::ceil(clampd(u0) - 1.5));
    r[2] = (int)std::min((double)(w - 1), std::floor(clampd(u1) + 0.5));
    r[1] = (int)std::max(0.0, std::ceil(clampd(v0) - 1.5));
    r[3] = (int)std::min((double)(h - 1), std::floor(clampd(v1) + 0.5));
}

// src_stride: floats per source payload row (0: 2C + 3K; .voct rows with
// edit channels carry 5 more, vv_voct_upload)
int tree_alloc_common(const vv_tree_desc *d, int device, vv_tree **out, bool host_src, int64_t src_stride = 0) {
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
    vv_tree *t = new vv_tree();  // value-initialised: every pointer and count zero
    static std::atomic<uint64_t> next_serial{1};
    t->serial = next_serial++;
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
    const int c4 = (C + 3) / 4;      // float4 chunks of w_sigma / w_gamma
    const int hh4 = (K3 + 3) / 4;    // float4 per w_hh row
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
    if ((rc = alloc((void **)&t->d_sig, (size_t)nrows * c4 * sizeof(float4)))) return fail(rc);
    if ((rc = alloc((void **)&t->d_gam, (size_t)nrows * c4 * sizeof(float4)))) return fail(rc);
    if ((rc = alloc((void **)&t->d_hh, (size_t)nrows * hh4 * sizeof(float4)))) return fail(rc);
    const size_t ab = (size_t)d->frames * C * sizeof(float);
    if ((rc = alloc((void **)&t->d_a, ab))) return fail(rc);
    if ((rc = alloc((void **)&t->d_b, ab))) return fail(rc);
    const cudaMemcpyKind kind = host_src ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    cudaError_t e;
    // host analysis of the table: walk-order leaf layout, mask tables, boxes
    TreeLayout lay;
    {
        std::vector<int32_t> hc;
        const int32_t *hchild = d->node_child;
        if (!host_src) {
            hc.resize((size_t)d->n_internal * 8);
            if ((e = cudaMemcpy(hc.data(), d->node_child, child_b, cudaMemcpyDeviceToHost)) != cudaSuccess)
                return fail(set_error(VV_E_CUDA, "node table copy failed: %s", cudaGetErrorString(e)));
            hchild = hc.data();
        }
        analyze_tree(t->depth, t->n_internal, nl, hchild, lay);
    }
    if (lay.tree) {
        t->h_perm = lay.perm;
        e = cudaMemcpy(t->d_child, lay.child.data(), child_b, cudaMemcpyHostToDevice);
    } else {
        e = cudaMemcpy(t->d_child, d->node_child, child_b, kind);
    }
    if (e != cudaSuccess) return fail(set_error(VV_E_CUDA, "tree copy failed: %s", cudaGetErrorString(e)));
    if ((rc = upload_layout(t, lay))) return fail(rc);
    if (
        (e = cudaMemcpy(t->d_a, d->basis_a, ab, kind)) != cudaSuccess ||
        (e = cudaMemcpy(t->d_b, d->basis_b, ab, kind)) != cudaSuccess)
        return fail(set_error(VV_E_CUDA, "tree copy failed: %s", cudaGetErrorString(e)));
    t->h_a.resize((size_t)d->frames * C);
    t->h_b.resize((size_t)d->frames * C);
    if (ab && ((e = cudaMemcpy(t->h_a.data(), t->d_a, ab, cudaMemcpyDeviceToHost)) != cudaSuccess ||
               (e = cudaMemcpy(t->h_b.data(), t->d_b, ab, cudaMemcpyDeviceToHost)) != cudaSuccess))
        return fail(set_error(VV_E_CUDA, "basis copy failed: %s", cudaGetErrorString(e)));
    if (t->has_edits && nl > 0) {
        if ((rc = alloc((void **)&t->d_edit_rgb, (size_t)nl * sizeof(float4)))) return fail(rc);
        if ((rc = alloc((void **)&t->d_edit_t, (size_t)nl * sizeof(int2)))) return fail(rc);
        if (lay.tree) {  // edit channels in device-row order
            std::vector<float> er((size_t)nl * 4), hr;
            std::vector<int32_t> et((size_t)nl * 2), ht;
            const float *srgb = d->edit_rgb;
            const int32_t *st_ = d->edit_t;
            if (!host_src) {
                hr.resize((size_t)nl * 4);
                ht.resize((size_t)nl * 2);
                if ((e = cudaMemcpy(hr.data(), d->edit_rgb, nl * sizeof(float4), cudaMemcpyDeviceToHost)) !=
                        cudaSuccess ||
                    (e = cudaMemcpy(ht.data(), d->edit_t, nl * sizeof(int2), cudaMemcpyDeviceToHost)) != cudaSuccess)
                    return fail(set_error(VV_E_CUDA, "edit copy failed: %s", cudaGetErrorString(e)));
                srgb = hr.data();
                st_ = ht.data();
            }
            for (int64_t g = 0; g < nl; ++g) {
                const int64_t r = lay.perm[g];
                memcpy(&er[4 * g], srgb + 4 * r, 16);
                memcpy(&et[2 * g], st_ + 2 * r, 8);
            }
            if ((e = cudaMemcpy(t->d_edit_rgb, er.data(), nl * sizeof(float4), cudaMemcpyHostToDevice)) !=
                    cudaSuccess ||
                (e = cudaMemcpy(t->d_edit_t, et.data(), nl * sizeof(int2), cudaMemcpyHostToDevice)) != cudaSuccess)
                return fail(set_error(VV_E_CUDA, "edit copy failed: %s", cudaGetErrorString(e)));
        } else if ((e = cudaMemcpy(t->d_edit_rgb, d->edit_rgb, nl * sizeof(float4), kind)) != cudaSuccess ||
                   (e = cudaMemcpy(t->d_edit_t, d->edit_t, nl * sizeof(int2), kind)) != cudaSuccess) {
            return fail(set_error(VV_E_CUDA, "edit copy failed: %s", cudaGetErrorString(e)));
        }
    }
    // payload rows -> padded planes, chunked through a device staging buffer
    if (nl > 0) {
        const int64_t stride = src_stride > 0 ? src_stride : P;
        const int64_t row_b = stride * (int64_t)sizeof(float);
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
            const float *src = d->leaf_data + r0 * stride;
            if (host_src) {
                if ((e = cudaMemcpy(stage, src, rows * row_b, cudaMemcpyHostToDevice)) != cudaSuccess) {
                    cudaFree(stage);
                    return fail(set_error(VV_E_CUDA, "payload upload failed: %s", cudaGetErrorString(e)));
                }
                src = stage;
            }
            const int lrc = launch_repack(src, rows, (int)stride, C, K3, c4, hh4, nrows, r0, t->d_dev_row, t->d_sig,
                                          t->d_gam, t->d_hh, nullptr);
            if (lrc) {
                if (stage) cudaFree(stage);
                return fail(lrc);
            }
        }
        // PDL invariant (launch_pdl, vv_kernels.cuh): the planes are complete
        // before any render or slice kernel can be launched on this tree
        e = cudaDeviceSynchronize();
        if (stage) cudaFree(stage);
        if (e != cudaSuccess) return fail(set_error(VV_E_CUDA, "repack failed: %s", cudaGetErrorString(e)));
    }
    TreeView &v = t->view;
    v.child = t->d_child;
    v.leaf_ref = t->d_leaf_ref;
    v.n_leaves = nl;
    v.n_internal = t->n_internal;
    v.dbg = debug_counter(device);

    v.sig = t->d_sig;
    v.gam = t->d_gam;
    v.hh = t->d_hh;
    v.lstride = nrows;
    v.edit_rgb = t->d_edit_rgb;
    v.edit_t = t->d_edit_t;
    v.basis_a = t->d_a;
    v.basis_b = t->d_b;
    v.lo0 = d->bbox_lo[0];
    v.lo1 = d->bbox_lo[1];
    v.lo2 = d->bbox_lo[2];
    v.side = d->side;
    {
        int ex = 0;
        const double m = frexp(d->side, &ex);  // side = m 2^ex, m in [0.5, 1)
        v.inv_side = 1.0 / d->side;
        v.side_pow2 = (m == 0.5 && std::isnormal(v.inv_side) && std::isnormal(d->side)) ? 1 : 0;
    }
    v.depth = d->depth;
    v.C = C;
    v.c4 = c4;
    v.hh4 = hh4;
    v.frames = d->frames;
    v.nmax = d->n_max;
    set_occupied_box(t, lay);
    // dark fraction over frames 0, T/2, T-1 (picks the camera kernel's
    // queue threshold; the images are bitwise the same either way)
    if (nl > 0) {
        unsigned long long *cnt = nullptr;
        if (cudaMalloc(&cnt, sizeof(unsigned long long)) == cudaSuccess) {
            const int fr[3] = {0, d->frames / 2, d->frames - 1};
            unsigned long long total = 0;
            int used = 0;
            for (int k = 0; k < 3; ++k) {
                if (k && fr[k] == fr[k - 1]) continue;
                unsigned long long v = 0;
                if (cudaMemset(cnt, 0, sizeof(v)) != cudaSuccess ||
                    launch_count_dark(t->view, fr[k], host_nz_chunks(t, fr[k], 0), nl, cnt, nullptr) != VV_OK ||
                    cudaMemcpy(&v, cnt, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess)
                    break;
                total += v;
                ++used;
            }
            if (used) t->dark_frac = (float)((double)total / ((double)nl * used));
            cudaFree(cnt);
        }
        cudaGetLastError();
    }
    *out = t;
    return VV_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

int vv_debug_checks(int32_t device, int32_t *enabled, uint32_t *violations, uint32_t *first_code,
                    uint32_t *stack_high_water, int32_t reset) {
    if (enabled) *enabled = kDebugChecks ? 1 : 0;
    if (violations) *violations = 0;
    if (first_code) *first_code = 0;
    if (stack_high_water) *stack_high_water = 0;
    if (!kDebugChecks) return VV_OK;
    DeviceGuard g(device);
    unsigned *c = debug_counter(device);
    if (!c) return set_error(VV_E_CUDA, "debug counter unavailable");
    unsigned h[3] = {0, 0, 0};
    VV_CUDA(cudaDeviceSynchronize());
    VV_CUDA(cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost));
    if (violations) *violations = h[0];
    if (first_code) *first_code = h[1];
    if (stack_high_water) *stack_high_water = h[2];
    if (reset) VV_CUDA(cudaMemset(c, 0, sizeof(h)));
    return VV_OK;
}

int vv_device_count(int *count) {
    cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) {
        *count = 0;
        return set_error(VV_E_CUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
    }
    return VV_OK;
}

int vv_tree_upload(const vv_tree_desc *host, int device, vv_tree **out) {
    NvtxRange nv("vv:tree_upload");
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
    cudaFree(t->d_gam);
    cudaFree(t->d_hh);
    cudaFree(t->d_edit_rgb);
    cudaFree(t->d_edit_t);
    cudaFree(t->d_a);
    cudaFree(t->d_b);
    cudaFree(t->d_parent);
    cudaFree(t->d_last);
    cudaFree(t->d_upper);
    cudaFree(t->d_box);
    cudaFree(t->d_leaf_ref);
    cudaFree(t->d_dev_row);
    cudaFree(t->d_vis);
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

int vv_tree_leaf_order(const vv_tree *t, int32_t *ref_rows) {
    if (!t || !ref_rows) return set_error(VV_E_INVALID, "null argument");
    if (t->h_perm.empty()) {
        for (int64_t g = 0; g < t->n_leaves; ++g) ref_rows[g] = (int32_t)g;
    } else {
        memcpy(ref_rows, t->h_perm.data(), (size_t)t->n_leaves * sizeof(int32_t));
    }
    return VV_OK;
}

int vv_tree_dark_fraction(const vv_tree *t, float *dark_frac) {
    if (!t || !dark_frac) return set_error(VV_E_INVALID, "null argument");
    *dark_frac = t->dark_frac;
    return VV_OK;
}

int vv_profile_split_event(void *event) {
    split_event = static_cast<cudaEvent_t>(event);
    return VV_OK;
}

int vv_tree_visible_count(const vv_tree *t, int64_t *n_visible, int64_t *n_chunks, void *stream) {
    if (!t || !n_visible) return set_error(VV_E_INVALID, "null argument");
    *n_visible = 0;
    if (n_chunks) *n_chunks = 0;
    std::lock_guard<std::mutex> lk(t->vis_mu);
    if (!t->d_vis) return VV_OK;
    DeviceGuard g(t->device);
    std::vector<uint32_t> h(2 * (size_t)t->vis_words);
    VV_CUDA(cudaMemcpyAsync(h.data(), t->d_vis, h.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                            (cudaStream_t)stream));
    VV_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    int64_t n = 0, c = 0;
    for (int64_t w = 0; w < t->vis_words; w += 2) {
        const uint64_t v = ((uint64_t)(h[w + 1] | h[t->vis_words + w + 1]) << 32) | (h[w] | h[t->vis_words + w]);
        n += __builtin_popcountll(v);
        c += v != 0;
    }
    *n_visible = n;
    if (n_chunks) *n_chunks = c;
    return VV_OK;
}

int vv_tree_visible_bits(const vv_tree *t, uint32_t *out, int64_t n_words, void *stream) {
    if (!t || !out) return set_error(VV_E_INVALID, "null argument");
    const int64_t need = ((t->n_leaves + 63) / 64) * 2;
    if (n_words < need) return set_error(VV_E_INVALID, "%lld words for %lld", (long long)n_words, (long long)need);
    std::lock_guard<std::mutex> lk(t->vis_mu);
    if (!t->d_vis) {
        memset(out, 0, (size_t)need * sizeof(uint32_t));
        return VV_OK;
    }
    DeviceGuard g(t->device);
    std::vector<uint32_t> h(2 * (size_t)t->vis_words);
    VV_CUDA(cudaMemcpyAsync(h.data(), t->d_vis, h.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                            (cudaStream_t)stream));
    VV_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    for (int64_t w = 0; w < need; ++w) out[w] = h[w] | h[t->vis_words + w];
    return VV_OK;
}

int vv_slice_build(const vv_tree *t, int32_t frame, void *stream, vv_slice **out) {
    NvtxRange nv("vv:slice_build");
    if (!t || !out) return set_error(VV_E_INVALID, "null argument");
    int rc = check_frame(t, frame);
    if (rc) return rc;
    DeviceGuard g(t->device);
    vv_slice *s = new vv_slice();
    s->tree = t;
    s->device = t->device;
    s->frame = frame;
    s->n_leaves = t->n_leaves;
    s->rec4 = slice_rec4(t->S);
    const int64_t nrows = std::max<int64_t>(t->n_leaves, 1);
    s->stream = (cudaStream_t)stream;
    pool_setup(t->device);
    if (cudaMallocAsync(&s->d_rec, nrows * s->rec4 * sizeof(float4), s->stream) != cudaSuccess) {
        cudaGetLastError();
        s->d_rec = nullptr;
        vv_slice_free(s);
        return set_error(VV_E_NOMEM, "slice allocation failed");
    }
    if (mask_wanted(t) && (rc = alloc_mask(t, s->stream, s->nmask))) {
        vv_slice_free(s);
        return rc;
    }
    rc = launch_build_slice(t, frame, s->d_rec, s->rec4, (cudaStream_t)stream, false,
                            s->nmask ? s->nmask->lit : nullptr);
    if (!rc && s->nmask) rc = build_mask(t, *s->nmask, s->stream);
    if (rc) {
        vv_slice_free(s);
        return rc;
    }
    *out = s;
    return VV_OK;
}

int vv_slice_build_multi(const vv_tree *t, int32_t n_frames, const int32_t *frames, void *stream, vv_slice **out) {
    return vv_slice_build_frames(t, n_frames, frames, 0, stream, out);
}

static int slice_build_frames_impl(const vv_tree *t, int32_t n_frames, const int32_t *frames, int32_t flags,
                                   vv_camera_plan *plan, void *stream, vv_slice **out);

int vv_slice_build_frames(const vv_tree *t, int32_t n_frames, const int32_t *frames, int32_t flags, void *stream,
                          vv_slice **out) {
    return slice_build_frames_impl(t, n_frames, frames, flags, nullptr, stream, out);
}

int vv_slice_build_visible(const vv_tree *t, int32_t frame, vv_camera_plan *plan, void *stream, vv_slice **out) {
    if (!plan) return set_error(VV_E_INVALID, "null camera plan");
    std::lock_guard<std::mutex> lk(plan->mu);
    if (plan->device != t->device) return set_error(VV_E_INVALID, "camera plan belongs to another device");
    return slice_build_frames_impl(t, 1, &frame, VV_SLICE_RENDER_ONLY | VV_SLICE_VISIBLE, plan, stream, out);
}

static int slice_build_frames_impl(const vv_tree *t, int32_t n_frames, const int32_t *frames, int32_t flags,
                                   vv_camera_plan *plan, void *stream, vv_slice **out) {
    NvtxRange nv("vv:slice_build_frames");
    if (!t || !frames || !out) return set_error(VV_E_INVALID, "null argument");
    if (flags & ~(VV_SLICE_RENDER_ONLY | VV_SLICE_VISIBLE))
        return set_error(VV_E_INVALID, "unknown slice flags 0x%x", flags);
    if (n_frames < 1 || n_frames > kMaxMulti)
        return set_error(VV_E_UNSUPPORTED, "%d frames per slice pass (1..%d)", n_frames, kMaxMulti);
    if ((flags & VV_SLICE_VISIBLE) && (n_frames != 1 || !(flags & VV_SLICE_RENDER_ONLY)))
        return set_error(VV_E_INVALID, "VV_SLICE_VISIBLE takes one frame and VV_SLICE_RENDER_ONLY");
    for (int f = 0; f < n_frames; ++f) {
        int rc = check_frame(t, frames[f]);
        if (rc) return rc;
        out[f] = nullptr;
    }
    DeviceGuard g(t->device);
    pool_setup(t->device);
    SliceParams p;
    memset(&p, 0, sizeof(p));
    p.T = t->view;
    p.K = make_consts(t->n_max);
    p.n_frames = n_frames;
    p.n_leaves = t->n_leaves;
    p.rec4 = slice_rec4(t->S);
    const int64_t nrows = std::max<int64_t>(t->n_leaves, 1) + ((flags & VV_SLICE_VISIBLE) ? 1 : 0);  // + stand-in row
    auto fail = [&](int rc) {
        for (int f = 0; f < n_frames; ++f) {
            vv_slice_free(out[f]);
            out[f] = nullptr;
        }
        return rc;
    };
    for (int f = 0; f < n_frames; ++f) {
        vv_slice *s = new vv_slice();
        s->tree = t;
        s->device = t->device;
        s->frame = frames[f];
        s->n_leaves = t->n_leaves;
        s->rec4 = p.rec4;
        s->stream = (cudaStream_t)stream;
        s->render_only = (flags & VV_SLICE_RENDER_ONLY) != 0;
        out[f] = s;
        if (cudaMallocAsync(&s->d_rec, nrows * s->rec4 * sizeof(float4), s->stream) != cudaSuccess) {
            cudaGetLastError();
            s->d_rec = nullptr;
            return fail(set_error(VV_E_NOMEM, "slice allocation failed"));
        }
        p.frame[f] = frames[f];
        p.rec[f] = s->d_rec;
    }
    if (t->n_leaves == 0) return VV_OK;
    p.skip_dark = (flags & VV_SLICE_RENDER_ONLY) && !t->has_edits;
    VisTicket vt;
    if (flags & VV_SLICE_VISIBLE) {
        int vrc = vis_begin(t, (cudaStream_t)stream, vt);
        if (vrc) return fail(vrc);
        out[0]->visible = vt.mark != nullptr;
        out[0]->vis_mark = vt.mark;
        out[0]->vis_census = vt.census;
        if ((vrc = vis_prepare(t, vt, (cudaStream_t)stream, &out[0]->d_vis_mem, plan))) return fail(vrc);
        out[0]->vis_table = vt.table;

    }
    set_slice_masks(t, p);
    // one node mask for the group: a subtree is kept if lit in any of its
    // frames (each frame's dark leaves still read sigma 0 from its record)
    std::shared_ptr<NodeMask> nm;
    int rc;
    if (mask_wanted(t) && (rc = alloc_mask(t, (cudaStream_t)stream, nm))) return fail(rc);
    p.lit = nm ? nm->lit : nullptr;
    rc = launch_slice_vis(t, p, &vt, (cudaStream_t)stream);
    if (!rc && nm) rc = build_mask(t, *nm, (cudaStream_t)stream);
    if (rc) return fail(rc);
    for (int f = 0; f < n_frames; ++f) out[f]->nmask = nm;
    return VV_OK;
}

int vv_slice_free(vv_slice *s) {
    if (!s) return VV_OK;
    DeviceGuard g(s->device);
    if (s->d_rec) cudaFreeAsync(s->d_rec, s->stream);
    if (s->d_vis_mem) cudaFreeAsync(s->d_vis_mem, s->stream);
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
    if (s->render_only && q)
        return set_error(VV_E_INVALID, "a render-only slice has no colour for dark leaves; build it without "
                                       "VV_SLICE_RENDER_ONLY to export q");
    if (s->visible)
        return set_error(VV_E_INVALID, "a VV_SLICE_VISIBLE slice holds -sigma outside the visible set: not "
                                       "exportable");
    DeviceGuard g(s->device);
    cudaStream_t st = (cudaStream_t)stream;
    const int S3 = 3 * s->tree->S;
    const size_t pitch = (size_t)s->rec4 * sizeof(float4);
    if (s->n_leaves == 0) return VV_OK;
    if (s->tree->d_dev_row)  // records are in device-row order: gather into reference order
        return launch_slice_export(s->d_rec, s->rec4, S3, s->n_leaves, s->tree->d_dev_row, sigma, q, st);
    if (sigma)
        VV_CUDA(cudaMemcpy2DAsync(sigma, sizeof(double), reinterpret_cast<const char *>(s->d_rec) + pitch - 8, pitch,
                                  sizeof(double), s->n_leaves, cudaMemcpyDeviceToDevice, st));
    if (q)
        VV_CUDA(cudaMemcpy2DAsync(q, S3 * sizeof(float), s->d_rec, pitch, S3 * sizeof(float), s->n_leaves,
                                  cudaMemcpyDeviceToDevice, st));
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
    if (cache && cache->visible)
        return set_error(VV_E_INVALID, "VV_SLICE_VISIBLE slices feed camera renders only");
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
    const size_t smem = stack_bytes(t->depth, wide, true);
    const unsigned grid = (unsigned)((n + kBlock - 1) / kBlock);
    cudaStream_t st = (cudaStream_t)stream;
    Transient tr;
    const int mode = cache ? 1 : decode_mode(t, (double)n, opts.frame_slice);
    if (!cache && mode != 0) {
        int r = build_transient(t, frame, st, p.S, tr);
        if (r) return r;
    }
    // plain image accumulators may walk the frame's node mask; counts and
    // visit lists need the reference's full walk (VV_STATS_MASKED=1: counts
    // of the masked walk itself -- instrumentation for roofline accounting)
    const char *sm = getenv("VV_STATS_MASKED");
    if (!visits && ((!used && !pops && !shaded) || (sm && sm[0] == '1')))
        p.T.child = image_child(t, cache ? cache->nmask.get() : tr.nmask.get());
    return launch_rays(t->n_max, mode, t->has_edits, wide, visits, p, grid, smem, st);
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
                              int tile, int shard, int n_shards, int peer, void *stream, int32_t *used = nullptr,
                              const int32_t *rect = nullptr, const int32_t *block_order = nullptr,
                              vv_camera_plan *plan = nullptr, unsigned *band_done = nullptr, int band_rows = 0,
                              bool force_queue = false, bool natural_order = false, int band_first = 0) {
    NvtxRange nv("vv:render_camera");
    if (!t || !cam) return set_error(VV_E_INVALID, "null argument");
    int rc = check_frame(t, frame);
    if (rc) return rc;
    if ((rc = check_cache(t, cache, frame))) return rc;
    if (cam->width <= 0 || cam->height <= 0) return set_error(VV_E_INVALID, "bad camera size");
    if (tile && (tile <= 0 || tile % 16 != 0 || n_shards < 1 || shard < 0 || shard >= n_shards))
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
    p.used = used;
    unsigned grid_blocks = 0;
    double share = 1.0;  // fraction of the frame's pixels this call renders
    p.peer = peer;
    if (tile) {
        p.packed = packed;
        p.tile = tile;
        p.shard = shard;
        p.n_shards = n_shards;
        p.tiles_x = (cam->width + tile - 1) / tile;
        const int tiles_y = (cam->height + tile - 1) / tile;
        const int total = p.tiles_x * tiles_y;
        const int mine = total > shard ? (total - shard + n_shards - 1) / n_shards : 0;
        if (mine == 0) return VV_OK;
        if (tile % kTW || tile % kTH) return set_error(VV_E_INVALID, "tile must be a multiple of %d", kTW);
        grid_blocks = (unsigned)mine * (unsigned)((tile / kTW) * (tile / kTH));
        share = (double)mine / (double)total;
    } else {
        p.rx0 = rect ? rect[0] : 0;
        p.ry0 = rect ? rect[1] : 0;
        p.rx1 = rect ? rect[2] : cam->width;
        p.ry1 = rect ? rect[3] : cam->height;
        if (p.rx0 < 0 || p.ry0 < 0 || p.rx1 > cam->width || p.ry1 > cam->height)
            return set_error(VV_E_INVALID, "region [%d, %d) x [%d, %d) outside the %dx%d image", p.rx0, p.rx1, p.ry0,
                             p.ry1, cam->width, cam->height);
        if (p.rx1 <= p.rx0 || p.ry1 <= p.ry0) return VV_OK;  // empty region
        p.blocks_x = (p.rx1 - p.rx0 + kTW - 1) / kTW;
        grid_blocks = (unsigned)p.blocks_x * (unsigned)((p.ry1 - p.ry0 + kTH - 1) / kTH);
        p.block_order = block_order;
        int rr[4];
        occupied_rect(t, p.cam, nullptr, cam->width, cam->height, rr);
        p.cx0 = rr[0]; p.cy0 = rr[1]; p.cx1 = rr[2]; p.cy1 = rr[3];
        p.band_done = band_done;
        p.band_rows = band_rows;
        p.band_first = band_first;
    }
    const bool wide = t->depth > kNarrowDepth;
    const size_t smem = stack_bytes(t->depth, wide);
    cudaStream_t st = (cudaStream_t)stream;
    Transient tr, tq;
    std::unique_lock<std::mutex> plan_lock;
    if (plan) {
        if (tile) return set_error(VV_E_INVALID, "camera plans render images or regions, not packed tiles");
        if (plan->device != t->device) return set_error(VV_E_INVALID, "camera plan belongs to another device");
        plan_lock = std::unique_lock<std::mutex>(plan->mu);
        int prc = plan_prepare(plan, (int)grid_blocks, p.blocks_x, st);
        if (prc) return prc;
        p.work = plan->counter;
        p.n_work = (int)grid_blocks * kWarpsPerTile;
        // natural order: bands finish top to bottom (banded host copies)
        p.block_order = plan->valid && !natural_order ? plan->order : nullptr;
        p.block_cost = plan->cost;
    } else if (!tile && (force_queue || warp_queue(block_order != nullptr))) {
        // persistent warps over the warp chunks: the chunk counter is zeroed
        // before the slice pass so the render keeps its PDL overlap
        pool_setup(t->device);
        if (cudaMallocAsync(&tq.mem, 256, st) != cudaSuccess) {
            cudaGetLastError();
            tq.mem = nullptr;
            return set_error(VV_E_NOMEM, "work counter allocation failed");
        }
        tq.st = st;
        VV_CUDA(cudaMemsetAsync(tq.mem, 0, 2 * sizeof(int), st));
        p.work = static_cast<int *>(tq.mem);
        p.n_work = (int)grid_blocks * kWarpsPerTile;
    }
    // coverage (planned renders: built once per tree and camera, ~30 us,
    // then reused by every frame of that view -- per call it costs about
    // what it saves, measured on cfg2 / cfg3)
    if (plan) {
        int r = plan_coverage(plan, t, *cam, p.cam, st);
        if (r) return r;
        p.cov = plan->cov;
    }
    const double lo[3] = {t->view.lo0, t->view.lo1, t->view.lo2};
    // a region render's slice covers only the chunks its pixels can reach,
    // so it is decided on the whole frame's footprint
    int mode = cache ? 1
                     : decode_mode(t, (rect ? 1.0 : share) * cube_footprint(*cam, lo, t->view.side, nullptr),
                                   opts.frame_slice);
    // visible-set slices (image / region mode): the deferred-chunk list of
    // k_camera_rewalk, zeroed before the slice pass (the PDL chain stays)
    // (not for small regions: a band's culled slice is already small, and a
    // walk table costs a whole-tree pass per band -- cfg2 in bands of 1/2 /
    // 1/4 / 1/8 of the frame: 0.459 / 0.350 / 0.234 ms with it, 0.526 /
    // 0.339 / 0.230 without; tools/tile_modes.py)
    const bool big = !rect || (double)(p.rx1 - p.rx0) * (p.ry1 - p.ry0) >= 0.4 * cam->width * cam->height;
    Transient td;
    if (!tile && ((cache && cache->visible) || (!cache && big && mode != 0 && vis_may_use(t, view_hash(*cam))))) {
        pool_setup(t->device);
        const size_t cap = (size_t)grid_blocks * kWarpsPerTile;
        if (cudaMallocAsync(&td.mem, 256 + cap * sizeof(int4), st) != cudaSuccess) {
            cudaGetLastError();
            td.mem = nullptr;
            return set_error(VV_E_NOMEM, "deferred-chunk list allocation failed");
        }
        td.st = st;
        VV_CUDA(cudaMemsetAsync(td.mem, 0, sizeof(int), st));
        p.n_deferred = static_cast<int *>(td.mem);
        p.deferred = reinterpret_cast<int4 *>(static_cast<char *>(td.mem) + 256);
    }
    if (!cache && mode != 0) {
        const bool vis = p.deferred != nullptr;
        int r = rect ? build_transient_region(t, frame, st, *cam, p.rx0, p.ry0, p.rx1, p.ry1, p.S, tr, vis)
                     : build_transient(t, frame, st, p.S, tr, vis, view_hash(*cam), plan, used == nullptr);
        if (r) return r;
    }
    // sample counts report the reference's full walk: the tree's own table
    const NodeMask *nm = used ? nullptr : (cache ? cache->nmask.get() : tr.nmask.get());
    p.T.child = image_child(t, nm);
    if (p.S.mark && !p.deferred) return set_error(VV_E_INVALID, "visible-set slices: image or region renders only");
    // a set in use: the walk table hides the leaves outside it (their
    // stand-in row n_leaves defers the pixel); the re-walk keeps the tree's table
    if (const int32_t *vt_table = cache ? cache->vis_table : tr.vis_table) {
        p.child_full = p.T.child;
        p.T.child = vt_table;
        p.T.n_leaves = t->n_leaves + 1;  // the stand-in row is a valid record row
    }
    const bool vis = p.S.mark != nullptr;
    if (split_event) {
        cudaEventRecord(split_event, st);
        split_event = nullptr;
    }
    rc = launch_camera(t->n_max, mode, t->has_edits, wide, p, grid_blocks, smem, st, long_queue(t, nm), vis);
    if (!rc && vis) rc = launch_camera_rewalk(t->n_max, wide, p, st);
    if (rc || !plan) return rc;
    return plan_finish(plan, st, mask_wanted(t));
}

// ---- render straight to the host: banded device->host copies behind the render
typedef CUresult (*WaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

static WaitValue32Fn wait_value32() {  // the driver's cuStreamWaitValue32 (stream memory ops)
    static WaitValue32Fn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        // the CUDA 12 ABI (cuStreamWaitValue32_v2): stream memory ops are
        // enabled by default (the v1 entry needs a driver module option)
        if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &f, 12000, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<WaitValue32Fn>(f);
        cudaGetLastError();
    });
    return fn;
}

// Per (device, caller stream): a non-blocking copy stream and the band
// counters (plain cudaMalloc: stream memory ops do not accept pool memory).
// Calls on one caller stream are ordered, and each ends with that stream
// waiting for its copies, so the counters are reused safely.
struct HostCopyState {
    int device;
    cudaStream_t caller, copy[2];  // bands alternate between two copy streams (per-copy setup overlaps)
    unsigned *counters;
    int capacity;
    cudaEvent_t ready, copied[2];  // reused by every call on this caller stream
};

static HostCopyState *host_copy_state(int device, cudaStream_t caller, int n_bands) {
    static std::mutex mu;
    static std::deque<HostCopyState> states;  // stable addresses: callers keep the pointer
    std::lock_guard<std::mutex> lk(mu);
    HostCopyState *st = nullptr;
    for (auto &e : states)
        if (e.device == device && e.caller == caller) st = &e;
    if (!st) {
        HostCopyState e{device, caller, {nullptr, nullptr}, nullptr, 0, nullptr, {nullptr, nullptr}};
        for (int k = 0; k < 2; ++k)
            if (cudaStreamCreateWithFlags(&e.copy[k], cudaStreamNonBlocking) != cudaSuccess ||
                cudaEventCreateWithFlags(&e.copied[k], cudaEventDisableTiming) != cudaSuccess) {
                cudaGetLastError();
                return nullptr;
            }
        if (cudaEventCreateWithFlags(&e.ready, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        states.push_back(e);
        st = &states.back();
    }
    if (st->capacity < n_bands) {
        cudaStreamSynchronize(st->copy[0]);
        cudaStreamSynchronize(st->copy[1]);
        cudaFree(st->counters);
        st->counters = nullptr;
        st->capacity = 0;
        if (cudaMalloc(&st->counters, (size_t)n_bands * sizeof(unsigned)) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        st->capacity = n_bands;
    }
    return st;
}

int vv_render_camera_to_host(const vv_tree *t, int32_t frame, const vv_slice *cache, const vv_render_opts *opts,
                             const vv_camera *cam, float *device_planes, float *host_planes, vv_camera_plan *plan,
                             void *stream) {
    NvtxRange nv("vv:render_camera_to_host");
    if (!t || !cam || !device_planes || !host_planes) return set_error(VV_E_INVALID, "null argument");
    if (cam->width <= 0 || cam->height <= 0) return set_error(VV_E_INVALID, "bad camera size");
    DeviceGuard g(t->device);
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t hw = (int64_t)cam->width * cam->height;
    float *rgb = device_planes, *alpha = device_planes + 3 * hw, *depth = device_planes + 4 * hw;
    WaitValue32Fn wait = wait_value32();
    // bands of 136 rows (whole camera-block rows), 8 at 1080p: measured
    // 1.28 ms per cfg2 render() -> host vs 1.34 / 1.36 for 272 / 64 rows and
    // 1.80 unbanded (VV_HOST_BAND_ROWS overrides: A/B runs)
    int band_rows = std::max(kTH, (136 / kTH) * kTH);
    if (const char *e = getenv("VV_HOST_BAND_ROWS")) band_rows = std::max(kTH, (atoi(e) / kTH) * kTH);
    // a shorter first band starts the copies sooner: 64 rows 1.177 vs 1.188 ms
    // with 136, 1.185 with 40 (VV_HOST_BAND_FIRST overrides)
    int band_first = std::max(kTH, (64 / kTH) * kTH);
    if (const char *e = getenv("VV_HOST_BAND_FIRST")) band_first = std::max(kTH, (atoi(e) / kTH) * kTH);
    band_first = std::min(band_first, band_rows);
    const int n_bands = cam->height <= band_first ? 1 : 1 + (cam->height - band_first + band_rows - 1) / band_rows;
    HostCopyState *hs = wait ? host_copy_state(t->device, st, n_bands) : nullptr;
    if (!hs) {  // no stream memory ops: render, then one copy
        int rc = render_camera_impl(t, frame, cache, opts, cam, rgb, alpha, depth, nullptr, 0, 0, 1, 0, stream);
        if (rc) return rc;
        VV_CUDA(cudaMemcpyAsync(host_planes, device_planes, (size_t)hw * 5 * sizeof(float), cudaMemcpyDeviceToHost,
                                st));
        return VV_OK;
    }
    // VV_HOST_COPY_STREAMS=1: every band on one copy stream (A/B)
    const char *ncs_env = getenv("VV_HOST_COPY_STREAMS");
    const int ncs = (ncs_env && ncs_env[0] == '1') ? 1 : 2;
    unsigned *band_done = hs->counters;
    VV_CUDA(cudaMemsetAsync(band_done, 0, (size_t)n_bands * sizeof(unsigned), st));
    cudaEvent_t ready = hs->ready, *copied = hs->copied;
    cudaEventRecord(ready, st);  // counters zeroed, earlier work on the caller's stream ordered
    for (int k = 0; k < ncs; ++k) cudaStreamWaitEvent(hs->copy[k], ready, 0);
    // persistent warps in row-major order: bands finish top to bottom (a
    // plan contributes its counters and cached coverage, not its cost order)
    int rc = render_camera_impl(t, frame, cache, opts, cam, rgb, alpha, depth, nullptr, 0, 0, 1, 0, stream, nullptr,
                                nullptr, nullptr, plan, band_done, band_rows, true, true, band_first);
    if (rc) {
        cudaStreamWaitEvent(st, ready, 0);
        return rc;
    }
    const int blocks_x = (cam->width + kTW - 1) / kTW;
    const size_t W = (size_t)cam->width;
    for (int b = 0; b < n_bands && !rc; ++b) {
        const int y0 = b == 0 ? 0 : band_first + (b - 1) * band_rows;
        const int y1 = std::min(cam->height, b == 0 ? band_first : y0 + band_rows);
        const unsigned target = (unsigned)(((y1 - y0 + kTH - 1) / kTH) * blocks_x * kWarpsPerTile);
        cudaStream_t cs = hs->copy[b % ncs];
        const CUresult wr = wait(reinterpret_cast<CUstream>(cs), reinterpret_cast<CUdeviceptr>(band_done + b), target,
                                 CU_STREAM_WAIT_VALUE_GEQ);
        if (wr != CUDA_SUCCESS) {
            rc = set_error(VV_E_CUDA, "cuStreamWaitValue32 failed (CUresult %d)", (int)wr);
            break;
        }
        const size_t px0 = (size_t)y0 * W, npx = (size_t)(y1 - y0) * W;
        // rgb rows, then the alpha and depth rows as one 2-row copy (the planes are hw floats apart)
        if (cudaMemcpyAsync(host_planes + 3 * px0, rgb + 3 * px0, npx * 12, cudaMemcpyDeviceToHost, cs) != cudaSuccess ||
            cudaMemcpy2DAsync(host_planes + 3 * hw + px0, (size_t)hw * 4, alpha + px0, (size_t)hw * 4, npx * 4, 2,
                              cudaMemcpyDeviceToHost, cs) != cudaSuccess)
            rc = set_error(VV_E_CUDA, "band copy failed");
    }
    for (int k = 0; k < ncs; ++k) {  // the caller's stream: frame on the host, counters free again
        cudaEventRecord(copied[k], hs->copy[k]);
        cudaStreamWaitEvent(st, copied[k], 0);
    }
    return rc;
}

int vv_camera_plan_create(int32_t device, vv_camera_plan **out) {
    if (!out) return set_error(VV_E_INVALID, "null argument");
    vv_camera_plan *p = new vv_camera_plan();
    p->device = device;
    *out = p;
    return VV_OK;
}

int vv_camera_plan_free(vv_camera_plan *plan) {
    if (!plan) return VV_OK;
    DeviceGuard g(plan->device);
    cudaDeviceSynchronize();  // a render may still read the order
    cudaFree(plan->order);
    cudaFree(plan->cov_mem);
    cudaFree(plan->vis_mem);
    delete plan;
    return VV_OK;
}

int vv_render_camera_planned(const vv_tree *t, int32_t frame, const vv_slice *cache, const vv_render_opts *opts,
                             const vv_camera *cam, const int32_t *region, vv_camera_plan *plan, float *rgb,
                             float *alpha, float *depth, int32_t peer, void *stream) {
    if (!plan) return set_error(VV_E_INVALID, "null camera plan");
    if (!rgb && !alpha && !depth) return set_error(VV_E_INVALID, "null image planes");
    return render_camera_impl(t, frame, cache, opts, cam, rgb, alpha, depth, nullptr, 0, 0, 1, peer ? 1 : 0, stream,
                              nullptr, region, nullptr, plan);
}

int vv_render_camera(const vv_tree *t, int32_t frame, const vv_slice *cache, const vv_render_opts *opts,
                     const vv_camera *cam, float *rgb, float *alpha, float *depth, void *stream) {
    return render_camera_impl(t, frame, cache, opts, cam, rgb, alpha, depth, nullptr, 0, 0, 1, 0, stream);
}

int vv_render_camera_region(const vv_tree *t, int32_t frame, const vv_slice *cache, const vv_render_opts *opts,
                            const vv_camera *cam, const int32_t *region, const int32_t *block_order, float *rgb,
                            float *alpha, float *depth, int32_t peer, void *stream) {
    if (!region) return set_error(VV_E_INVALID, "null region");
    if (!rgb && !alpha && !depth) return set_error(VV_E_INVALID, "null image planes");
    return render_camera_impl(t, frame, cache, opts, cam, rgb, alpha, depth, nullptr, 0, 0, 1, peer ? 1 : 0, stream,
                              nullptr, region, block_order);
}

int vv_camera_block_shape(int32_t *width, int32_t *height) {
    if (!width || !height) return set_error(VV_E_INVALID, "null argument");
    *width = kTW;
    *height = kTH;
    return VV_OK;
}

int vv_render_camera_counts(const vv_tree *t, int32_t frame, const vv_slice *cache, const vv_render_opts *opts,
                            const vv_camera *cam, float *rgb, float *alpha, float *depth, int32_t *sample_count,
                            void *stream) {
    if (!sample_count) return set_error(VV_E_INVALID, "null sample_count");
    return render_camera_impl(t, frame, cache, opts, cam, rgb, alpha, depth, nullptr, 0, 0, 1, 0, stream,
                              sample_count);
}

int vv_camera_decode_mode(const vv_tree *t, const vv_camera *cam, const vv_render_opts *o, int32_t *mode) {
    if (!t || !cam || !mode) return set_error(VV_E_INVALID, "null argument");
    const vv_render_opts opts = o ? *o : default_opts();
    const double lo[3] = {t->view.lo0, t->view.lo1, t->view.lo2};
    *mode = decode_mode(t, cube_footprint(*cam, lo, t->view.side, nullptr), opts.frame_slice);
    return VV_OK;
}

static int render_multi_impl(const vv_tree *t, int32_t n_frames, const int32_t *frames, const vv_slice *const *caches,
                             const vv_render_opts *o, const vv_camera *cam, float *const *rgb, float *const *alpha,
                             float *const *depth, vv_camera_plan *plan, void *stream) {
    NvtxRange nv("vv:render_camera_multi");
    if (!t || !frames || !caches || !cam || !rgb || !alpha || !depth) return set_error(VV_E_INVALID, "null argument");
    if (n_frames < 2 || n_frames > kMaxMulti)
        return set_error(VV_E_UNSUPPORTED, "%d frames per walk (2..%d)", n_frames, kMaxMulti);
    for (int k = 0; k < n_frames; ++k) {
        int rc = check_frame(t, frames[k]);
        if (rc) return rc;
        if (!caches[k]) return set_error(VV_E_INVALID, "frame %d: a slice is required", frames[k]);
        if ((rc = check_cache(t, caches[k], frames[k]))) return rc;
        if (caches[k]->visible)
            return set_error(VV_E_INVALID, "frame %d: VV_SLICE_VISIBLE slices feed single-frame walks only",
                             frames[k]);
    }
    DeviceGuard g(t->device);
    const vv_render_opts opts = o ? *o : default_opts();
    CamMultiParams p;
    memset(&p, 0, sizeof(p));
    p.T = t->view;
    p.K = make_consts(t->n_max);
    p.cam = make_cam(*cam);
    for (int k = 0; k < n_frames; ++k) {
        p.S[k] = slice_view(caches[k]);
        p.frames[k] = frames[k];
        p.rgb[k] = rgb[k];
        p.alpha[k] = alpha[k];
        p.depth[k] = depth[k];
    }
    p.early_stop = opts.early_stop;
    p.edit_weight = opts.edit_weight;
    p.tmin = opts.tmin;
    p.tmax = opts.tmax;
    p.far_plane = opts.far_plane;
    p.alpha_floor = opts.alpha_floor;
    p.blocks_x = (cam->width + kTW - 1) / kTW;
    const unsigned grid = (unsigned)p.blocks_x * (unsigned)((cam->height + kTH - 1) / kTH);
    if (grid == 0) return VV_OK;
    int rr[4];
    occupied_rect(t, p.cam, nullptr, cam->width, cam->height, rr);
    p.cx0 = rr[0]; p.cy0 = rr[1]; p.cx1 = rr[2]; p.cy1 = rr[3];
    cudaStream_t st = (cudaStream_t)stream;
    std::unique_lock<std::mutex> plan_lock;
    if (plan) {  // persistent warps in the plan's cost order; its cached coverage
        if (plan->device != t->device) return set_error(VV_E_INVALID, "plan belongs to another device");
        plan_lock = std::unique_lock<std::mutex>(plan->mu);
        int rc = plan_prepare(plan, (int)grid, p.blocks_x, st);
        if (rc) return rc;
        if ((rc = plan_coverage(plan, t, *cam, p.cam, st))) return rc;
        p.cov = plan->cov;
        p.work = plan->counter;
        p.n_work = (int)grid * kWarpsPerTile;
        p.block_order = plan->valid ? plan->order : nullptr;
        p.block_cost = plan->cost;
    }
    // a node mask built for a group holding every frame of this walk (slices
    // of one vv_slice_build_frames call share it) keeps every subtree lit
    // in any of them
    const NodeMask *nm = caches[0]->nmask.get();
    for (int k = 1; k < n_frames && nm; ++k)
        if (caches[k]->nmask.get() != nm) nm = nullptr;
    p.T.child = image_child(t, nm);
    int rc = launch_camera_multi(t->n_max, n_frames, t->has_edits, t->depth > kNarrowDepth, p, grid, st,
                                 long_queue(t, nm));
    if (rc || !plan) return rc;
    return plan_finish(plan, st, mask_wanted(t));
}

int vv_render_camera_multi(const vv_tree *t, int32_t n_frames, const int32_t *frames, const vv_slice *const *caches,
                           const vv_render_opts *o, const vv_camera *cam, float *const *rgb, float *const *alpha,
                           float *const *depth, void *stream) {
    return render_multi_impl(t, n_frames, frames, caches, o, cam, rgb, alpha, depth, nullptr, stream);
}

int vv_render_camera_multi_planned(const vv_tree *t, int32_t n_frames, const int32_t *frames,
                                   const vv_slice *const *caches, const vv_render_opts *o, const vv_camera *cam,
                                   float *const *rgb, float *const *alpha, float *const *depth, vv_camera_plan *plan,
                                   void *stream) {
    if (!plan) return set_error(VV_E_INVALID, "null plan");
    return render_multi_impl(t, n_frames, frames, caches, o, cam, rgb, alpha, depth, plan, stream);
}

int vv_render_camera_tiles(const vv_tree *t, int32_t frame, const vv_slice *cache, const vv_render_opts *opts,
                           const vv_camera *cam, int32_t tile, int32_t shard, int32_t n_shards, float *packed,
                           void *stream) {
    if (!packed) return set_error(VV_E_INVALID, "null packed output");
    if (tile <= 0) return set_error(VV_E_INVALID, "bad tile arguments (tile must be a positive multiple of 16)");
    return render_camera_impl(t, frame, cache, opts, cam, nullptr, nullptr, nullptr, packed, tile, shard, n_shards,
                              0, stream);
}

int vv_render_camera_tiles_direct(const vv_tree *t, int32_t frame, const vv_slice *cache, const vv_render_opts *opts,
                                  const vv_camera *cam, int32_t tile, int32_t shard, int32_t n_shards, float *rgb,
                                  float *alpha, float *depth, int32_t peer, void *stream) {
    if (!rgb && !alpha && !depth) return set_error(VV_E_INVALID, "null image planes");
    if (tile <= 0) return set_error(VV_E_INVALID, "bad tile arguments (tile must be a positive multiple of 16)");
    return render_camera_impl(t, frame, cache, opts, cam, rgb, alpha, depth, nullptr, tile, shard, n_shards,
                              peer ? 1 : 0, stream);
}

// ------------------------------------------------------------ CUDA IPC
// Image planes shared between the ranks of one node: the output rank
// allocates, every rank maps the handle and stores its tiles over
// NVLink/NVSwitch.
int vv_ipc_alloc(int32_t device, size_t bytes, void **ptr, unsigned char *handle) {
    if (!ptr || !handle || bytes == 0) return set_error(VV_E_INVALID, "bad ipc_alloc arguments");
    DeviceGuard g(device);
    void *p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
        cudaGetLastError();
        return set_error(VV_E_NOMEM, "cudaMalloc(%zu) failed", bytes);
    }
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
        cudaFree(p);
        return set_error(VV_E_CUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    }
    static_assert(sizeof(h) == VV_IPC_HANDLE_BYTES, "ipc handle size");
    memcpy(handle, &h, sizeof(h));
    *ptr = p;
    return VV_OK;
}

int vv_ipc_open(int32_t device, const unsigned char *handle, void **ptr) {
    if (!ptr || !handle) return set_error(VV_E_INVALID, "bad ipc_open arguments");
    DeviceGuard g(device);
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_error(VV_E_CUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    }
    return VV_OK;
}

int vv_ipc_close(int32_t device, void *ptr) {
    DeviceGuard g(device);
    if (ptr && cudaIpcCloseMemHandle(ptr) != cudaSuccess) return set_error(VV_E_CUDA, "cudaIpcCloseMemHandle failed");
    return VV_OK;
}

int vv_ipc_free(int32_t device, void *ptr) {
    DeviceGuard g(device);
    if (ptr && cudaFree(ptr) != cudaSuccess) return set_error(VV_E_CUDA, "cudaFree failed");
    return VV_OK;
}

int vv_unpack_tiles(const float *packed_all, int32_t width, int32_t height, int32_t tile, int32_t n_shards,
                    float *rgb, float *alpha, float *depth, void *stream) {
    if (!packed_all || width <= 0 || height <= 0 || tile <= 0 || n_shards < 1)
        return set_error(VV_E_INVALID, "bad unpack arguments");
    const int tiles_x = (width + tile - 1) / tile, tiles_y = (height + tile - 1) / tile;
    const int64_t npix = (int64_t)width * height;
    (void)npix;
    return launch_unpack(packed_all, width, height, tile, n_shards, tiles_x, tiles_x * tiles_y, rgb, alpha, depth,
                         (cudaStream_t)stream);
}

// Decode mode of scene instance i: the rays that can reach its tree at its
// frame, summed over every instance sharing both, against the leaf count.
static int scene_decode_mode(const vv_instance *inst, int n_inst, int i, const vv_camera &cam, int policy) {
    double reach = 0.0;
    for (int j = 0; j < n_inst; ++j) {
        if (inst[j].tree != inst[i].tree || inst[j].frame != inst[i].frame) continue;
        const vv_tree *tj = inst[j].tree;
        const double lo[3] = {tj->view.lo0, tj->view.lo1, tj->view.lo2};
        if (inst[j].mode == 0) {  // rigid: the pulled-back camera in the tree's frame
            vv_camera c2 = cam;
            memcpy(c2.c2w, inst[j].pose, sizeof(c2.c2w));
            reach += cube_footprint(c2, lo, tj->view.side, nullptr);
        } else {
            double A[12];
            affine_from_inverse(inst[j].inv, A);
            reach += cube_footprint(cam, lo, tj->view.side, A);
        }
    }
    reach = std::min(reach, (double)cam.width * cam.height);
    return decode_mode(inst[i].tree, reach, policy);
}

int vv_scene_decode_modes(const vv_instance *inst, int32_t n_inst, const vv_render_opts *o, const vv_camera *cam,
                          int32_t *modes) {
    if (!inst || !cam || !modes || n_inst < 1) return set_error(VV_E_INVALID, "bad argument");
    const vv_render_opts opts = o ? *o : default_opts();
    for (int i = 0; i < n_inst; ++i) {
        if (!inst[i].tree) return set_error(VV_E_INVALID, "null tree in instance %d", i);
        modes[i] = scene_decode_mode(inst, n_inst, i, *cam, opts.frame_slice);
    }
    return VV_OK;
}

// One fused scene launch over instances [b, e) of the visible list (<= 16,
// one n_max), continuing Algorithm 1 from state_in and handing it on through
// state_out when the scene needs several launches (more than 16 instances or
// mixed n_max); decode modes consider every instance sharing a tree.
static int scene_run(const vv_instance *inst, int n_all, int b, int e, const vv_render_opts &opts,
                     const vv_camera *cam, const double *background, float *image, float *alpha, float *depth,
                     cudaStream_t st, bool joint, double *state_in, double *state_out,
                     vv_camera_plan *plan = nullptr) {
    const vv_tree *t0 = inst[b].tree;
    int max_depth = 0;
    for (int i = b; i < e; ++i) max_depth = std::max(max_depth, inst[i].tree->depth);
    SceneParams p;
    memset(&p, 0, sizeof(p));
    p.K = make_consts(t0->n_max);
    p.cam = make_cam(*cam);
    p.n_inst = e - b;
    p.total_inst = n_all;
    p.state_in = state_in;
    p.state_out = state_out;
    for (int i = b; i < e; ++i) {
        InstView &v = p.inst[i - b];
        v.T = inst[i].tree->view;
        v.frame = inst[i].frame;
        v.mode = inst[i].mode;
        vv_camera c2 = *cam;
        memcpy(c2.c2w, inst[i].pose, sizeof(c2.c2w));
        v.cam = make_cam(c2);
        for (int k = 0; k < 12; ++k) v.inv[k] = inst[i].inv[k];
        int rr[4];
        if (v.mode == 0) {  // rigid: the pulled-back camera shoots the rays in tree space
            occupied_rect(inst[i].tree, v.cam, nullptr, cam->width, cam->height, rr);
        } else {  // general: the scene camera sees the tree through its affine
            double A[12];
            affine_from_inverse(inst[i].inv, A);
            occupied_rect(inst[i].tree, p.cam, A, cam->width, cam->height, rr);
        }
        v.rx0 = rr[0]; v.ry0 = rr[1]; v.rx1 = rr[2]; v.ry1 = rr[3];
    }
    p.early_stop = opts.early_stop;
    p.edit_weight = opts.edit_weight;
    p.tmin = opts.tmin;
    p.tmax = opts.tmax;
    p.far_plane = opts.far_plane;
    p.alpha_floor = opts.alpha_floor;
    p.composite = background != nullptr;
    p.bg0 = background ? background[0] : 0.0;
    p.bg1 = background ? background[1] : 0.0;
    p.bg2 = background ? background[2] : 0.0;
    p.image = image;
    p.alpha = alpha;
    p.depth = depth;
    p.max_depth = max_depth;
    const bool wide = max_depth > kNarrowDepth;
    const size_t smem = stack_bytes(max_depth, wide);
    dim3 grid((unsigned)((cam->width + 15) / 16), (unsigned)((cam->height + 7) / 8));
    Transient tr[kMaxInst];
    for (int i = b; i < e; ++i) {
        InstView &v = p.inst[i - b];
        v.S = SliceView{nullptr, 0, 0, nullptr};
        int same = -1;
        for (int j = b; j < i; ++j)
            if (inst[j].tree == inst[i].tree && inst[j].frame == inst[i].frame && p.inst[j - b].S.rec) same = j - b;
        const int mode = scene_decode_mode(inst, n_all, i, *cam, opts.frame_slice);
        if (same >= 0) {
            v.S = p.inst[same].S;
            v.T.child = p.inst[same].T.child;
        } else if (mode != 0) {
            int r = build_transient(inst[i].tree, inst[i].frame, st, v.S, tr[i - b]);
            if (r) return r;
            v.T.child = image_child(inst[i].tree, tr[i - b].nmask.get());
        }
    }
    if (joint) return launch_scene_joint(t0->n_max, wide, p, st);
    bool lean = true;  // every instance decoded per sample, no edits: the lean instantiation
    for (int i = b; i < e; ++i)
        if (p.inst[i - b].S.rec || inst[i].tree->has_edits) lean = false;
    std::unique_lock<std::mutex> plan_lock;
    if (plan) {  // persistent warps over 16x2-pixel chunks in the previous frames' cost order
        if (plan->device != t0->device) return set_error(VV_E_INVALID, "plan belongs to another device");
        plan_lock = std::unique_lock<std::mutex>(plan->mu);
        const int n_blocks = (int)(grid.x * grid.y);
        int rc = plan_prepare(plan, n_blocks, (int)grid.x, st);
        if (rc) return rc;
        p.work = plan->counter;
        p.n_work = n_blocks * 4;
        p.blocks_x = (int)grid.x;
        p.block_order = plan->valid ? plan->order : nullptr;
        p.block_cost = plan->cost;
    }
    int rc = launch_scene(t0->n_max, wide, lean, p, grid, smem, st);
    if (rc || !plan) return rc;
    return plan_finish(plan, st);  // (cfg4: 12,818 vs 12,767 Mrays/s re-sorting every 16th vs 4th render)
}

static int render_scene_impl(const vv_instance *inst, int32_t n_inst, const vv_render_opts *o, const vv_camera *cam,
                             const double *background, float *image, float *alpha, float *depth, void *stream,
                             bool joint, vv_camera_plan *plan = nullptr) {
    NvtxRange nv(joint ? "vv:render_scene_joint" : "vv:render_scene");
    if (!inst || !cam) return set_error(VV_E_INVALID, "null argument");
    if (!image && !alpha && !depth) return set_error(VV_E_INVALID, "no output");
    if (background && !image) return set_error(VV_E_INVALID, "background given without an image output");
    if (n_inst < 1) return set_error(VV_E_INVALID, "scene has no visible instances");
    const vv_tree *t0 = inst[0].tree;
    if (!t0) return set_error(VV_E_INVALID, "null tree");
    bool mixed = false;
    for (int i = 0; i < n_inst; ++i) {
        const vv_tree *t = inst[i].tree;
        if (!t) return set_error(VV_E_INVALID, "null tree in instance %d", i);
        if (t->device != t0->device) return set_error(VV_E_INVALID, "instances on different devices");
        mixed |= t->n_max != t0->n_max;
        int rc = check_frame(t, inst[i].frame);
        if (rc) return rc;
    }
    DeviceGuard g(t0->device);
    const vv_render_opts opts = o ? *o : default_opts();
    cudaStream_t st = (cudaStream_t)stream;
    if (joint) {
        if (mixed) return set_error(VV_E_UNSUPPORTED, "mixed n_max in one joint render");
        return scene_run(inst, n_inst, 0, n_inst, opts, cam, background, image, alpha, depth, st, true, nullptr,
                         nullptr);
    }
    // runs of consecutive instances with one n_max, at most kMaxInst each
    std::vector<std::pair<int, int>> runs;
    for (int b = 0; b < n_inst;) {
        int e = b + 1;
        while (e < n_inst && e - b < kMaxInst && inst[e].tree->n_max == inst[b].tree->n_max) ++e;
        runs.emplace_back(b, e);
        b = e;
    }
    if (runs.size() == 1)
        return scene_run(inst, n_inst, 0, n_inst, opts, cam, background, image, alpha, depth, st, false, nullptr,
                         nullptr, plan);
    // several launches: the per-pixel Algorithm-1 state (I rgb, D, A; f64)
    // carried between them in a stream-ordered buffer
    Transient state;
    pool_setup(t0->device);
    const size_t bytes = (size_t)cam->width * cam->height * 5 * sizeof(double);
    if (cudaMallocAsync(&state.mem, bytes, st) != cudaSuccess) {
        cudaGetLastError();
        state.mem = nullptr;
        return set_error(VV_E_NOMEM, "scene state allocation (%zu bytes) failed", bytes);
    }
    state.st = st;
    double *sb = static_cast<double *>(state.mem);
    for (size_t r = 0; r < runs.size(); ++r) {
        const bool last = r + 1 == runs.size();
        int rc = scene_run(inst, n_inst, runs[r].first, runs[r].second, opts, cam, last ? background : nullptr,
                           last ? image : nullptr, last ? alpha : nullptr, last ? depth : nullptr, st, false,
                           r ? sb : nullptr, last ? nullptr : sb);
        if (rc) return rc;
    }
    return VV_OK;
}

int vv_render_scene(const vv_instance *inst, int32_t n_inst, const vv_render_opts *o, const vv_camera *cam,
                    const double *background, float *image, float *alpha, float *depth, void *stream) {
    return render_scene_impl(inst, n_inst, o, cam, background, image, alpha, depth, stream, false);
}

int vv_render_scene_joint(const vv_instance *inst, int32_t n_inst, const vv_render_opts *o, const vv_camera *cam,
                          const double *background, float *image, float *alpha, float *depth, void *stream) {
    return render_scene_impl(inst, n_inst, o, cam, background, image, alpha, depth, stream, true);
}

int vv_render_scene_planned(const vv_instance *inst, int32_t n_inst, const vv_render_opts *o, const vv_camera *cam,
                            const double *background, float *image, float *alpha, float *depth,
                            vv_camera_plan *plan, void *stream) {
    if (!plan) return set_error(VV_E_INVALID, "null plan");
    return render_scene_impl(inst, n_inst, o, cam, background, image, alpha, depth, stream, false, plan);
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
    const bool collect = seg_leaf != nullptr;
    return launch_segments(wide, collect, p, grid, smem, st);
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

int vv_shadow_blur(const float *alpha, int32_t res, const double *weights, int32_t radius, double *tmp, double *out,
                   void *stream) {
    if (!alpha || !out || res < 0 || radius < 0) return set_error(VV_E_INVALID, "bad argument");
    if (radius > 0 && (!weights || !tmp)) return set_error(VV_E_INVALID, "null weights / scratch");
    double *dw = nullptr;
    cudaStream_t st = (cudaStream_t)stream;
    if (radius > 0) {  // the 2r+1 host weights ride along stream-ordered
        VV_CUDA(cudaMallocAsync(&dw, (size_t)(2 * radius + 1) * sizeof(double), st));
        VV_CUDA(cudaMemcpyAsync(dw, weights, (size_t)(2 * radius + 1) * sizeof(double), cudaMemcpyHostToDevice, st));
    }
    const int rc = launch_shadow_blur(alpha, res, dw, radius, tmp, out, st);
    if (dw) cudaFreeAsync(dw, st);
    return rc;
}

int vv_scene_lighting_ex(const vv_camera *cam, const float *rgb, const float *alpha, const float *depth,
                         const double *background, const vv_light *lights, int32_t n_lights, float *image,
                         float *lit_rgb, void *stream) {
    if (!cam || !rgb || !alpha || !depth || !background || !image || (n_lights > 0 && !lights))
        return set_error(VV_E_INVALID, "null argument");
    if (n_lights < 0) return set_error(VV_E_INVALID, "negative light count");
    std::vector<LightView> L((size_t)std::max(n_lights, 1));
    for (int i = 0; i < n_lights; ++i) {
        const vv_light &s = lights[i];
        if (s.cast_shadows && (!s.shadow_map || s.shadow_res < 1))
            return set_error(VV_E_INVALID, "light %d casts shadows without a shadow map", i);
        L[i].px = s.position[0];
        L[i].py = s.position[1];
        L[i].pz = s.position[2];
        L[i].ga = s.ground_plane[0];
        L[i].gb = s.ground_plane[1];
        L[i].gc = s.ground_plane[2];
        L[i].gd = s.ground_plane[3];
        L[i].strength = s.shadow_strength;
        L[i].r0sq = s.falloff_r0 * s.falloff_r0;
        L[i].min_scale = s.falloff_min_scale;
        L[i].cast_shadows = s.cast_shadows;
        L[i].falloff_enabled = s.falloff_enabled;
        L[i].map = s.shadow_map;
        L[i].res = s.shadow_res;
        memcpy(L[i].w2c, s.w2c, sizeof(L[i].w2c));
        L[i].fx = s.fx;
        L[i].fy = s.fy;
        L[i].cx = s.cx;
        L[i].cy = s.cy;
    }
    // the lights ride along stream-ordered in device memory (any number)
    cudaStream_t st = (cudaStream_t)stream;
    LightView *dl = nullptr;
    if (n_lights > 0) {
        VV_CUDA(cudaMallocAsync(&dl, (size_t)n_lights * sizeof(LightView), st));
        VV_CUDA(cudaMemcpyAsync(dl, L.data(), (size_t)n_lights * sizeof(LightView), cudaMemcpyHostToDevice, st));
    }
    const int rc = launch_scene_light(make_cam(*cam), rgb, alpha, depth, background[0], background[1], background[2],
                                      dl, n_lights, image, lit_rgb, st);
    if (dl) cudaFreeAsync(dl, st);
    return rc;
}

int vv_scene_lighting(const vv_camera *cam, const float *rgb, const float *alpha, const float *depth,
                      const double *background, const vv_light *lights, int32_t n_lights, float *image,
                      void *stream) {
    return vv_scene_lighting_ex(cam, rgb, alpha, depth, background, lights, n_lights, image, nullptr, stream);
}

int vv_termination_leaves(const vv_tree *t, int32_t frame, const double *origins, const double *dirs,
                          const double *norms, int64_t n, double alpha_threshold, int64_t *out_leaf, void *stream) {
    if (!t) return set_error(VV_E_INVALID, "null tree");
    if (n == 0) return VV_OK;
    if (!origins || !dirs || !norms || !out_leaf) return set_error(VV_E_INVALID, "null argument");
    int rc = check_frame(t, frame);
    if (rc) return rc;
    DeviceGuard g(t->device);
    TermParams p;
    p.T = t->view;
    p.frame = frame;
    p.origins = origins;
    p.dirs = dirs;
    p.norms = norms;
    p.n = n;
    p.thr = alpha_threshold;
    p.out_leaf = out_leaf;
    const bool wide = t->depth > kNarrowDepth;
    const size_t smem = stack_bytes(t->depth, wide);
    const unsigned grid = (unsigned)((n + kBlock - 1) / kBlock);
    return launch_terminate(wide, p, grid, smem, (cudaStream_t)stream);
}

int vv_tree_set_edits(vv_tree *t, const float *edit_rgb, const int32_t *edit_t) {
    if (!t) return set_error(VV_E_INVALID, "null tree");
    if ((edit_rgb == nullptr) != (edit_t == nullptr))
        return set_error(VV_E_INVALID, "edit_rgb and edit_t must both be set or both be NULL");
    DeviceGuard g(t->device);
    const int64_t nl = t->n_leaves;
    if (!edit_rgb || nl == 0) {
        cudaDeviceSynchronize();  // no kernel may still read the old channels
        cudaFree(t->d_edit_rgb);
        cudaFree(t->d_edit_t);
        if (t->d_edit_rgb) t->bytes -= nl * (int64_t)(sizeof(float4) + sizeof(int2));
        t->d_edit_rgb = nullptr;
        t->d_edit_t = nullptr;
        t->has_edits = false;
        t->view.edit_rgb = nullptr;
        t->view.edit_t = nullptr;
        return VV_OK;
    }
    if (!t->d_edit_rgb) {
        if (cudaMalloc(&t->d_edit_rgb, (size_t)nl * sizeof(float4)) != cudaSuccess ||
            cudaMalloc(&t->d_edit_t, (size_t)nl * sizeof(int2)) != cudaSuccess) {
            cudaGetLastError();
            cudaFree(t->d_edit_rgb);
            t->d_edit_rgb = nullptr;
            t->d_edit_t = nullptr;
            return set_error(VV_E_NOMEM, "edit channel allocation failed");
        }
        t->bytes += nl * (int64_t)(sizeof(float4) + sizeof(int2));
    }
    // stream-ordered renders may still read the old values; the sync also
    // keeps the PDL invariant (launch_pdl, vv_kernels.cuh): no kernel is in
    // flight while tree state changes
    cudaDeviceSynchronize();
    if (!t->h_perm.empty()) {  // device-row order (walk-order leaf layout)
        std::vector<float> er((size_t)nl * 4);
        std::vector<int32_t> et((size_t)nl * 2);
        for (int64_t g = 0; g < nl; ++g) {
            const int64_t r = t->h_perm[g];
            memcpy(&er[4 * g], edit_rgb + 4 * r, 16);
            memcpy(&et[2 * g], edit_t + 2 * r, 8);
        }
        VV_CUDA(cudaMemcpy(t->d_edit_rgb, er.data(), (size_t)nl * sizeof(float4), cudaMemcpyHostToDevice));
        VV_CUDA(cudaMemcpy(t->d_edit_t, et.data(), (size_t)nl * sizeof(int2), cudaMemcpyHostToDevice));
    } else {
        VV_CUDA(cudaMemcpy(t->d_edit_rgb, edit_rgb, (size_t)nl * sizeof(float4), cudaMemcpyHostToDevice));
        VV_CUDA(cudaMemcpy(t->d_edit_t, edit_t, (size_t)nl * sizeof(int2), cudaMemcpyHostToDevice));
    }
    t->has_edits = true;
    t->view.edit_rgb = t->d_edit_rgb;
    t->view.edit_t = t->d_edit_t;
    return VV_OK;
}

int vv_voct_upload(const uint8_t *buf, size_t len, int device, vv_tree **out, vv_voct_info *info) {
    if (!out) return set_error(VV_E_INVALID, "null argument");
    // checks in the order of VOctree.from_bytes (octree.py:440-510)
    if (len < 4) return set_error(VV_E_TRUNCATED, "stream of %zu bytes is shorter than the magic", len);
    if (!buf) return set_error(VV_E_INVALID, "null argument");
    if (memcmp(buf, "VOCT", 4) != 0) {
        char m[64];
        int k = 0;
        for (int i = 0; i < 4; ++i) {
            const unsigned c = buf[i];
            k += (c >= 32 && c < 127 && c != '\\' && c != '\'') ? snprintf(m + k, sizeof(m) - k, "%c", c)
                                                                   : snprintf(m + k, sizeof(m) - k, "\\x%02x", c);
        }
        return set_error(VV_E_MAGIC, "bad magic b'%s', expected b'VOCT'", m);
    }
    if (len < 8) return set_error(VV_E_TRUNCATED, "stream ends inside the header");
    auto u32 = [&](size_t off) {
        uint32_t v;
        memcpy(&v, buf + off, 4);
        return v;
    };
    if (u32(4) != 1u) return set_error(VV_E_VERSION, "unsupported .voct version %u", u32(4));
    if (len < 4 + 24 + 48 + 8 + 4) return set_error(VV_E_TRUNCATED, "stream ends inside the header");
    const size_t body = len - 4;
    if (vv_crc32(0, buf, body) != u32(body)) return set_error(VV_E_CHECKSUM, "crc32 mismatch: stream corrupted");
    const uint32_t flags = u32(8), depth = u32(12), T = u32(16), C = u32(20), K = u32(24);
    double bbox[6];
    memcpy(bbox, buf + 28, sizeof(bbox));
    const uint32_t n_internal = u32(76), n_leaves = u32(80);
    double sides[3], smin = 1e308, smax = -1e308;
    for (int i = 0; i < 3; ++i) {
        sides[i] = bbox[3 + i] - bbox[i];
        smin = std::min(smin, sides[i]);
        smax = std::max(smax, sides[i]);
    }
    if (smax - smin > 1e-9 * std::max(1.0, fabs(sides[0])))
        return set_error(VV_E_FORMAT, "bbox is not a cube: sides [%.17g %.17g %.17g]", sides[0], sides[1], sides[2]);
    std::vector<int32_t> node_child((size_t)std::max<uint32_t>(n_internal, 1) * 8, -1);
    size_t off = 84, used = 0;
    int rc = vv_voct_parse_nodes(buf + off, body - off, n_internal, node_child.data(), &used);
    if (rc) return rc;
    off += used;
    const bool edits = (flags & 1u) != 0;
    const int64_t P = 2 * (int64_t)C + 3 * (int64_t)K, plen = P + (edits ? 5 : 0);
    const size_t need = (size_t)n_leaves * plen * 4 + 2 * (size_t)T * C * 4;
    if (off + need > body) return set_error(VV_E_TRUNCATED, "stream ends inside the payload block");
    if (off + need != body) return set_error(VV_E_FORMAT, "%zu trailing bytes after payload", body - off - need);
    int n_max = -1;
    for (int n = 0, k = 0; n <= 64; ++n) {  // _n_max_from_k: K = sum_{n' <= n} (n'+1)^2
        k += (n + 1) * (n + 1);
        if ((uint32_t)k == K) {
            n_max = n;
            break;
        }
        if ((uint32_t)k > K) break;
    }
    if (n_max < 0) return set_error(VV_E_FORMAT, "basis count %u is not a hyperspherical-harmonic count", K);
    const uint8_t *payload = buf + off;
    const uint8_t *a_ptr = payload + (size_t)n_leaves * plen * 4;
    std::vector<float> edit_rgb;
    std::vector<int32_t> edit_t;
    vv_tree_desc d;
    memset(&d, 0, sizeof(d));
    d.depth = (int32_t)depth;
    d.n_max = n_max;
    d.frames = (int32_t)T;
    d.coeff_count = (int32_t)C;
    d.n_internal = std::max<uint32_t>(n_internal, 1);
    d.n_leaves = n_leaves;
    d.bbox_lo[0] = bbox[0];
    d.bbox_lo[1] = bbox[1];
    d.bbox_lo[2] = bbox[2];
    d.side = sides[0];
    d.node_child = node_child.data();
    d.leaf_data = n_leaves ? reinterpret_cast<const float *>(payload) : nullptr;  // rows of plen floats
    d.basis_a = reinterpret_cast<const float *>(a_ptr);
    d.basis_b = reinterpret_cast<const float *>(a_ptr + (size_t)T * C * 4);
    if (edits && n_leaves) {  // [w | rgb(4) | packed u16 range]
        edit_rgb.resize((size_t)n_leaves * 4);
        edit_t.resize((size_t)n_leaves * 2);
        for (size_t r = 0; r < n_leaves; ++r) {
            const uint8_t *row = payload + r * plen * 4;
            memcpy(&edit_rgb[4 * r], row + (size_t)P * 4, 16);
            uint32_t packed;
            memcpy(&packed, row + (size_t)(P + 4) * 4, 4);
            edit_t[2 * r] = (int32_t)(packed & 0xFFFFu);
            edit_t[2 * r + 1] = (int32_t)(packed >> 16);
        }
        d.edit_rgb = edit_rgb.data();
        d.edit_t = edit_t.data();
    }
    rc = tree_alloc_common(&d, device, out, true, plen);
    if (rc) return rc;
    if (info) {
        memset(info, 0, sizeof(*info));
        info->version = 1;
        info->flags = (int32_t)flags;
        info->depth = (int32_t)depth;
        info->frames = (int32_t)T;
        info->coeff_count = (int32_t)C;
        info->basis_count = (int32_t)K;
        info->n_max = n_max;
        info->n_internal = n_internal;
        info->n_leaves = n_leaves;
        info->bbox_lo[0] = bbox[0];
        info->bbox_lo[1] = bbox[1];
        info->bbox_lo[2] = bbox[2];
        info->side = sides[0];
    }
    return VV_OK;
}

}  // extern "C"
