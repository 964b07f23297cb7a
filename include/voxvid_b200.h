/*
 * voxvid_b200.h -- C ABI of the B200-native VOctree renderer.
 *
 * This is the drop-in boundary for the reference package `voxvid`'s render
 * path.  The reference has no plugin registry: its boundary is the numba
 * kernel call inside render.render_rays (pkg/src/voxvid/render.py:204-214)
 * and its companion kernels.  Each entry point below names the reference
 * interface it replaces.  All compute entry points run hand-written sm_100a
 * CUDA kernels; there is no CPU fallback.  Every function returns 0 on
 * success or a negative VV_E* code; vv_last_error() returns the message of
 * the last failure on the calling thread.
 *
 * Pointers marked "device" are CUDA device pointers on the tree's device.
 * `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 * asynchronous with respect to the host unless stated otherwise.
 */
#ifndef VOXVID_B200_H
#define VOXVID_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VV_ABI_VERSION 1

enum {
    VV_OK = 0,
    VV_E_INVALID = -1,  /* bad argument (the reference raises ValueError) */
    VV_E_CUDA = -2,     /* CUDA runtime failure */
    VV_E_NOMEM = -3,    /* device allocation failed */
    VV_E_UNSUPPORTED = -4,
    VV_E_FORMAT = -5,   /* .voct parse errors, see vv_voct_* */
    VV_E_MAGIC = -6,
    VV_E_VERSION = -7,
    VV_E_TRUNCATED = -8,
    VV_E_CHECKSUM = -9
};

typedef struct vv_tree vv_tree;    /* device replica of one VOctree */
typedef struct vv_slice vv_slice;  /* per-frame slice cache (FrameSlice) */
typedef struct vv_camera_plan vv_camera_plan;  /* launch plan of one camera stream */

/* Host description of a VOctree: the arrays of voxvid.octree.VOctree
 * (octree.py:84-108).  Pointers are HOST pointers for vv_tree_upload. */
typedef struct {
    int32_t depth;            /* leaf depth d >= 1 */
    int32_t n_max;            /* HH truncation; K = sum_{n<=n_max} (n+1)^2 */
    int32_t frames;           /* T */
    int32_t coeff_count;      /* C */
    int64_t n_internal;       /* rows of node_child */
    int64_t n_leaves;         /* rows of leaf_data */
    double bbox_lo[3];
    double side;
    const int32_t *node_child;  /* (n_internal, 8), BFS order, -1 = empty */
    const float *leaf_data;     /* (n_leaves, 2C+3K) [w_sigma | w_gamma | w_hh] */
    const float *basis_a;       /* (T, C) */
    const float *basis_b;       /* (T, C) */
    const float *edit_rgb;      /* (n_leaves, 4) or NULL (no edits) */
    const int32_t *edit_t;      /* (n_leaves, 2) or NULL */
} vv_tree_desc;

/* RenderOptions (render.py:148-153) plus the ray-parameter clip that
 * render_rays passes to render_kernel (tmin = 0, tmax = 1e30, render.py:212). */
typedef struct {
    double early_stop;   /* terminate once transmittance < early_stop */
    double far_plane;    /* depth where alpha < alpha_floor */
    double alpha_floor;
    double edit_weight;
    double tmin;
    double tmax;
    /* Leaf decode strategy when no cache is passed (results are bitwise
     * identical either way, as for the reference's FrameSlice):
     * VV_SLICE_AUTO picks per call, VV_SLICE_PER_SAMPLE decodes each visited
     * leaf inside the render kernel (render_kernel's uncached branch),
     * VV_SLICE_PER_FRAME first decodes every leaf once into a transient
     * stream-ordered slice, then renders from it. */
    int32_t frame_slice;
    int32_t reserved;
} vv_render_opts;

enum { VV_SLICE_AUTO = 0, VV_SLICE_PER_SAMPLE = 1, VV_SLICE_PER_FRAME = 2 };

/* Pinhole camera (render.py:42-125): intrinsics in pixels, row-major c2w. */
typedef struct {
    int32_t width;
    int32_t height;
    double fx, fy, cx, cy;
    double c2w[16];
} vv_camera;

/* One placed instance for vv_render_scene (compose.py:160-199, 418-440).
 * mode 0 (rigid): rays are generated from the pulled-back camera pose
 *   `pose` = inv(affine) @ c2w (compose.py:427-431).
 * mode 1 (general affine): rays are generated from the scene camera and
 *   pulled back per ray through `inv` = inv(affine) (compose.py:432-440). */
typedef struct {
    const vv_tree *tree;
    int32_t frame;   /* local frame = timemap(global frame), host-resolved */
    int32_t mode;
    double pose[16]; /* mode 0 */
    double inv[16];  /* mode 1 */
} vv_instance;

int vv_abi_version(void);
const char *vv_last_error(void);
int vv_device_count(int *count);
/* Device-side bounds checks (the bounds-checked build, `make debug` ->
 * _lib/debug/libvoxvid_b200.so, -DVV_DEBUG_CHECKS): node rows, stack slots,
 * segment-queue fill, leaf rows and slice chunks are checked in the render
 * kernels; a failed check is counted (no trap).  enabled = 1 in that build;
 * violations / first_code (VV_DBG_* codes in vv_device.cuh) and the deepest
 * traversal stack (slots in use) since the last reset.  Synchronizes the
 * device. */
int vv_debug_checks(int32_t device, int32_t *enabled, uint32_t *violations, uint32_t *first_code,
                    uint32_t *stack_high_water, int32_t reset);

/* Basis tables of kernels.basis_tables (kernels.py:56-76); host only, for
 * parity checks of the constants.  sizes = {K, S, n_pairs}. */
int vv_basis_tables(int n_max, int64_t *pair_n, int64_t *pair_l, double *pair_norm,
                    int64_t *k2pair, int64_t *k2sh, double *sh_pref, int32_t *sizes);

/* ---- tree replica --------------------------------------------------------
 * Replaces: the implicit host arrays handed to render_kernel by
 * render.render_rays (render.py:204-214) -- uploaded once per device.
 * vv_tree_upload copies host arrays; vv_tree_bind takes a desc whose array
 * pointers are DEVICE pointers (e.g. torch tensors) and copies on device.
 * The replica owns its device memory either way.  Synchronous. */
int vv_tree_upload(const vv_tree_desc *host, int device, vv_tree **out);
int vv_tree_bind(const vv_tree_desc *dev, int device, vv_tree **out);
int vv_tree_free(vv_tree *tree);
int vv_tree_info(const vv_tree *tree, int64_t *n_leaves, int64_t *n_internal, int32_t *depth,
                 int32_t *frames, int64_t *device_bytes);
/* Share of leaves with sigma 0, measured at upload over frames 0, T/2 and
 * T-1.  Above 0.5 the sliced camera and playback kernels walk with the long
 * segment queue (a kernel choice only: images are bitwise the same). */
int vv_tree_dark_fraction(const vv_tree *tree, float *dark_frac);
/* (No reference counterpart: instrumentation.)  Benchmarking: the calling
 * thread's next camera render records `event`
 * (a cudaEvent_t) on its stream between its slice pass and its camera
 * kernel, so the two can be timed apart on the render()/render_into path. */
int vv_profile_split_event(void *event);
/* (No reference counterpart: the visible set is this renderer's.)  Size of
 * the tree's visible set (VV_SLICE_VISIBLE): leaves in it and
 * 64-leaf slice chunks holding one (synchronises `stream`). */
int vv_tree_visible_count(const vv_tree *tree, int64_t *n_visible, int64_t *n_chunks, void *stream);
/* The visible set itself: bit L of out (n_words >= 2 per 64 leaves) set
 * iff device leaf row L is in it (synchronises `stream`). */
int vv_tree_visible_bits(const vv_tree *tree, uint32_t *out, int64_t n_words, void *stream);
/* The device's leaf layout: ref_rows[g] = reference row id of device row g
 * (n_leaves int32, host).  Leaves are stored in walk (BFS = Morton) order
 * when the node table is a tree, else in reference order. */
int vv_tree_leaf_order(const vv_tree *tree, int32_t *ref_rows);

/* ---- per-frame slice cache -----------------------------------------------
 * Replaces build_frame_cache (render.py:170-179) -> build_slice_kernel
 * (kernels.py:397-407).  sigma is float64 per leaf (bit-exact with the
 * uncached path); the sliced SH coefficients are stored as fp32.
 * Error: frame outside [0, T) -> VV_E_INVALID ("frame F out of range"). */
int vv_slice_build(const vv_tree *tree, int32_t frame, void *stream, vv_slice **out);
/* The slice is allocated stream-ordered on `stream` (the device's default
 * memory pool) and released stream-ordered on the same stream: work already
 * queued on that stream may still read it. */
/* Slices of n_frames (1..4) frames from ONE pass over the payload (each
 * leaf row is read once and sliced per frame): out[k] is frames[k]'s slice,
 * equal to vv_slice_build(frames[k]).  Playback groups use it. */
int vv_slice_build_multi(const vv_tree *tree, int32_t n_frames, const int32_t *frames, void *stream,
                         vv_slice **out);
/* vv_slice_build_multi with flags.  VV_SLICE_RENDER_ONLY: slices only for
 * rendering -- where a chunk of 64 consecutive leaves has sigma 0 in every
 * frame, only sigma is written, and while chunks stay dark their w_gamma /
 * w_hh rows are not read.  The renderers never read the colour of a leaf
 * with sigma 0 (kernels.py:556-559), so images are bitwise the same; q of
 * such a slice cannot be exported.  Ignored for trees with edits (an edit
 * can give a dark leaf density).  render()'s transient slices and the
 * playback groups are built this way. */
#define VV_SLICE_RENDER_ONLY 1
/* VV_SLICE_VISIBLE (with VV_SLICE_RENDER_ONLY, one frame): records only for
 * the leaves in the tree's visible set (the leaves its camera walks have
 * visited lately) and a walk table in which every other leaf points at a
 * stand-in row; a camera walk that meets one re-walks that pixel per sample
 * (bitwise the same) and adds what it visits to the set.  Images are
 * bitwise unchanged.  Not exportable; camera renders only (VV_E_INVALID
 * from vv_render_rays and vv_render_camera_multi). */
#define VV_SLICE_VISIBLE 2
int vv_slice_build_frames(const vv_tree *tree, int32_t n_frames, const int32_t *frames, int32_t flags,
                          void *stream, vv_slice **out);
/* build_frame_cache (render.py:170-179) for camera renders only: a
 * VV_SLICE_VISIBLE slice of one frame whose walk table lives in `plan`
 * (kept across frames, rebuilt only when the set changes; the slice must
 * be used before the plan builds its next one).  Several cameras of one
 * frame (stereo) may share it. */
int vv_slice_build_visible(const vv_tree *tree, int32_t frame, vv_camera_plan *plan, void *stream, vv_slice **out);
int vv_slice_free(vv_slice *slice);
/* Copies the cache to caller device buffers: sigma (n_leaves) f64,
 * q (n_leaves, 3S) f32 (q: VV_E_INVALID for a VV_SLICE_RENDER_ONLY slice). */
int vv_slice_export(const vv_slice *slice, double *sigma, float *q, void *stream);
int vv_slice_frame(const vv_slice *slice, int32_t *frame);

/* ---- ray rendering -------------------------------------------------------
 * Replaces render_rays (render.py:182-215) -> render_kernel
 * (kernels.py:410-652).  origins/dirs: device (n, 3) f64, dirs unit length.
 * Outputs (device): premult (n, 3) f64, alpha (n) f64, tbar (n) f64.
 * Optional (NULL to skip): sample_count (n) i32 = leaf segments consumed
 * up to and including the early-stop one (shade_forward's `used`,
 * kernels.py:700-738); node_pops (n) i32 = internal-node pops; shaded (n)
 * i32 = leaves with sigma > 0.  cache may be NULL (uncached).
 * Errors: frame out of range; cache built for another frame. */
int vv_render_rays(const vv_tree *tree, int32_t frame, const vv_slice *cache,
                   const vv_render_opts *opts, const double *origins, const double *dirs,
                   int64_t n, double *premult, double *alpha, double *tbar,
                   int32_t *sample_count, int32_t *node_pops, int32_t *shaded, void *stream);

/* Visited-leaf CSR for the same rays: visit_start (n+1) i64 device prefix
 * sum of sample_count; writes visit_leaf[visit_start[r] + i] = leaf row of
 * the i-th consumed segment of ray r (reference row ids). */
int vv_render_rays_visits(const vv_tree *tree, int32_t frame, const vv_slice *cache,
                          const vv_render_opts *opts, const double *origins,
                          const double *dirs, int64_t n, const int64_t *visit_start,
                          int64_t *visit_leaf, void *stream);

/* ---- camera rendering ----------------------------------------------------
 * Replaces render (render.py:236-240) = Camera.rays + render_rays +
 * finalize_layer (render.py:218-233), fused into one kernel.  Outputs
 * (device, fp32, row-major pixels): rgb (H, W, 3) unpremultiplied, alpha
 * (H, W), depth (H, W) (far_plane where alpha < alpha_floor).  Any output
 * may be NULL. */
int vv_render_camera(const vv_tree *tree, int32_t frame, const vv_slice *cache,
                     const vv_render_opts *opts, const vv_camera *cam, float *rgb,
                     float *alpha, float *depth, void *stream);
/* vv_render_camera for the pixel rectangle region = {x0, y0, x1, y1}
 * ([x0, x1) x [y0, y1)) of full-size planes, which may be a peer GPU's
 * memory mapped with vv_ipc_open (peer != 0: a system-scope fence at kernel
 * exit).  Pixels outside the rectangle are not touched.  Without a cache,
 * only the leaf chunks whose cells can project into the rectangle are
 * decoded: one rank's share of a frame split into regions across GPUs
 * costs its share of the decode as well as of the walk.
 * block_order (optional, device int32): the launch order of the region's
 * camera blocks -- a permutation of 0 .. nbx*nby-1 (block b covers pixels
 * x0 + (b % nbx) * bw, y0 + (b / nbx) * bh, bw x bh from
 * vv_camera_block_shape) -- costliest first, so that the expensive blocks
 * do not form the tail of a short kernel.  Not validated: anything but a
 * permutation renders some pixels twice and others not at all. */
int vv_render_camera_region(const vv_tree *tree, int32_t frame, const vv_slice *cache,
                            const vv_render_opts *opts, const vv_camera *cam, const int32_t *region,
                            const int32_t *block_order, float *rgb, float *alpha, float *depth,
                            int32_t peer, void *stream);
/* render() to the host: vv_render_camera into device_planes (5 H W floats:
 * rgb | alpha | depth, as LayerImages' planes), each 64-row band of the
 * frame copied into host_planes (pinned, same layout) as soon as the
 * kernel has stored it -- the device->host copy overlaps the render (a copy
 * stream waits on per-band counters with cuStreamWaitValue32).  All work
 * is ordered on `stream`: the frame is on the host once it has reached the
 * end of it.  plan (optional, vv_camera_plan_create): its chunk counters
 * and cached coverage; the blocks run in row-major order regardless. */
int vv_render_camera_to_host(const vv_tree *tree, int32_t frame, const vv_slice *cache,
                             const vv_render_opts *opts, const vv_camera *cam, float *device_planes,
                             float *host_planes, vv_camera_plan *plan, void *stream);

/* Camera plans: renders of a camera stream (playback, a fixed view, one
 * rank's region) through a plan run the camera kernel as persistent warps
 * that take the frame's warp chunks from a counter in the previous render's
 * measured cost order (costliest blocks first) and record this render's
 * costs for the next one.  Scheduling only: any plan renders bitwise the
 * same pixels as vv_render_camera.  A plan is used from one stream at a
 * time; it resizes itself when the image or region size changes.
 * region: {x0, y0, x1, y1} as vv_render_camera_region, or NULL (whole
 * image). */
int vv_camera_plan_create(int32_t device, vv_camera_plan **plan);
int vv_camera_plan_free(vv_camera_plan *plan);
int vv_render_camera_planned(const vv_tree *tree, int32_t frame, const vv_slice *cache,
                             const vv_render_opts *opts, const vv_camera *cam, const int32_t *region,
                             vv_camera_plan *plan, float *rgb, float *alpha, float *depth, int32_t peer,
                             void *stream);
/* Pixel footprint of one camera-kernel block (block_order units). */
int vv_camera_block_shape(int32_t *width, int32_t *height);
/* vv_render_camera plus, per pixel, the leaf samples the ray consumed
 * (int32, device, (H, W)): the reference's per-ray `used` count
 * (shade_forward_kernel, kernels.py:700-738; Trainer._forward, train.py:
 * 269-296), written by the same kernel instantiation vv_render_camera runs. */
int vv_render_camera_counts(const vv_tree *tree, int32_t frame, const vv_slice *cache,
                            const vv_render_opts *opts, const vv_camera *cam, float *rgb,
                            float *alpha, float *depth, int32_t *sample_count, void *stream);

/* Tile-sharded variant for multi-GPU: renders only the square tiles of
 * size `tile` whose linear index i (row-major over the tile grid) has
 * i % n_shards == shard, writing them packed in tile order into `packed`
 * as (n_my_tiles, tile*tile, 5) fp32 [r, g, b, alpha, depth]. */
int vv_render_camera_tiles(const vv_tree *tree, int32_t frame, const vv_slice *cache,
                           const vv_render_opts *opts, const vv_camera *cam, int32_t tile,
                           int32_t shard, int32_t n_shards, float *packed, void *stream);
/* Scatter packed tiles of every shard (shard-major, as all-gathered) into
 * full images rgb (H, W, 3), alpha (H, W), depth (H, W). */
int vv_unpack_tiles(const float *packed_all, int32_t width, int32_t height, int32_t tile,
                    int32_t n_shards, float *rgb, float *alpha, float *depth, void *stream);

/* Fused tile render + gather (no all-gather, no unpack): renders this
 * shard's tiles (same assignment as vv_render_camera_tiles) straight into
 * the FULL-image planes rgb (H, W, 3), alpha (H, W), depth (H, W); pixels
 * of other shards' tiles are not touched.  The planes may be another GPU's
 * memory mapped with vv_ipc_open (the output rank's frame, written over
 * NVLink/NVSwitch as the tiles finish); `peer` != 0 then makes the kernel
 * fence its stores system-wide before it retires, so one stream-ordered
 * barrier after the launch publishes the frame.  Replaces the per-frame
 * gather of SURVEY.md section 8(e) (the reference has no multi-device
 * path: it renders frames sequentially, cli.py:189-200). */
int vv_render_camera_tiles_direct(const vv_tree *tree, int32_t frame, const vv_slice *cache,
                                  const vv_render_opts *opts, const vv_camera *cam, int32_t tile,
                                  int32_t shard, int32_t n_shards, float *rgb, float *alpha,
                                  float *depth, int32_t peer, void *stream);

/* CUDA IPC for the planes above: vv_ipc_alloc (output rank) allocates
 * `bytes` on `device` and returns its VV_IPC_HANDLE_BYTES-byte handle;
 * the other ranks of the node map it with vv_ipc_open (a different
 * process; peer access is enabled lazily), unmap with vv_ipc_close; the
 * owner releases it with vv_ipc_free. */
#define VV_IPC_HANDLE_BYTES 64
int vv_ipc_alloc(int32_t device, size_t bytes, void **ptr, unsigned char *handle);
int vv_ipc_open(int32_t device, const unsigned char *handle, void **ptr);
int vv_ipc_close(int32_t device, void *ptr);
int vv_ipc_free(int32_t device, void *ptr);

/* The leaf-decode mode VV_SLICE_AUTO picks for a camera render of this tree
 * (1 = per-frame slice pass, 0 = decode per sample): slice when the leaves
 * number <= 4 x the rays that can reach the tree (its projected footprint). */
int vv_camera_decode_mode(const vv_tree *tree, const vv_camera *cam, const vv_render_opts *opts, int32_t *mode);
/* Playback: n_frames (2..4) frames of ONE camera in one walk -- the rays and
 * therefore the traversal are frame-independent, so one walk serves every
 * frame; each frame keeps its own slice (caches[k], required, built for
 * frames[k]), accumulators and early termination.  Per-frame outputs are
 * bitwise identical to vv_render_camera(frames[k]).  rgb/alpha/depth:
 * arrays of n_frames device pointers (entries may be NULL). */
int vv_render_camera_multi(const vv_tree *tree, int32_t n_frames, const int32_t *frames,
                           const vv_slice *const *caches, const vv_render_opts *opts, const vv_camera *cam,
                           float *const *rgb, float *const *alpha, float *const *depth, void *stream);
/* vv_render_camera_multi scheduled by a plan (vv_camera_plan_create):
 * persistent warps in the previous walks' cost order, the plan's cached
 * coverage; bitwise vv_render_camera_multi.  Use a plan of its own. */
int vv_render_camera_multi_planned(const vv_tree *tree, int32_t n_frames, const int32_t *frames,
                                   const vv_slice *const *caches, const vv_render_opts *opts, const vv_camera *cam,
                                   float *const *rgb, float *const *alpha, float *const *depth,
                                   vv_camera_plan *plan, void *stream);

/* ---- multi-instance scene -------------------------------------------------
 * Replaces render_scene (compose.py:443-475) without lights: per pixel,
 * every instance is rendered through its pulled-back ray (render_instance,
 * compose.py:418-440), finalized, blended by Algorithm 1 in instance order
 * (blend_layers, compose.py:373-406), unpremultiplied (compose.py:457-460)
 * and composited over `background` (composite_background,
 * render.py:243-251).  Outputs (device fp32): image (H, W, 3); optional
 * blended alpha (H, W) and depth (H, W).  background = NULL: image gets the
 * blended, unpremultiplied layer rgb instead (input of the lighting passes,
 * vv_scene_lighting); image may then be NULL too (alpha/depth only). */
int vv_render_scene(const vv_instance *instances, int32_t n_instances,
                    const vv_render_opts *opts, const vv_camera *cam, const double *background,
                    float *image, float *alpha, float *depth, void *stream);
/* Per-sample depth-ordered joint composition (north-star kernel 4; an
 * extension: the reference composes by Algorithm 1 and checks it against
 * this joint rendering in its tests, pkg/tests/util.py:205-245).  Same
 * arguments as vv_render_scene (<= 8 instances): every instance walks its
 * tree along its pulled-back ray, the leaf segments of all walks are merged
 * by world depth (ties to the earlier instance) and composited once,
 * tau = sigma (t1 - t0) in tree units, front to back, early termination at
 * opts->early_stop (0: none).  image = C + (1 - A) background (premultiplied
 * joint colour C), or C / A without a background; alpha A; depth = expected
 * world t (far_plane below alpha_floor).  Equal to vv_render_scene where the
 * instances do not interleave along any ray. */
int vv_render_scene_joint(const vv_instance *inst, int32_t n_inst, const vv_render_opts *opts,
                          const vv_camera *cam, const double *background, float *image, float *alpha,
                          float *depth, void *stream);
/* vv_render_scene scheduled by a plan (vv_camera_plan_create): persistent
 * warps over the frame's 16x2-pixel chunks in the previous frames' cost
 * order (a scene of <= 16 instances of one n_max; larger scenes chain
 * launches without one).  Bitwise vv_render_scene.  Use a plan of its own
 * (not one shared with camera renders). */
int vv_render_scene_planned(const vv_instance *inst, int32_t n_inst, const vv_render_opts *opts,
                            const vv_camera *cam, const double *background, float *image, float *alpha,
                            float *depth, vv_camera_plan *plan, void *stream);
/* Leaf-decode mode vv_render_scene picks for each instance (0: per sample
 * inside the scene kernel -- every instance 0 and no edits runs the lean
 * instantiation --, 1: a per-frame slice pass first). */
int vv_scene_decode_modes(const vv_instance *inst, int32_t n_inst, const vv_render_opts *opts,
                          const vv_camera *cam, int32_t *modes);

/* ---- traversal only --------------------------------------------------------
 * Replace count_segments_kernel / collect_segments_kernel
 * (kernels.py:313-367) and VOctree.ray_segments (octree.py:296-326).
 * Rays in world space (dirs need not be unit; t stays the world parameter). */
int vv_count_segments(const vv_tree *tree, const double *origins, const double *dirs,
                      int64_t n, double tmin, double tmax, int64_t *count, void *stream);
int vv_collect_segments(const vv_tree *tree, const double *origins, const double *dirs,
                        int64_t n, double tmin, double tmax, const int64_t *ray_start,
                        int64_t *seg_leaf, double *seg_t0, double *seg_t1, void *stream);

/* ---- lighting passes (compose.py:539-619) ---------------------------------
 * One point light: falloff scale clamp(r0^2 / (r0^2 + d^2), min, 1) on the
 * blended colour where alpha > 0 (falloff_pass, compose.py:606-619), and a
 * ground-plane shadow factor 1 - strength * occ on the background, occ
 * sampled bilinearly (map_coordinates order 1, mode "constant") from the
 * light's blurred alpha map through its camera (ShadowMap.background_factor
 * / factor_at_points, compose.py:547-582).  w2c: row-major 3x4 of
 * inv(light_cam.c2w) as the host computed it. */
typedef struct {
    double position[3];
    double ground_plane[4];
    double shadow_strength, falloff_r0, falloff_min_scale;
    int32_t cast_shadows, falloff_enabled;
    const double *shadow_map; /* (res, res) device f64, row = y */
    int32_t shadow_res, reserved;
    double w2c[12];
    double fx, fy, cx, cy;    /* light camera intrinsics */
} vv_light;
/* shadow_pass's blur (compose.py:590-602): scipy gaussian_filter, mode
 * "constant", truncate 4 -- weights (2 radius + 1, host, normalised as
 * scipy's _gaussian_kernel1d) correlated along rows then columns in
 * scipy's symmetric summation order, f64.  alpha: (res, res) device fp32
 * joint alpha; tmp, out: (res, res) device f64.  radius 0: plain copy. */
int vv_shadow_blur(const float *alpha, int32_t res, const double *weights, int32_t radius, double *tmp,
                   double *out, void *stream);
/* Lights applied in order to the blended layer (vv_render_scene with
 * background NULL), then composite_background over `background`
 * (render_scene, compose.py:462-471).  Device fp32 images; any number of
 * lights (0: the plain background composite). */
int vv_scene_lighting(const vv_camera *cam, const float *rgb, const float *alpha, const float *depth,
                      const double *background, const vv_light *lights, int32_t n_lights, float *image,
                      void *stream);
/* vv_scene_lighting that also writes lit_rgb (H, W, 3): the blended rgb
 * after every light's falloff -- the `blended` layer render_scene returns
 * with want_layers (compose.py:462-466). */
int vv_scene_lighting_ex(const vv_camera *cam, const float *rgb, const float *alpha, const float *depth,
                         const double *background, const vv_light *lights, int32_t n_lights, float *image,
                         float *lit_rgb, void *stream);

/* ---- paint / termination voxel ---------------------------------------------
 * Replaces the per-pixel loop of compose.paint (compose.py:482-532): for
 * each ray, walk every leaf segment (ray_segments, octree.py:296-326, no
 * early stop), accumulate alpha with sigma = max(0, w_sigma . A[frame]) and
 * delta = (t1 - t0) * norms[r], and write the first leaf row where the
 * accumulated alpha reaches alpha_threshold, or -1.  Device pointers;
 * norms[r] = |dirs[r]| as the caller computed it (np.linalg.norm). */
int vv_termination_leaves(const vv_tree *tree, int32_t frame, const double *origins,
                          const double *dirs, const double *norms, int64_t n,
                          double alpha_threshold, int64_t *out_leaf, void *stream);
/* Replace a replica's edit channels (VOctree.edit_rgb / edit_t, octree.py:
 * 84-108, written by paint) from HOST arrays of n_leaves rows, without
 * re-uploading the payload; both NULL removes them.  Synchronous. */
int vv_tree_set_edits(vv_tree *tree, const float *edit_rgb, const int32_t *edit_t);

/* ---- .voct codec (host) ----------------------------------------------------
 * Replaces the node-table loops of VOctree.to_bytes / from_bytes
 * (octree.py:383-394, 440-455).  parse: reads n_internal BFS records
 * (u8 mask + one u32 per set bit) starting at buf, writes node_child
 * (n_internal, 8) and the byte length consumed; VV_E_TRUNCATED if the
 * records run past len.  encode: writes into buf (capacity cap) and returns
 * the bytes written in *used (pass buf = NULL to size). */
int vv_voct_parse_nodes(const uint8_t *buf, size_t len, int64_t n_internal,
                        int32_t *node_child, size_t *consumed);
int vv_voct_encode_nodes(const int32_t *node_child, int64_t n_internal, uint8_t *buf,
                         size_t cap, size_t *used);
/* Whole .voct stream -> device replica, no host arrays (octree.py:371-510,
 * VOctree.from_bytes + upload): validates in the reference's order with its
 * error classes (VV_E_TRUNCATED / VV_E_MAGIC / VV_E_VERSION / VV_E_CHECKSUM /
 * VV_E_FORMAT for a non-cube bbox, trailing bytes or a K that is no HH
 * count), checks the CRC (host threads), parses the node table and streams
 * the payload block from buf through the device repack; edit channels are
 * unpacked from the 5 extra columns.  info (optional) receives the header. */
typedef struct {
    int32_t version, flags, depth, frames, coeff_count, basis_count, n_max;
    int32_t reserved;
    int64_t n_internal, n_leaves;
    double bbox_lo[3];
    double side;
} vv_voct_info;
int vv_voct_upload(const uint8_t *buf, size_t len, int device, vv_tree **out, vv_voct_info *info);
/* CRC-32 (zlib polynomial) of buf, continuing from crc. */
uint32_t vv_crc32(uint32_t crc, const uint8_t *buf, size_t len);

#ifdef __cplusplus
}
#endif
#endif /* VOXVID_B200_H */
