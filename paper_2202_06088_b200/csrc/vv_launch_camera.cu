// vv_launch_camera.cu -- instantiations of k_render_camera (render / tiles path).
#include "vv_kernels.cuh"
#include <type_traits>

namespace vvk {

// queue threshold for trees whose frames are mostly dark (long walks, few
// shaded leaves: the cfg3 motion tree renders 6% faster with 8 than with 6)
#ifndef VV_SEG_LONG
#define VV_SEG_LONG 8
#endif
constexpr int kSegLong = VV_SEG_LONG;

template <int NM, int CACHED, bool EDITS, class Entry, int SEG = VV_SEG_MIN, int VIS = 0>
static int go(const CamParams &p, unsigned max_blocks, size_t smem, cudaStream_t st) {
    auto kern = k_render_camera<NM, CACHED, EDITS, Entry, SEG, VIS>;
    int r = prep_smem(kern, smem);
    if (r) return r;
    // persistent warps: one resident grid pulls the warp chunks
    const unsigned grid = p.work ? persistent_grid(kern, kTileRays, smem, max_blocks) : max_blocks;
    launch_pdl(kern, dim3(grid), dim3(kTileRays), smem, st, p);
    return check_launch("render_camera");
}

template <int NM, int MODE, class Entry>
static int pick_e(bool edits, const CamParams &p, unsigned grid, size_t smem, cudaStream_t st) {
    return edits ? go<NM, MODE, true, Entry>(p, grid, smem, st) : go<NM, MODE, false, Entry>(p, grid, smem, st);
}

template <int NM, class Entry>
static int pick(int mode, bool edits, const CamParams &p, unsigned grid, size_t smem, cudaStream_t st) {
    if (mode == 1) return pick_e<NM, 1, Entry>(edits, p, grid, smem, st);
    return pick_e<NM, 0, Entry>(edits, p, grid, smem, st);
}

template <int NM, class Entry>
static int go_rewalk(const CamParams &p, cudaStream_t st) {
    auto kern = k_camera_rewalk<NM, Entry>;
    const size_t smem = stack_bytes(p.T.depth, std::is_same<Entry, EntryW>::value, false, kTileRays);
    int r = prep_smem(kern, smem);
    if (r) return r;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    launch_pdl(kern, dim3((unsigned)(2 * sms)), dim3(kTileRays), smem, st, p);
    return check_launch("camera_rewalk");
}

int launch_camera_rewalk(int nmax, bool wide, const CamParams &p, cudaStream_t st) {
    return with_nmax(nmax, [&](auto N) {
        constexpr int NM = decltype(N)::value;
        return wide ? go_rewalk<NM, EntryW>(p, st) : go_rewalk<NM, EntryN>(p, st);
    });
}

int launch_camera(int nmax, int mode, bool edits, bool wide, const CamParams &p, unsigned grid, size_t smem,
                  cudaStream_t st, bool long_queue, bool vis) {
    if (vis && (mode != 1 || edits)) return set_error(VV_E_INVALID, "visible-set slices: sliced walks without edits");
    if (long_queue && mode == 1 && !edits) {
        smem = stack_bytes(p.T.depth, wide, false, kTileRays, kSegLong + 3);
        return with_nmax(nmax, [&](auto N) {
            constexpr int NM = decltype(N)::value;
            if (vis && p.S.census)
                return wide ? go<NM, 1, false, EntryW, kSegLong, 3>(p, grid, smem, st)
                            : go<NM, 1, false, EntryN, kSegLong, 3>(p, grid, smem, st);
            if (vis)
                return wide ? go<NM, 1, false, EntryW, kSegLong, 1>(p, grid, smem, st)
                            : go<NM, 1, false, EntryN, kSegLong, 1>(p, grid, smem, st);
            return wide ? go<NM, 1, false, EntryW, kSegLong>(p, grid, smem, st)
                        : go<NM, 1, false, EntryN, kSegLong>(p, grid, smem, st);
        });
    }
    if (vis) {
        smem = stack_bytes(p.T.depth, wide, false, kTileRays);
        return with_nmax(nmax, [&](auto N) {
            constexpr int NM = decltype(N)::value;
            if (p.S.census)  // a census frame: the instantiation that marks every visited leaf
                return wide ? go<NM, 1, false, EntryW, VV_SEG_MIN, 3>(p, grid, smem, st)
                            : go<NM, 1, false, EntryN, VV_SEG_MIN, 3>(p, grid, smem, st);
            return wide ? go<NM, 1, false, EntryW, VV_SEG_MIN, 1>(p, grid, smem, st)
                        : go<NM, 1, false, EntryN, VV_SEG_MIN, 1>(p, grid, smem, st);
        });
    }
    smem = stack_bytes(p.T.depth, wide, false, kTileRays);  // this TU's queue geometry (A/B builds vary it)
    return with_nmax(nmax, [&](auto N) {
        constexpr int NM = decltype(N)::value;
        return wide ? pick<NM, EntryW>(mode, edits, p, grid, smem, st) : pick<NM, EntryN>(mode, edits, p, grid, smem, st);
    });
}

}  // namespace vvk
