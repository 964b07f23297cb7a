// vv_launch_multi.cu -- instantiations of k_render_camera_multi (playback:
// several frames of one camera in one walk).
#include "vv_kernels.cuh"

namespace vvk {

// queue threshold for mostly dark trees (as vv_launch_camera.cu)
#ifndef VV_SEG_LONG
#define VV_SEG_LONG 8
#endif
constexpr int kSegLong = VV_SEG_LONG;

template <int NM, int KF, bool EDITS, class Entry, int SEG = VV_SEG_MIN>
static int go(const CamMultiParams &p, unsigned grid, cudaStream_t st) {
    auto kern = k_render_camera_multi<NM, KF, EDITS, Entry, SEG>;
    const size_t smem = stack_bytes(p.T.depth, Entry::kBytes == EntryW::kBytes, false, kTileRays, SEG + 3);
    int r = prep_smem(kern, smem);
    if (r) return r;
    // persistent warps (a plan): one resident grid pulls the warp chunks
    kern<<<p.work ? persistent_grid(kern, kTileRays, smem, grid) : grid, kTileRays, smem, st>>>(p);
    return check_launch("render_camera_multi");
}

template <int NM, class Entry>
static int pick(int kf, bool edits, const CamMultiParams &p, unsigned grid, cudaStream_t st) {
    switch (kf) {
        case 2: return edits ? go<NM, 2, true, Entry>(p, grid, st) : go<NM, 2, false, Entry>(p, grid, st);
        case 3: return edits ? go<NM, 3, true, Entry>(p, grid, st) : go<NM, 3, false, Entry>(p, grid, st);
        case 4: return edits ? go<NM, 4, true, Entry>(p, grid, st) : go<NM, 4, false, Entry>(p, grid, st);
        default: return set_error(VV_E_UNSUPPORTED, "%d frames per walk (2..%d)", kf, kMaxMulti);
    }
}

template <int NM, class Entry>
static int pick_long(int kf, const CamMultiParams &p, unsigned grid, cudaStream_t st) {
    switch (kf) {
        case 2: return go<NM, 2, false, Entry, kSegLong>(p, grid, st);
        case 3: return go<NM, 3, false, Entry, kSegLong>(p, grid, st);
        case 4: return go<NM, 4, false, Entry, kSegLong>(p, grid, st);
        default: return set_error(VV_E_UNSUPPORTED, "%d frames per walk (2..%d)", kf, kMaxMulti);
    }
}

int launch_camera_multi(int nmax, int kf, bool edits, bool wide, const CamMultiParams &p, unsigned grid,
                        cudaStream_t st, bool long_queue) {
    if (long_queue && !edits)
        return with_nmax(nmax, [&](auto N) {
            constexpr int NM = decltype(N)::value;
            return wide ? pick_long<NM, EntryW>(kf, p, grid, st) : pick_long<NM, EntryN>(kf, p, grid, st);
        });
    return with_nmax(nmax, [&](auto N) {
        constexpr int NM = decltype(N)::value;
        return wide ? pick<NM, EntryW>(kf, edits, p, grid, st) : pick<NM, EntryN>(kf, edits, p, grid, st);
    });
}

}  // namespace vvk
