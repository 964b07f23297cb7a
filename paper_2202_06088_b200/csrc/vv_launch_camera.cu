// vv_launch_camera.cu -- instantiations of k_render_camera (render / tiles path).
#include "vv_kernels.cuh"

namespace vvk {

template <int NM, int CACHED, bool EDITS, class Entry>
static int go(const CamParams &p, unsigned max_blocks, size_t smem, cudaStream_t st) {
    auto kern = k_render_camera<NM, CACHED, EDITS, Entry>;
    int r = prep_smem(kern, smem);
    if (r) return r;
    kern<<<max_blocks, kBlock, smem, st>>>(p);
    return check_launch("render_camera");
}

int launch_camera(int nmax, bool cached, bool edits, bool wide, const CamParams &p, unsigned grid, size_t smem,
                  cudaStream_t st) {
    return with_nmax(nmax, [&](auto N) {
        constexpr int NM = decltype(N)::value;
        if (wide) {
            if (cached) return edits ? go<NM, 1, true, EntryW>(p, grid, smem, st) : go<NM, 1, false, EntryW>(p, grid, smem, st);
            return edits ? go<NM, 0, true, EntryW>(p, grid, smem, st) : go<NM, 0, false, EntryW>(p, grid, smem, st);
        }
        if (cached) return edits ? go<NM, 1, true, EntryN>(p, grid, smem, st) : go<NM, 1, false, EntryN>(p, grid, smem, st);
        return edits ? go<NM, 0, true, EntryN>(p, grid, smem, st) : go<NM, 0, false, EntryN>(p, grid, smem, st);
    });
}

}  // namespace vvk
