// vv_launch_rays.cu -- instantiations of k_render_rays (render_rays path).
#include "vv_kernels.cuh"

namespace vvk {

template <int NM, int CACHED, bool EDITS, class Entry, bool VIS>
static int go(const RaysParams &p, unsigned grid, size_t smem, cudaStream_t st) {
    auto kern = k_render_rays<NM, CACHED, EDITS, Entry, VIS>;
    int r = prep_smem(kern, smem);
    if (r) return r;
    kern<<<grid, kBlock, smem, st>>>(p);
    return check_launch("render_rays");
}

template <int NM, int MODE, class Entry, bool VIS>
static int pick_e(bool edits, const RaysParams &p, unsigned grid, size_t smem, cudaStream_t st) {
    return edits ? go<NM, MODE, true, Entry, VIS>(p, grid, smem, st) : go<NM, MODE, false, Entry, VIS>(p, grid, smem, st);
}

template <int NM, class Entry, bool VIS>
static int pick(int mode, bool edits, const RaysParams &p, unsigned grid, size_t smem, cudaStream_t st) {
    if (mode == 1) return pick_e<NM, 1, Entry, VIS>(edits, p, grid, smem, st);
    return pick_e<NM, 0, Entry, VIS>(edits, p, grid, smem, st);
}

int launch_rays(int nmax, int mode, bool edits, bool wide, bool visits, const RaysParams &p, unsigned grid,
                size_t smem, cudaStream_t st) {
    return with_nmax(nmax, [&](auto N) {
        constexpr int NM = decltype(N)::value;
        if (wide) return visits ? pick<NM, EntryW, true>(mode, edits, p, grid, smem, st)
                                : pick<NM, EntryW, false>(mode, edits, p, grid, smem, st);
        return visits ? pick<NM, EntryN, true>(mode, edits, p, grid, smem, st)
                      : pick<NM, EntryN, false>(mode, edits, p, grid, smem, st);
    });
}

}  // namespace vvk
