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

template <int NM, class Entry, bool VIS>
static int pick(bool cached, bool edits, const RaysParams &p, unsigned grid, size_t smem, cudaStream_t st) {
    if (cached) return edits ? go<NM, 1, true, Entry, VIS>(p, grid, smem, st) : go<NM, 1, false, Entry, VIS>(p, grid, smem, st);
    return edits ? go<NM, 0, true, Entry, VIS>(p, grid, smem, st) : go<NM, 0, false, Entry, VIS>(p, grid, smem, st);
}

int launch_rays(int nmax, bool cached, bool edits, bool wide, bool visits, const RaysParams &p, unsigned grid,
                size_t smem, cudaStream_t st) {
    return with_nmax(nmax, [&](auto N) {
        constexpr int NM = decltype(N)::value;
        if (wide) return visits ? pick<NM, EntryW, true>(cached, edits, p, grid, smem, st)
                                : pick<NM, EntryW, false>(cached, edits, p, grid, smem, st);
        return visits ? pick<NM, EntryN, true>(cached, edits, p, grid, smem, st)
                      : pick<NM, EntryN, false>(cached, edits, p, grid, smem, st);
    });
}

}  // namespace vvk
