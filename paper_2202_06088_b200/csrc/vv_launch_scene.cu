// vv_launch_scene.cu -- instantiations of k_render_scene (render_scene path).
#include "vv_kernels.cuh"

namespace vvk {

template <int NM, class Entry>
static int go(const SceneParams &p, dim3 grid, size_t smem, cudaStream_t st) {
    auto kern = k_render_scene<NM, Entry>;
    int r = prep_smem(kern, smem);
    if (r) return r;
    kern<<<grid, kBlock, smem, st>>>(p);
    return check_launch("render_scene");
}

int launch_scene(int nmax, bool wide, const SceneParams &p, dim3 grid, size_t smem, cudaStream_t st) {
    return with_nmax(nmax, [&](auto N) {
        constexpr int NM = decltype(N)::value;
        return wide ? go<NM, EntryW>(p, grid, smem, st) : go<NM, EntryN>(p, grid, smem, st);
    });
}

}  // namespace vvk
