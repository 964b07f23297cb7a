// vv_launch_scene.cu -- instantiations of k_render_scene (render_scene path).
#include "vv_kernels.cuh"

namespace vvk {

template <int NM, class Entry, bool LEAN>
static int go(const SceneParams &p, dim3 grid, size_t smem, cudaStream_t st) {
    auto kern = LEAN ? k_render_scene_lean<NM, Entry> : k_render_scene<NM, Entry>;
    int r = prep_smem(kern, smem);
    if (r) return r;
    if (p.work) {  // persistent warps: one resident grid pulls the warp chunks
        kern<<<persistent_grid(kern, kBlock, smem, grid.x * grid.y), kBlock, smem, st>>>(p);
        return check_launch("render_scene");
    }
    kern<<<grid, kBlock, smem, st>>>(p);
    return check_launch("render_scene");
}

int launch_scene(int nmax, bool wide, bool lean, const SceneParams &p, dim3 grid, size_t smem, cudaStream_t st) {
    return with_nmax(nmax, [&](auto N) {
        constexpr int NM = decltype(N)::value;
        if (lean) return wide ? go<NM, EntryW, true>(p, grid, smem, st) : go<NM, EntryN, true>(p, grid, smem, st);
        return wide ? go<NM, EntryW, false>(p, grid, smem, st) : go<NM, EntryN, false>(p, grid, smem, st);
    });
}

}  // namespace vvk
