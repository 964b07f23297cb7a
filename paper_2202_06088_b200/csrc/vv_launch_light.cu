// vv_launch_light.cu -- lighting passes of render_scene (compose.py:539-619):
// the shadow map blur and the per-pixel falloff / ground-shadow / background
// composite.  f64 throughout, in the reference's operation order.
#include "vv_kernels.cuh"

namespace vvk {

// ------------------------------------------------------------------ shadow blur
// scipy.ndimage.gaussian_filter (mode "constant", cval 0): correlate1d along
// axis 0 (rows), then axis 1, each with scipy's symmetric-kernel loop
//   out[i] = x[i] w[r] + sum_{j = r..1} (x[i - j] + x[i + j]) w[r - j]
// (ni_filters.c, NI_Correlate1D), zero outside the map.
template <bool ROWS, class In>
__global__ void k_blur1d(const In *__restrict__ in, int res, const double *__restrict__ w, int r,
                         double *__restrict__ out) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= res * res) return;
    const int y = idx / res, x = idx % res;
    auto at = [&](int k) -> double {  // element k along the filtered axis, 0 outside
        if (k < 0 || k >= res) return 0.0;
        return (double)(ROWS ? in[(size_t)k * res + x] : in[(size_t)y * res + k]);
    };
    const int c = ROWS ? y : x;
    double acc = xmul(at(c), w[r]);
    for (int j = r; j >= 1; --j) acc = xadd(acc, xmul(xadd(at(c - j), at(c + j)), w[r - j]));
    out[idx] = acc;
}

__global__ void k_widen(const float *__restrict__ in, int n, double *__restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (double)in[i];
}

int launch_shadow_blur(const float *alpha, int res, const double *weights, int radius, double *tmp, double *out,
                       cudaStream_t st) {
    const int n = res * res, g = (n + 255) / 256;
    if (n <= 0) return VV_OK;
    if (radius <= 0) {
        k_widen<<<g, 256, 0, st>>>(alpha, n, out);
        return check_launch("shadow_widen");
    }
    k_blur1d<true, float><<<g, 256, 0, st>>>(alpha, res, weights, radius, tmp);
    k_blur1d<false, double><<<g, 256, 0, st>>>(tmp, res, weights, radius, out);
    return check_launch("shadow_blur");
}

// ------------------------------------------------------------------ lights + composite
struct LightParams {
    CamView cam;
    const float *rgb, *alpha, *depth;
    double bg0, bg1, bg2;
    const LightView *L;  // (n_lights) device array
    int n_lights;
    float *image;
    float *lit_rgb;  // optional: the blended rgb after the falloffs (render_scene's returned `blended`)
};

// map_coordinates(order=1, mode="constant", cval=0): bilinear inside
// [0, res-1] on both axes, 0 outside (scipy 1.18)
__device__ __forceinline__ double sample_map(const double *m, int res, double py, double px) {
    const double hi = (double)(res - 1);
    if (!(py >= 0.0 && py <= hi && px >= 0.0 && px <= hi)) return 0.0;  // NaN -> 0 too
    const int y0 = min((int)floor(py), res - 1), x0 = min((int)floor(px), res - 1);
    const int y1 = min(y0 + 1, res - 1), x1 = min(x0 + 1, res - 1);
    const double fy = xsub(py, (double)y0), fx = xsub(px, (double)x0);
    const double v00 = m[(size_t)y0 * res + x0], v01 = m[(size_t)y0 * res + x1];
    const double v10 = m[(size_t)y1 * res + x0], v11 = m[(size_t)y1 * res + x1];
    const double top = xadd(xmul(v00, xsub(1.0, fx)), xmul(v01, fx));
    const double bot = xadd(xmul(v10, xsub(1.0, fx)), xmul(v11, fx));
    return xadd(xmul(top, xsub(1.0, fy)), xmul(bot, fy));
}

__global__ void k_scene_light(const __grid_constant__ LightParams p) {
    const int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t npix = (int64_t)p.cam.width * p.cam.height;
    if (pix >= npix) return;
    const int ix = (int)(pix % p.cam.width), iy = (int)(pix / p.cam.width);
    double dx, dy, dz;
    camera_ray(p.cam, ix, iy, dx, dy, dz);  // Camera.rays (render.py:74-83)
    const double ox = p.cam.ox, oy = p.cam.oy, oz = p.cam.oz;
    const double a = (double)p.alpha[pix], dep = (double)p.depth[pix];
    double r = p.rgb[3 * pix + 0], g = p.rgb[3 * pix + 1], b = p.rgb[3 * pix + 2];
    double bg0 = p.bg0, bg1 = p.bg1, bg2 = p.bg2;  // bg *= factor per light
    for (int li = 0; li < p.n_lights; ++li) {
        const LightView L = p.L[li];
        if (L.falloff_enabled && a > 0.0) {  // falloff_pass (compose.py:606-619)
            const double qx = xsub(xadd(ox, xmul(dep, dx)), L.px);
            const double qy = xsub(xadd(oy, xmul(dep, dy)), L.py);
            const double qz = xsub(xadd(oz, xmul(dep, dz)), L.pz);
            const double d2 = xadd(xadd(xmul(qx, qx), xmul(qy, qy)), xmul(qz, qz));
            const double dist = sqrt(d2);
            double s = xdiv(L.r0sq, xadd(L.r0sq, xmul(dist, dist)));
            s = s < L.min_scale ? L.min_scale : (s > 1.0 ? 1.0 : s);
            r = xmul(r, s);
            g = xmul(g, s);
            b = xmul(b, s);
        }
        if (L.cast_shadows) {  // ShadowMap.background_factor (compose.py:564-582)
            const double denom = xadd(xadd(xmul(dx, L.ga), xmul(dy, L.gb)), xmul(dz, L.gc));
            const double num = -xadd(xadd(xadd(xmul(ox, L.ga), xmul(oy, L.gb)), xmul(oz, L.gc)), L.gd);
            const double t = xdiv(num, denom);
            if (isfinite(t) && t > 0.0) {
                const double wx = xadd(ox, xmul(t, dx)), wy = xadd(oy, xmul(t, dy)), wz = xadd(oz, xmul(t, dz));
                const double *m = L.w2c;  // factor_at_points (compose.py:547-561)
                const double p0 = xadd(xadd(xadd(xmul(wx, m[0]), xmul(wy, m[1])), xmul(wz, m[2])), m[3]);
                const double p1 = xadd(xadd(xadd(xmul(wx, m[4]), xmul(wy, m[5])), xmul(wz, m[6])), m[7]);
                const double p2 = xadd(xadd(xadd(xmul(wx, m[8]), xmul(wy, m[9])), xmul(wz, m[10])), m[11]);
                double occ = 0.0;
                if (p2 > 0.0) {
                    const double px = xsub(xadd(xdiv(xmul(L.fx, p0), p2), L.cx), 0.5);
                    const double py = xsub(xadd(xdiv(xmul(L.fy, p1), p2), L.cy), 0.5);
                    occ = sample_map(L.map, L.res, py, px);
                }
                const double f = xsub(1.0, xmul(L.strength, occ));
                bg0 = xmul(bg0, f);
                bg1 = xmul(bg1, f);
                bg2 = xmul(bg2, f);
            }
        }
    }
    if (p.lit_rgb) {
        p.lit_rgb[3 * pix + 0] = (float)r;
        p.lit_rgb[3 * pix + 1] = (float)g;
        p.lit_rgb[3 * pix + 2] = (float)b;
    }
    // composite_background (render.py:243-251) over the darkened background
    const double om = xsub(1.0, a);
    p.image[3 * pix + 0] = (float)xadd(xmul(a, r), xmul(om, bg0));
    p.image[3 * pix + 1] = (float)xadd(xmul(a, g), xmul(om, bg1));
    p.image[3 * pix + 2] = (float)xadd(xmul(a, b), xmul(om, bg2));
}

int launch_scene_light(const CamView &cam, const float *rgb, const float *alpha, const float *depth, double bg0,
                       double bg1, double bg2, const LightView *lights, int n_lights, float *image, float *lit_rgb,
                       cudaStream_t st) {
    LightParams p;
    p.cam = cam;
    p.rgb = rgb;
    p.alpha = alpha;
    p.depth = depth;
    p.bg0 = bg0;
    p.bg1 = bg1;
    p.bg2 = bg2;
    p.n_lights = n_lights;
    p.L = lights;
    p.image = image;
    p.lit_rgb = lit_rgb;
    const int64_t npix = (int64_t)cam.width * cam.height;
    if (npix == 0) return VV_OK;
    k_scene_light<<<(unsigned)((npix + 255) / 256), 256, 0, st>>>(p);
    return check_launch("scene_light");
}

}  // namespace vvk
