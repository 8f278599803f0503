// ref_glue.cpp — the darbs_cpu.h interface implemented by CALLING THE REFERENCE.
//
// TEST INFRASTRUCTURE, NOT PRODUCT.  oracle/Makefile compiles this file together
// with the reference's own, unmodified sources
//   /root/reference/proj/core/src/{kernel,geometry,rasterizer,loss,fit3d,fit2d,scene_io,image}.cpp
// (read where they lie; never copied) against oracle/eigen_shim into
// oracle/_ref/libdarbs_ref.so.  It only marshals flat FP64 arrays into the
// reference's types and back; no algorithm of the hot path is restated here
// except the ten-line per-splat chain of fit_scene's evaluate lambda
// (fit3d.cpp:134-159), which is not callable from outside fit_scene and is
// therefore spelled out below with the reference's own types and
// backward_projection.
#include <cmath>
#include <cstring>
#include <random>
#include <vector>

#include "darbs/errors.hpp"
#include "darbs/fit2d.hpp"
#include "darbs/fit3d.hpp"
#include "darbs/fit_common.hpp"
#include "darbs/geometry.hpp"
#include "darbs/kernel.hpp"
#include "darbs/loss.hpp"
#include "darbs/optim.hpp"
#include "darbs/psi_table.hpp"
#include "darbs/rasterizer.hpp"
#include "darbs/scene_io.hpp"
#include "darbs_cpu.h"

using namespace darbs;

namespace {

KernelSpec to_spec(const darbs_cpu_kernel* k) {
    KernelSpec s;
    s.family = static_cast<KernelFamily>(k->family);
    s.beta = k->beta;
    s.xi = k->xi;
    s.lobes = k->lobes;
    s.cutoff = k->cutoff;
    s.unbounded = k->unbounded != 0;
    return s;
}

void from_spec(const KernelSpec& s, darbs_cpu_kernel* k) {
    k->family = static_cast<int>(s.family);
    k->beta = s.beta;
    k->xi = s.xi;
    k->lobes = s.lobes;
    k->cutoff = s.cutoff;
    k->unbounded = s.unbounded ? 1 : 0;
}

int status_of_current_exception() {
    try {
        throw;
    } catch (const invalid_parameter&) {
        return DARBS_CPU_INVALID_PARAMETER;
    } catch (const contract_violation&) {
        return DARBS_CPU_CONTRACT_VIOLATION;
    } catch (const numeric_error&) {
        return DARBS_CPU_NUMERIC_ERROR;
    } catch (...) {
        return DARBS_CPU_NUMERIC_ERROR;
    }
}

std::vector<ProjectedSplat> to_splats(int n, const double* mu2, const double* conic,
                                      const double* radius, const double* depth,
                                      const double* opacity, const double* rgb) {
    std::vector<ProjectedSplat> v(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) {
        ProjectedSplat& s = v[i];
        s.mu2 = Vec2(mu2[2 * i], mu2[2 * i + 1]);
        s.conic = Conic{conic[3 * i], conic[3 * i + 1], conic[3 * i + 2]};
        s.radius = radius ? radius[i] : 0.0;
        s.depth = depth ? depth[i] : 0.0;
        s.opacity = opacity ? opacity[i] : 1.0;
        if (rgb) s.color = Vec3(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]);
    }
    return v;
}

Primitive3D to_prim(const double* p) {
    Primitive3D q;
    q.mu = Vec3(p[0], p[1], p[2]);
    q.scale = Vec3(p[3], p[4], p[5]);
    q.rot = Eigen::Quaterniond(p[6], p[7], p[8], p[9]);
    q.opacity = p[10];
    q.color = Vec3(p[11], p[12], p[13]);
    return q;
}

Camera to_camera(const double* c) {
    Camera cam;
    cam.fx = c[0];
    cam.fy = c[1];
    cam.cx = c[2];
    cam.cy = c[3];
    cam.width = static_cast<int>(c[4]);
    cam.height = static_cast<int>(c[5]);
    for (int r = 0; r < 4; ++r)
        for (int col = 0; col < 4; ++col) cam.w(r, col) = c[6 + 4 * r + col];
    return cam;
}

inline double rf(double v, int round_f32) {
    return round_f32 ? static_cast<double>(static_cast<float>(v)) : v;
}

struct ForwardHandle {
    ForwardResult res;
};

}  // namespace

extern "C" {

const char* darbs_cpu_kind(void) { return "reference"; }

int darbs_cpu_make_kernel(int family, double beta, double xi, int lobes, darbs_cpu_kernel* out) {
    if (family < 0 || family > 4) return DARBS_CPU_INVALID_PARAMETER;
    try {
        from_spec(make_kernel(static_cast<KernelFamily>(family), beta, xi, lobes), out);
    } catch (...) {
        return status_of_current_exception();
    }
    return DARBS_CPU_OK;
}

int darbs_cpu_kernel_preset(const char* name, darbs_cpu_kernel* out) {
    auto s = kernel_preset(name);
    if (!s) return DARBS_CPU_INVALID_PARAMETER;
    from_spec(*s, out);
    return DARBS_CPU_OK;
}

double darbs_cpu_default_psi(const char* name) {
    auto p = default_psi(name);
    return p ? p->psi : -1.0;
}

int darbs_cpu_eval(const darbs_cpu_kernel* k, int n, const double* dm2, double* weight,
                   double* dweight_ddm2) {
    KernelSpec s = to_spec(k);
    try {
        for (int i = 0; i < n; ++i) {
            KernelSample ks = eval(s, dm2[i]);
            if (weight) weight[i] = ks.weight;
            if (dweight_ddm2) dweight_ddm2[i] = ks.dweight_ddm2;
        }
    } catch (...) {
        return status_of_current_exception();
    }
    return DARBS_CPU_OK;
}

int darbs_cpu_conic_and_radius(const darbs_cpu_kernel* k, int n, const double* cov2,
                               double* conic, double* radius, double* lambda12) {
    KernelSpec s = to_spec(k);
    try {
        for (int i = 0; i < n; ++i) {
            Mat2 c;
            c << cov2[3 * i], cov2[3 * i + 1], cov2[3 * i + 1], cov2[3 * i + 2];
            ConicRadius cr = conic_and_radius(c, s);
            conic[3 * i] = cr.conic.a;
            conic[3 * i + 1] = cr.conic.b;
            conic[3 * i + 2] = cr.conic.c;
            radius[i] = cr.radius;
            if (lambda12) {
                lambda12[2 * i] = cr.lambda1;
                lambda12[2 * i + 1] = cr.lambda2;
            }
        }
    } catch (...) {
        return status_of_current_exception();
    }
    return DARBS_CPU_OK;
}

int darbs_cpu_random_scene(const darbs_cpu_kernel* k, int count, int width, int height,
                           uint64_t seed, int round_f32, double* mu2, double* cov2,
                           double* conic, double* radius, double* depth, double* opacity,
                           double* rgb) {
    // The fixture of benchmarks/bench.cpp:20-46, built from the real
    // std::mt19937_64 / std::uniform_real_distribution.
    KernelSpec kernel = to_spec(k);
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> ux(-5.0, width + 5.0);
    std::uniform_real_distribution<double> uy(-5.0, height + 5.0);
    std::uniform_real_distribution<double> uvar(0.6, 12.0);
    std::uniform_real_distribution<double> ucorr(-0.6, 0.6);
    std::uniform_real_distribution<double> uop(0.1, 0.95);
    std::uniform_real_distribution<double> ucol(0.0, 1.0);
    std::uniform_real_distribution<double> udep(0.5, 9.5);
    try {
        for (int i = 0; i < count; ++i) {
            double a = uvar(rng), c = uvar(rng);
            double b = ucorr(rng) * std::sqrt(a * c);
            double mx = ux(rng);
            double my = uy(rng);
            a = rf(a, round_f32);
            b = rf(b, round_f32);
            c = rf(c, round_f32);
            Mat2 cov;
            cov << a, b, b, c;
            ConicRadius cr = conic_and_radius(cov, kernel);
            cov2[3 * i] = a;
            cov2[3 * i + 1] = b;
            cov2[3 * i + 2] = c;
            mu2[2 * i] = rf(mx, round_f32);
            mu2[2 * i + 1] = rf(my, round_f32);
            conic[3 * i] = rf(cr.conic.a, round_f32);
            conic[3 * i + 1] = rf(cr.conic.b, round_f32);
            conic[3 * i + 2] = rf(cr.conic.c, round_f32);
            radius[i] = cr.radius;
            depth[i] = rf(udep(rng), round_f32);
            opacity[i] = rf(uop(rng), round_f32);
            for (int e = 0; e < 3; ++e) rgb[3 * i + e] = rf(ucol(rng), round_f32);
        }
    } catch (...) {
        return status_of_current_exception();
    }
    return DARBS_CPU_OK;
}

void darbs_cpu_random_image_grad(int width, int height, uint64_t seed, int round_f32,
                                 double* grad_image) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    std::size_t n = std::size_t(width) * height * 3;
    for (std::size_t i = 0; i < n; ++i) grad_image[i] = rf(u(rng), round_f32);
}

int64_t darbs_cpu_bin(int n, const double* mu2, const double* conic, const double* radius,
                      const double* depth, int width, int height, int64_t* tile_offsets,
                      int32_t* point_list, int64_t capacity, int32_t* depth_order) {
    auto splats = to_splats(n, mu2, conic, radius, depth, nullptr, nullptr);
    TileBins bins = bin_splats(splats, width, height);
    int64_t k = 0;
    for (std::size_t t = 0; t < bins.lists.size(); ++t) {
        if (tile_offsets) tile_offsets[t] = k;
        k += static_cast<int64_t>(bins.lists[t].size());
    }
    if (tile_offsets) tile_offsets[bins.lists.size()] = k;
    if (point_list && k <= capacity) {
        int64_t o = 0;
        for (const auto& l : bins.lists)
            for (int idx : l) point_list[o++] = idx;
    }
    if (depth_order) {
        // The reference does not expose its depth order; recover it the way
        // bin_splats builds it (rasterizer.cpp:31-35).
        std::vector<int> order(n);
        for (int i = 0; i < n; ++i) order[i] = i;
        std::stable_sort(order.begin(), order.end(),
                         [&](int a, int b) { return depth[a] < depth[b]; });
        for (int i = 0; i < n; ++i) depth_order[i] = order[i];
    }
    return k;
}

void* darbs_cpu_forward(const darbs_cpu_kernel* k, int n, const double* mu2, const double* conic,
                        const double* radius, const double* depth, const double* opacity,
                        const double* rgb, int width, int height, const double* background,
                        int threads, double* image, double* t_final, int32_t* processed,
                        int32_t* contributors, int32_t* skipped_nonfinite) {
    auto splats = to_splats(n, mu2, conic, radius, depth, opacity, rgb);
    auto* h = new ForwardHandle;
    try {
        h->res = forward(splats, to_spec(k), width, height,
                         Vec3(background[0], background[1], background[2]), threads);
    } catch (...) {
        delete h;
        return nullptr;
    }
    const BlendAux& aux = h->res.aux;
    std::size_t px = std::size_t(width) * height;
    if (image) std::memcpy(image, h->res.image.rgb.data(), sizeof(double) * px * 3);
    if (t_final) std::memcpy(t_final, aux.t_final.data(), sizeof(double) * px);
    if (processed) std::memcpy(processed, aux.processed.data(), sizeof(int32_t) * px);
    if (contributors) std::memcpy(contributors, aux.contributors.data(), sizeof(int32_t) * px);
    if (skipped_nonfinite) *skipped_nonfinite = aux.skipped_nonfinite;
    return h;
}

void darbs_cpu_forward_free(void* handle) { delete static_cast<ForwardHandle*>(handle); }

int darbs_cpu_oracle_forward(const darbs_cpu_kernel* k, int n, const double* mu2,
                             const double* conic, const double* radius, const double* depth,
                             const double* opacity, const double* rgb, int width, int height,
                             const double* background, double* image) {
    auto splats = to_splats(n, mu2, conic, radius, depth, opacity, rgb);
    try {
        ImageBuffer img = oracle_forward(splats, to_spec(k), width, height,
                                         Vec3(background[0], background[1], background[2]));
        std::memcpy(image, img.rgb.data(), sizeof(double) * img.rgb.size());
    } catch (...) {
        return status_of_current_exception();
    }
    return DARBS_CPU_OK;
}

int darbs_cpu_backward(void* handle, const darbs_cpu_kernel* k, int grad_width, int grad_height,
                       const double* grad_image, int n, const double* mu2, const double* conic,
                       const double* opacity, const double* rgb, int threads, double* grads) {
    auto* h = static_cast<ForwardHandle*>(handle);
    if (!h) return DARBS_CPU_CONTRACT_VIOLATION;
    ImageBuffer g(grad_width, grad_height);
    std::memcpy(g.rgb.data(), grad_image, sizeof(double) * g.rgb.size());
    auto splats = to_splats(n, mu2, conic, nullptr, nullptr, opacity, rgb);
    try {
        std::vector<SplatGrads> sg = backward(g, splats, to_spec(k), h->res.aux, threads);
        for (int i = 0; i < n; ++i) {
            double* o = grads + 9 * std::size_t(i);
            o[0] = sg[i].d_color[0];
            o[1] = sg[i].d_color[1];
            o[2] = sg[i].d_color[2];
            o[3] = sg[i].d_opacity;
            o[4] = sg[i].d_conic_a;
            o[5] = sg[i].d_conic_b;
            o[6] = sg[i].d_conic_c;
            o[7] = sg[i].d_mu2[0];
            o[8] = sg[i].d_mu2[1];
        }
    } catch (...) {
        return status_of_current_exception();
    }
    return DARBS_CPU_OK;
}

void darbs_cpu_realize(int n, const double* raw, double* prims) {
    // realize() is file-local in fit3d.cpp:17-25; same expressions, using the
    // reference's sigmoid (fit_common.hpp:40).
    for (int i = 0; i < n; ++i) {
        const double* q = raw + 14 * std::size_t(i);
        double* p = prims + 14 * std::size_t(i);
        p[0] = q[0];
        p[1] = q[1];
        p[2] = q[2];
        for (int a = 3; a < 6; ++a) p[a] = std::exp(q[a]);
        for (int a = 6; a < 10; ++a) p[a] = q[a];
        for (int a = 10; a < 14; ++a) p[a] = sigmoid(q[a]);
    }
}

int darbs_cpu_project(const darbs_cpu_kernel* k, double psi, double dilation, int n,
                      const double* prims, const double* camera, int32_t* valid, double* mu2,
                      double* cov2, double* conic, double* radius, double* depth) {
    KernelSpec kernel = to_spec(k);
    Camera cam = to_camera(camera);
    try {
        for (int i = 0; i < n; ++i) {
            auto s = project_primitive(to_prim(prims + 14 * std::size_t(i)), cam, kernel, psi,
                                       dilation);
            valid[i] = s ? 1 : 0;
            if (!s) {
                mu2[2 * i] = mu2[2 * i + 1] = 0.0;
                cov2[3 * i] = cov2[3 * i + 1] = cov2[3 * i + 2] = 0.0;
                conic[3 * i] = conic[3 * i + 1] = conic[3 * i + 2] = 0.0;
                radius[i] = depth[i] = 0.0;
                continue;
            }
            mu2[2 * i] = s->mu2.x();
            mu2[2 * i + 1] = s->mu2.y();
            cov2[3 * i] = s->cov2(0, 0);
            cov2[3 * i + 1] = s->cov2(0, 1);
            cov2[3 * i + 2] = s->cov2(1, 1);
            conic[3 * i] = s->conic.a;
            conic[3 * i + 1] = s->conic.b;
            conic[3 * i + 2] = s->conic.c;
            radius[i] = s->radius;
            depth[i] = s->depth;
        }
    } catch (...) {
        return status_of_current_exception();
    }
    return DARBS_CPU_OK;
}

void darbs_cpu_backward_projection(double psi, int n, const double* grad_cov2,
                                   const double* grad_mu2, const double* prims,
                                   const double* camera, double* d_mu, double* d_scale,
                                   double* d_rot) {
    Camera cam = to_camera(camera);
    for (int i = 0; i < n; ++i) {
        Mat2 gc;
        gc << grad_cov2[4 * i], grad_cov2[4 * i + 1], grad_cov2[4 * i + 2], grad_cov2[4 * i + 3];
        ProjectionGrads pg = backward_projection(gc, Vec2(grad_mu2[2 * i], grad_mu2[2 * i + 1]),
                                                 to_prim(prims + 14 * std::size_t(i)), cam, psi);
        for (int a = 0; a < 3; ++a) d_mu[3 * i + a] = pg.d_mu[a];
        for (int a = 0; a < 3; ++a) d_scale[3 * i + a] = pg.d_scale[a];
        for (int a = 0; a < 4; ++a) d_rot[4 * i + a] = pg.d_rot[a];
    }
}

void darbs_cpu_param_grads(double psi, int m, const int32_t* owner, const double* splat_grads,
                           const double* conic, const double* opacity, const double* rgb,
                           const double* prims, const double* camera, double* param_grads) {
    Camera cam = to_camera(camera);
    for (int k = 0; k < m; ++k) {
        const double* gi = splat_grads + 9 * std::size_t(k);
        int i = owner[k];
        double* g = param_grads + 14 * std::size_t(i);
        Primitive3D prim = to_prim(prims + 14 * std::size_t(i));
        // fit3d.cpp:140-144
        Mat2 gc;
        gc << gi[4], 0.5 * gi[5], 0.5 * gi[5], gi[6];
        Mat2 cmat;
        cmat << conic[3 * k], conic[3 * k + 1], conic[3 * k + 1], conic[3 * k + 2];
        Mat2 d_cov2 = -cmat * gc * cmat;
        ProjectionGrads pg = backward_projection(d_cov2, Vec2(gi[7], gi[8]), prim, cam, psi);
        // fit3d.cpp:148-158
        g[0] += pg.d_mu.x();
        g[1] += pg.d_mu.y();
        g[2] += pg.d_mu.z();
        for (int a = 0; a < 3; ++a) g[3 + a] += pg.d_scale[a] * prim.scale[a];
        for (int a = 0; a < 4; ++a) g[6 + a] += pg.d_rot[a];
        g[10] += gi[3] * opacity[k] * (1.0 - opacity[k]);
        for (int c = 0; c < 3; ++c) g[11 + c] += gi[c] * rgb[3 * k + c] * (1.0 - rgb[3 * k + c]);
    }
}

void darbs_cpu_random_image(int width, int height, uint64_t seed, int round_f32, double* rgb) {
    std::mt19937_64 rng(seed);  // tests/test_loss.cpp:13-19
    std::uniform_real_distribution<double> u(0.0, 1.0);
    std::size_t n = std::size_t(width) * height * 3;
    for (std::size_t i = 0; i < n; ++i) rgb[i] = rf(u(rng), round_f32);
}

static ImageBuffer to_image(int width, int height, const double* rgb) {
    ImageBuffer img(width, height);
    std::memcpy(img.rgb.data(), rgb, sizeof(double) * img.rgb.size());
    return img;
}

int darbs_cpu_loss_total(int width, int height, const double* rendered, const double* target,
                         double lambda, double out[3], double* grad) {
    try {
        LossResult r = loss_total(to_image(width, height, rendered), to_image(width, height, target), lambda);
        out[0] = r.total;
        out[1] = r.l1;
        out[2] = r.dssim;
        if (grad) std::memcpy(grad, r.grad.rgb.data(), sizeof(double) * r.grad.rgb.size());
    } catch (...) {
        return status_of_current_exception();
    }
    return DARBS_CPU_OK;
}

int darbs_cpu_ssim(int width, int height, const double* a, const double* b, double* out) {
    try {
        *out = ssim(to_image(width, height, a), to_image(width, height, b));
    } catch (...) {
        return status_of_current_exception();
    }
    return DARBS_CPU_OK;
}

// ---- file formats (reference build only): src/scene_io.cpp, src/image.cpp.  Used by
// tests/golden/make_golden.py to write the I/O fixtures the C++ mirror is byte-compared with.
int darbs_cpu_write_scene(const char* path, int n, const double* prims) {
    try {
        std::vector<Primitive3D> v;
        for (int i = 0; i < n; ++i) v.push_back(to_prim(prims + 14 * std::size_t(i)));
        write_scene(v, path);
    } catch (...) {
        return status_of_current_exception();
    }
    return DARBS_CPU_OK;
}

int darbs_cpu_read_scene(const char* path, int capacity, double* prims) {
    try {
        std::vector<Primitive3D> v = read_scene(path);
        for (std::size_t i = 0; i < v.size() && int(i) < capacity; ++i) {
            double* o = prims + 14 * i;
            for (int k = 0; k < 3; ++k) o[k] = v[i].mu[k];
            for (int k = 0; k < 3; ++k) o[3 + k] = v[i].scale[k];
            o[6] = v[i].rot.w();
            o[7] = v[i].rot.x();
            o[8] = v[i].rot.y();
            o[9] = v[i].rot.z();
            o[10] = v[i].opacity;
            for (int k = 0; k < 3; ++k) o[11 + k] = v[i].color[k];
        }
        return int(v.size());
    } catch (...) {
        return -status_of_current_exception();
    }
}

int darbs_cpu_write_cameras(const char* path, int n, const double* cams22) {
    try {
        std::vector<Camera> v;
        for (int i = 0; i < n; ++i) v.push_back(to_camera(cams22 + 22 * std::size_t(i)));
        write_cameras(v, path);
    } catch (...) {
        return status_of_current_exception();
    }
    return DARBS_CPU_OK;
}

int darbs_cpu_write_image(const char* path, int width, int height, const double* rgb, int as_ppm) {
    try {
        ImageBuffer img = to_image(width, height, rgb);
        if (as_ppm)
            write_ppm(img, path);
        else
            write_float_dump(img, path);
    } catch (...) {
        return status_of_current_exception();
    }
    return DARBS_CPU_OK;
}

int darbs_cpu_adam_step(int64_t dim, double* params, const double* grads, double* m, double* v,
                        const double* lrs, int t) {
    AdamState st(static_cast<std::size_t>(dim));
    std::memcpy(st.m.data(), m, sizeof(double) * dim);
    std::memcpy(st.v.data(), v, sizeof(double) * dim);
    try {
        adam_step(std::span<double>(params, static_cast<std::size_t>(dim)),
                  std::span<const double>(grads, static_cast<std::size_t>(dim)), st,
                  std::span<const double>(lrs, static_cast<std::size_t>(dim)), t);
    } catch (...) {
        return status_of_current_exception();
    }
    std::memcpy(m, st.m.data(), sizeof(double) * dim);
    std::memcpy(v, st.v.data(), sizeof(double) * dim);
    return DARBS_CPU_OK;
}

// ---- the callers of the hot path (reference build only): src/fit3d.cpp, src/fit2d.cpp.  Used by
// tests/golden/make_golden.py to record the reference's own optimisation trajectories on
// proj/data/demo_scene.txt + demo_cameras.txt, which the C++ mirror's fit_scene / fit_image
// (paper_2501_12369_b200/host/darbs_b200_fit.hpp) are compared with on the GPU.
namespace {

void prim_to_flat(const Primitive3D& p, double* o) {
    for (int k = 0; k < 3; ++k) o[k] = p.mu[k];
    for (int k = 0; k < 3; ++k) o[3 + k] = p.scale[k];
    o[6] = p.rot.w();
    o[7] = p.rot.x();
    o[8] = p.rot.y();
    o[9] = p.rot.z();
    o[10] = p.opacity;
    for (int k = 0; k < 3; ++k) o[11 + k] = p.color[k];
}

FitConfig to_config(const double* cfg) {
    // cfg = lambda, lr_position, lr_scale, lr_rotation, lr_opacity, lr_color, iters, seed, threads
    FitConfig c;
    c.lambda = cfg[0];
    c.lr_position = cfg[1];
    c.lr_scale = cfg[2];
    c.lr_rotation = cfg[3];
    c.lr_opacity = cfg[4];
    c.lr_color = cfg[5];
    c.iters = int(cfg[6]);
    c.seed = std::uint64_t(cfg[7]);
    c.threads = int(cfg[8]);
    return c;
}

void report_out(const FitReport& r, double* curves, double* finals) {
    // curves = [4][iters]: loss, l1, dssim, psnr; finals = mse, psnr, ssim
    const std::size_t n = r.loss_curve.size();
    for (std::size_t i = 0; i < n; ++i) {
        curves[i] = r.loss_curve[i];
        curves[n + i] = r.l1_curve[i];
        curves[2 * n + i] = r.dssim_curve[i];
        curves[3 * n + i] = r.psnr_curve[i];
    }
    finals[0] = r.final_mse;
    finals[1] = r.final_psnr;
    finals[2] = r.final_ssim;
}

}  // namespace

// render_scene fit3d.cpp:29-40.  prims are realized (to_prim layout); image = 3*w*h.
int darbs_cpu_render_scene(const darbs_cpu_kernel* k, double psi, int n, const double* prims,
                           const double* camera, const double* background, int threads, double* image) {
    try {
        std::vector<Primitive3D> v;
        for (int i = 0; i < n; ++i) v.push_back(to_prim(prims + 14 * std::size_t(i)));
        ImageBuffer img = render_scene(v, to_camera(camera), to_spec(k), psi,
                                       Vec3(background[0], background[1], background[2]), threads);
        std::memcpy(image, img.rgb.data(), sizeof(double) * img.rgb.size());
    } catch (...) {
        return status_of_current_exception();
    }
    return DARBS_CPU_OK;
}

// fit_scene fit3d.cpp:42-203.  targets = n_views images of the cameras' sizes, concatenated.
// curves must hold 4 * max(iters, 1) doubles, per_view_psnr n_views, out_prims 14 * n.
int darbs_cpu_fit_scene(const darbs_cpu_kernel* k, double psi, int n, const double* init_prims, int n_views,
                        const double* cameras22, const double* targets, const double* cfg, double* curves,
                        double* finals, double* per_view_psnr, double* out_prims) {
    try {
        std::vector<Primitive3D> init;
        for (int i = 0; i < n; ++i) init.push_back(to_prim(init_prims + 14 * std::size_t(i)));
        std::vector<View> views;
        const double* t = targets;
        for (int v = 0; v < n_views; ++v) {
            Camera cam = to_camera(cameras22 + 22 * std::size_t(v));
            views.push_back(View{cam, to_image(cam.width, cam.height, t)});
            t += std::size_t(3) * cam.width * cam.height;
        }
        Fit3DResult r = fit_scene(views, to_spec(k), psi, init, to_config(cfg));
        report_out(r.report, curves, finals);
        for (int v = 0; v < n_views; ++v) per_view_psnr[v] = r.per_view_psnr[v];
        for (int i = 0; i < n; ++i) prim_to_flat(r.primitives[i], out_prims + 14 * std::size_t(i));
    } catch (...) {
        return status_of_current_exception();
    }
    return DARBS_CPU_OK;
}

// fit_image fit2d.cpp:45-188.  out_splats = 9 per splat (mu2, log_scale2, angle, opacity logit, colour logits 3).
int darbs_cpu_fit_image(const darbs_cpu_kernel* k, int width, int height, const double* target, int n_splats,
                        const double* cfg, double* curves, double* finals, double* rendered, double* out_splats) {
    try {
        Fit2DResult r = fit_image(to_image(width, height, target), to_spec(k), n_splats, to_config(cfg));
        report_out(r.report, curves, finals);
        std::memcpy(rendered, r.rendered.rgb.data(), sizeof(double) * r.rendered.rgb.size());
        for (int i = 0; i < n_splats; ++i) {
            const Splat2DParams& p = r.splats[i];
            double* o = out_splats + 9 * std::size_t(i);
            o[0] = p.mu2.x();
            o[1] = p.mu2.y();
            o[2] = p.log_scale.x();
            o[3] = p.log_scale.y();
            o[4] = p.angle;
            o[5] = p.opacity_logit;
            for (int c = 0; c < 3; ++c) o[6 + c] = p.color_logit[c];
        }
    } catch (...) {
        return status_of_current_exception();
    }
    return DARBS_CPU_OK;
}

// read_cameras scene_io.cpp; returns the count (or a negative status).
int darbs_cpu_read_cameras(const char* path, int capacity, double* cams22) {
    try {
        std::vector<Camera> v = read_cameras(path);
        for (std::size_t i = 0; i < v.size() && int(i) < capacity; ++i) {
            double* o = cams22 + 22 * i;
            o[0] = v[i].fx;
            o[1] = v[i].fy;
            o[2] = v[i].cx;
            o[3] = v[i].cy;
            o[4] = v[i].width;
            o[5] = v[i].height;
            for (int r = 0; r < 4; ++r)
                for (int c = 0; c < 4; ++c) o[6 + 4 * r + c] = v[i].w(r, c);
        }
        return int(v.size());
    } catch (...) {
        return -status_of_current_exception();
    }
}

}  // extern "C"
