// test_fit.cpp — drives the callers of the hot path through the C++ mirror (darbs_b200_fit.hpp)
// the way the reference's own tests do (tests/test_geometry.cpp, test_loss.cpp, test_fit.cpp).
// Needs a B200; run by tests/test_gpu_host_mirror.py.  Prints "host fit ok" when every check holds.
#define DARBS_B200_AS_DARBS
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "darbs_b200_fit.hpp"

using namespace darbs;

#define CHECK(cond)                                                                       \
    do {                                                                                  \
        if (!(cond)) {                                                                    \
            std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #cond); \
            std::exit(1);                                                                 \
        }                                                                                 \
    } while (0)

static Camera look_down_z(double f, int size, double tz) {
    Camera cam;
    cam.fx = cam.fy = f;
    cam.cx = cam.cy = size / 2.0;
    cam.width = cam.height = size;
    cam.w[2][3] = tz;
    return cam;
}

static Camera rotated_y(Camera cam, double angle, double tz) {
    const double c = std::cos(angle), s = std::sin(angle);
    cam.w[0][0] = c;
    cam.w[0][2] = s;
    cam.w[2][0] = -s;
    cam.w[2][2] = c;
    cam.w[2][3] = tz;
    return cam;
}

int main() {
    const KernelSpec g = *kernel_preset("gaussian");

    // full projection of one primitive (tests/test_geometry.cpp:298-314): scale .5, fx = fy = 10,
    // depth 1 -> cov2 = 25 I + 0.3 I, conic.a = 1 / 25.3
    {
        Primitive3D p;
        p.mu = Vec3(0, 0, 0);
        p.scale = Vec3(0.5, 0.5, 0.5);
        Camera cam = look_down_z(10.0, 64, 1.0);
        auto s = project_primitive(p, cam, g, 1.0);
        CHECK(s.has_value());
        CHECK(std::fabs(s->cov2(0, 0) - 25.3) < 1e-4 && std::fabs(s->cov2(1, 1) - 25.3) < 1e-4);
        CHECK(std::fabs(s->cov2(0, 1)) < 1e-5);
        CHECK(std::fabs(s->conic.a - 1.0 / 25.3) < 1e-7);
        CHECK(std::fabs(s->depth - 1.0) < 1e-6);
        p.mu = Vec3(0, 0, -2.0);  // behind the near plane (geometry.cpp:22)
        CHECK(!project_primitive(p, cam, g, 1.0).has_value());
        // zero upstream gradient -> zero parameter gradient (tests/test_geometry.cpp:222-230)
        p.mu = Vec3(0.1, -0.2, 0.3);
        Mat2 zero;
        zero(0, 0) = zero(1, 1) = 0.0;
        ProjectionGrads pg = backward_projection(zero, Vec2::Zero(), p, cam, 1.0);
        for (int k = 0; k < 3; ++k) CHECK(pg.d_mu[k] == 0.0 && pg.d_scale[k] == 0.0);
        // conic_and_radius known answers (tests/test_geometry.cpp:181-197)
        Mat2 unit;
        CHECK(conic_and_radius(unit, g).radius == 3.0);
        bool threw = false;
        try {
            Mat2 bad;
            bad(0, 1) = bad(1, 0) = 2.0;
            conic_and_radius(bad, g);
        } catch (const numeric_error&) {
            threw = true;
        }
        CHECK(threw);
        KernelSample ks = eval(g, 0.0);
        CHECK(std::fabs(ks.weight - 1.0) < 1e-7);
    }

    // loss: identical images and a constant offset (tests/test_loss.cpp:23-45)
    {
        std::mt19937_64 rng(1);
        std::uniform_real_distribution<double> u(0.0, 0.8);
        ImageBuffer x(16, 16);
        for (double& v : x.rgb) v = (float)u(rng);
        CHECK(std::fabs(ssim(x, x) - 1.0) < 1e-6);
        LossResult same = loss_total(x, x, 0.2);
        CHECK(std::fabs(same.total) < 1e-6);
        for (double v : same.grad.rgb) CHECK(std::fabs(v) < 1e-9);
        ImageBuffer y = x;
        for (double& v : y.rgb) v = (float)(v + 0.1);
        LossResult off = loss_total(y, x, 0.0);
        CHECK(std::fabs(off.total - 0.1) < 1e-6 && std::fabs(off.l1 - 0.1) < 1e-6);
        bool threw = false;
        try {
            loss_total(ImageBuffer(8, 8), ImageBuffer(8, 9), 0.2);
        } catch (const invalid_parameter&) {
            threw = true;
        }
        CHECK(threw);
    }

    // adam (tests/test_loss.cpp:84-115)
    {
        std::vector<double> p{1.0, -2.0, 3.0}, zero{0.0, 0.0, 0.0}, lrs{0.1, 0.1, 0.1};
        AdamState st(3);
        adam_step(p, zero, st, lrs, 1);
        CHECK(p[0] == 1.0 && p[1] == -2.0 && p[2] == 3.0);
        std::vector<double> grad{0.5, -0.5, 2.0};
        adam_step(p, grad, st, lrs, 1);
        CHECK(std::fabs(p[0] - 0.9) < 1e-6 && std::fabs(p[1] + 1.9) < 1e-6 && std::fabs(p[2] - 2.9) < 1e-6);
        bool threw = false;
        try {
            std::vector<double> shorter{0.0, 0.0};
            adam_step(p, shorter, st, lrs, 1);
        } catch (const contract_violation&) {
            threw = true;
        }
        CHECK(threw);
    }

    // scene fit: zero iterations change nothing and report the initial loss (tests/test_fit.cpp:134-172)
    std::vector<Primitive3D> truth;
    {
        std::mt19937_64 rng(3);
        std::uniform_real_distribution<double> u(-0.5, 0.5);
        for (int i = 0; i < 5; ++i) {
            Primitive3D p;
            p.mu = Vec3((float)u(rng), (float)u(rng), (float)u(rng));
            p.scale = Vec3(0.2, 0.25, 0.15);
            p.opacity = 0.8;
            p.color = Vec3(0.9, 0.4, 0.2);
            truth.push_back(p);
        }
    }
    const Camera cam1 = look_down_z(60.0, 48, 3.0);
    const Camera cam2 = rotated_y(cam1, 0.3, 3.2);
    std::vector<View> views;
    for (const Camera& c : {cam1, cam2}) views.push_back(View{c, render_scene(truth, c, g, 1.0, Vec3::Zero())});
    {
        double lit = 0.0;
        for (double v : views[0].target.rgb) lit += v;
        CHECK(lit > 1.0);  // the scene is in view
        FitConfig cfg;
        cfg.iters = 0;
        Fit3DResult r = fit_scene(views, g, 1.0, truth, cfg);
        CHECK(r.report.loss_curve.size() == 1);
        // raw parameters are float32 on the device: realize(raw(truth)) is truth to FP32 rounding
        CHECK(std::fabs(r.report.loss_curve[0]) < 1e-5);
        for (std::size_t i = 0; i < truth.size(); ++i)
            for (int k = 0; k < 3; ++k) {
                CHECK(std::fabs(r.primitives[i].mu[k] - truth[i].mu[k]) < 1e-6);
                CHECK(std::fabs(r.primitives[i].scale[k] - truth[i].scale[k]) < 1e-6);
            }
        for (double v : r.per_view_psnr) CHECK(v > 60.0);
        // input validation (tests/test_fit.cpp:213-225)
        bool threw = false;
        try {
            fit_scene({views[0]}, g, 1.0, truth, cfg);
        } catch (const invalid_parameter&) {
            threw = true;
        }
        CHECK(threw);
        threw = false;
        try {
            fit_scene(views, g, 1.0, {}, cfg);
        } catch (const invalid_parameter&) {
            threw = true;
        }
        CHECK(threw);
    }
    // a perturbed start converges back towards the targets
    {
        std::vector<Primitive3D> init = truth;
        for (auto& p : init) {
            p.mu[0] += 0.05;
            p.mu[1] -= 0.04;
            p.mu[2] += 0.03;
        }
        FitConfig cfg;
        cfg.iters = 150;
        cfg.lr_position = 0.002;
        Fit3DResult r = fit_scene(views, g, 1.0, init, cfg);
        CHECK(r.report.loss_curve.size() == 150);
        CHECK(r.report.loss_curve.back() < 0.6 * r.report.loss_curve.front());
        CHECK(r.report.final_psnr > r.report.psnr_curve.front());
        // Reruns (tests/test_fit.cpp:174-211 asks 1e-6 across thread counts of a bitwise-deterministic
        // rasterizer): gradients here are accumulated with FP32 atomics, so two runs start identical and
        // drift apart by rounding noise that Adam amplifies; they must agree closely early and end alike.
        Fit3DResult r2 = fit_scene(views, g, 1.0, init, cfg);
        CHECK(r.report.loss_curve[0] == r2.report.loss_curve[0]);
        for (int it = 0; it < 10; ++it) CHECK(std::fabs(r.report.loss_curve[it] - r2.report.loss_curve[it]) < 1e-6);
        std::printf("fit_scene rerun: final loss differs by %.3g\n",
                    std::fabs(r.report.loss_curve.back() - r2.report.loss_curve.back()));
        CHECK(std::fabs(r.report.loss_curve.back() - r2.report.loss_curve.back()) < 0.01 * r.report.loss_curve.front());
        std::printf("fit_scene: loss %.5f -> %.5f, psnr %.2f -> %.2f dB\n", r.report.loss_curve.front(),
                    r.report.loss_curve.back(), r.report.psnr_curve.front(), r.report.final_psnr);
    }

    // image fit: a constant target is reproduced by one splat (tests/test_fit.cpp:120-132)
    {
        ImageBuffer target(24, 24);
        for (std::size_t i = 0; i < target.rgb.size(); i += 3) {
            target.rgb[i] = 0.8;
            target.rgb[i + 1] = 0.3;
            target.rgb[i + 2] = 0.5;
        }
        FitConfig cfg;
        cfg.iters = 600;
        cfg.seed = 2;
        Fit2DResult r = fit_image(target, g, 1, cfg);
        std::printf("fit_image: psnr %.2f dB after %d iterations\n", r.report.final_psnr, cfg.iters);
        CHECK(r.report.final_psnr > 35.0);
        bool threw = false;
        try {
            fit_image(target, g, 0, cfg);
        } catch (const invalid_parameter&) {
            threw = true;
        }
        CHECK(threw);
    }
    std::printf("host fit ok\n");
    return 0;
}
