// test_host.cpp — drives the C++ mirror (darbs_b200.hpp) the way the reference's own tests drive
// darbs::forward / darbs::backward (tests/test_rasterizer.cpp).  Needs a B200; run by
// tests/test_gpu_host_mirror.py.  Prints "host mirror ok" and exits 0 when every check holds.
#define DARBS_B200_AS_DARBS
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "darbs_b200.hpp"

using namespace darbs;

#define CHECK(cond)                                                        \
    do {                                                                   \
        if (!(cond)) {                                                     \
            std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #cond); \
            std::exit(1);                                                  \
        }                                                                  \
    } while (0)

// make_splat of the reference's fixtures for an isotropic covariance s * I
static ProjectedSplat iso_splat(Vec2 mu, double s, double depth, double opacity, Vec3 color, const KernelSpec& k) {
    ProjectedSplat p;
    p.mu2 = mu;
    p.cov2(0, 0) = p.cov2(1, 1) = s;
    p.conic.a = p.conic.c = 1.0 / s;
    p.conic.b = 0.0;
    p.radius = std::ceil(std::sqrt(k.cutoff) * std::sqrt(s));  // geometry.cpp:62
    p.depth = depth;
    p.opacity = opacity;
    p.color = color;
    return p;
}

int main() {
    const KernelSpec g = *kernel_preset("gaussian");
    CHECK(!kernel_preset("no-such-kernel"));
    CHECK(g.unbounded && std::fabs(cutoff_dm2(g) - 9.0) < 1e-12);
    // kernel.cpp:43-51
    bool threw = false;
    try {
        make_kernel(KernelFamily::Gaussian, -1.0, 1.0);
    } catch (const invalid_parameter&) {
        threw = true;
    }
    CHECK(threw);

    // empty scene returns the background (test_rasterizer.cpp:98-102)
    {
        ForwardResult r = forward({}, g, 8, 8, Vec3(0.2, 0.2, 0.2));
        for (double v : r.image.rgb) CHECK(std::fabs(v - 0.2) < 1e-6);
        for (double t : r.aux.t_final) CHECK(t == 1.0);
    }
    // opaque splat saturates at the alpha clamp (:103-111)
    {
        auto s = iso_splat(Vec2(4.5, 4.5), 1.0, 1.0, 1.0, Vec3(1, 0, 0), g);
        ForwardResult r = forward({s}, g, 8, 8, Vec3::Zero());
        CHECK(std::fabs(r.image.at(4, 4, 0) - 0.99) < 1e-6);
        CHECK(std::fabs(r.image.at(4, 4, 1)) < 1e-6);
        CHECK(std::fabs(r.aux.t_final[4 * 8 + 4] - 0.01) < 1e-6);
    }
    // single splat closed-form blend over the background (:112-130), float32 tolerance
    {
        auto s = iso_splat(Vec2(4.5, 4.5), 4.0, 1.0, 0.6, Vec3(0.3, 0.9, 0.1), g);
        Vec3 bg(0.2, 0.1, 0.4);
        ForwardResult r = forward({s}, g, 8, 8, bg);
        for (int y = 0; y < 8; ++y)
            for (int x = 0; x < 8; ++x) {
                double dm2 = ((x - 4.0) * (x - 4.0) + (y - 4.0) * (y - 4.0)) / 4.0;
                double w = dm2 > g.cutoff ? 0.0 : std::exp(-dm2 / 2.0);
                double alpha = std::min(0.99, 0.6 * w);
                if (alpha < 1.0 / 255.0) alpha = 0.0;
                for (int c = 0; c < 3; ++c)
                    CHECK(std::fabs(r.image.at(x, y, c) - (s.color[c] * alpha + bg[c] * (1.0 - alpha))) < 2e-6);
            }
    }
    // binning membership and ordering (:59-94)
    {
        std::vector<ProjectedSplat> splats;
        splats.push_back(iso_splat(Vec2(8, 8), 0.4, 1.0, 0.9, Vec3::Ones(), g));
        TileBins bins = bin_splats(splats, 32, 32);
        CHECK(bins.tiles_x == 2 && bins.tiles_y == 2);
        CHECK(bins.lists[0].size() == 1 && bins.lists[1].empty() && bins.lists[2].empty() && bins.lists[3].empty());
        splats.push_back(iso_splat(Vec2(16, 16), 400.0, 0.5, 0.9, Vec3::Ones(), g));
        bins = bin_splats(splats, 32, 32);
        for (const auto& l : bins.lists) CHECK(!l.empty() && l.front() == 1);
        CHECK(bins.lists[0].back() == 0);
    }
    // a random scene: backward contract, zero upstream, stale aux replay, linearity
    {
        std::mt19937_64 rng(3);
        std::uniform_real_distribution<double> u(0.0, 1.0);
        const KernelSpec k = *kernel_preset("half-cosine-sq");
        std::vector<ProjectedSplat> splats;
        for (int i = 0; i < 300; ++i)
            splats.push_back(iso_splat(Vec2(64 * u(rng), 48 * u(rng)), 1.0 + 6.0 * u(rng), 0.5 + 9.0 * u(rng),
                                       0.1 + 0.85 * u(rng), Vec3(u(rng), u(rng), u(rng)), k));
        ForwardResult r = forward(splats, k, 64, 48, Vec3(0.1, 0.2, 0.3));
        long visits = 0;
        for (int p : r.aux.processed) visits += p;
        CHECK(visits > 0);
        threw = false;
        try {
            backward(ImageBuffer(32, 48), splats, k, r.aux);
        } catch (const contract_violation&) {
            threw = true;
        }
        CHECK(threw);  // test_rasterizer.cpp:176-185
        auto zero = backward(ImageBuffer(64, 48, 0.0), splats, k, r.aux);
        for (const auto& z : zero) CHECK(z.d_opacity == 0.0 && z.d_mu2.x() == 0.0 && z.d_color[0] == 0.0);  // :187-197
        ImageBuffer g1(64, 48);
        for (double& v : g1.rgb) v = 2.0 * u(rng) - 1.0;
        auto a = backward(g1, splats, k, r.aux);
        // another forward in between: the old aux must still work (value semantics of the reference)
        forward({splats[0]}, k, 16, 16, Vec3::Zero());
        auto b = backward(g1, splats, k, r.aux);
        double worst = 0.0, scale = 0.0;
        for (std::size_t i = 0; i < a.size(); ++i) {
            worst = std::max(worst, std::fabs(a[i].d_opacity - b[i].d_opacity));
            scale = std::max(scale, std::fabs(a[i].d_opacity));
        }
        CHECK(scale > 0.0 && worst <= 1e-5 * scale);
    }
    std::printf("host mirror ok\n");
    return 0;
}
