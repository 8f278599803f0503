// darbs_b200.hpp — C++ mirror of the reference's rasterizer entry points over the C ABI.
//
// Same names, argument meaning and error behaviour as the reference's
//   include/darbs/kernel.hpp:20-72      KernelSpec, make_kernel, kernel_preset
//   include/darbs/geometry.hpp:45-53    Conic, ProjectedSplat
//   include/darbs/image.hpp:9-20        ImageBuffer
//   include/darbs/rasterizer.hpp:16-68  TileBins, BlendAux, ForwardResult, SplatGrads,
//                                       bin_splats, forward, backward
//   include/darbs/errors.hpp:10-36      invalid_parameter, numeric_error, contract_violation
// so that a caller of darbs::forward / darbs::backward (fit2d.cpp:115,126, fit3d.cpp:120,133,
// benchmarks/bench.cpp:62,73) compiles against this header unchanged (define
// DARBS_B200_AS_DARBS to get `namespace darbs`).  Everything here only marshals AoS FP64
// values into the SoA float32 arrays of include/darbs_cuda.h and back; the work happens in
// libdarbs_cuda.so on the GPU.  There is no CPU path.
//
// Differences from the reference, by construction of the boundary:
//  * element type on the device is float32;
//  * Eigen is not required: Vec2 / Vec3 / Mat2 are minimal PODs with the members the
//    rasterizer interface uses (x(), y(), operator[], operator(), Zero(), Ones(), Identity());
//  * BlendAux keeps the per-pixel vectors by value like the reference, but the bins stay on the
//    device: `aux.bins` is filled only when Session::keep_bins is set.  backward() accepts any
//    aux: if it is not the one of the session's last forward, the forward is replayed first.
//  * `threads` is accepted and ignored.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "darbs_cuda.h"

namespace darbs_b200 {

// ---- errors (include/darbs/errors.hpp:10-36)
struct invalid_parameter : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct numeric_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct contract_violation : std::logic_error {
    using std::logic_error::logic_error;
};
struct io_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct cuda_error : std::runtime_error {  // no reference analogue
    using std::runtime_error::runtime_error;
};

inline void throw_status(darbs_status st, const darbs_cuda_ctx* ctx) {
    const std::string msg = darbs_cuda_last_error(ctx);
    switch (st) {
        case DARBS_OK: return;
        case DARBS_INVALID_PARAMETER: throw invalid_parameter(msg);
        case DARBS_NUMERIC_ERROR: throw numeric_error(msg);
        case DARBS_IO_ERROR: throw io_error(msg);
        case DARBS_CONTRACT_VIOLATION: throw contract_violation(msg);
        default: throw cuda_error(msg);
    }
}

// ---- small value types
struct Vec2 {
    double v[2] = {0.0, 0.0};
    Vec2() = default;
    Vec2(double a, double b) : v{a, b} {}
    double& x() { return v[0]; }
    double& y() { return v[1]; }
    double x() const { return v[0]; }
    double y() const { return v[1]; }
    double& operator[](int i) { return v[i]; }
    double operator[](int i) const { return v[i]; }
    static Vec2 Zero() { return Vec2(); }
    static Vec2 Ones() { return Vec2(1.0, 1.0); }
};
struct Vec3 {
    double v[3] = {0.0, 0.0, 0.0};
    Vec3() = default;
    Vec3(double a, double b, double c) : v{a, b, c} {}
    double& operator[](int i) { return v[i]; }
    double operator[](int i) const { return v[i]; }
    static Vec3 Zero() { return Vec3(); }
    static Vec3 Ones() { return Vec3(1.0, 1.0, 1.0); }
};
struct Mat2 {
    double m[2][2] = {{1.0, 0.0}, {0.0, 1.0}};
    double& operator()(int r, int c) { return m[r][c]; }
    double operator()(int r, int c) const { return m[r][c]; }
    static Mat2 Identity() { return Mat2(); }
};

// ---- kernel family (include/darbs/kernel.hpp:12-33)
enum class KernelFamily { Gaussian, HalfCosine, RaisedCosine, ModulusSinc, InverseMultiquadratic };

struct KernelSpec {
    KernelFamily family = KernelFamily::Gaussian;
    double beta = 2.0;
    double xi = 2.0;
    int lobes = 1;
    double cutoff = 9.0;
    bool unbounded = true;
};

inline darbs_kernel_spec to_abi(const KernelSpec& k) {
    darbs_kernel_spec s;
    s.family = (int32_t)k.family;
    s.beta = k.beta;
    s.xi = k.xi;
    s.lobes = k.lobes;
    s.cutoff = k.cutoff;
    s.unbounded = k.unbounded ? 1 : 0;
    return s;
}
inline KernelSpec from_abi(const darbs_kernel_spec& s) {
    KernelSpec k;
    k.family = (KernelFamily)s.family;
    k.beta = s.beta;
    k.xi = s.xi;
    k.lobes = s.lobes;
    k.cutoff = s.cutoff;
    k.unbounded = s.unbounded != 0;
    return k;
}
inline KernelSpec make_kernel(KernelFamily family, double beta, double xi, int lobes = 1) {
    darbs_kernel_spec s;
    throw_status(darbs_cuda_make_kernel((int)family, beta, xi, lobes, &s), nullptr);
    return from_abi(s);
}
// kernel_preset, kernel.hpp:71 / kernel.cpp:223-240: empty for an unknown name
inline std::optional<KernelSpec> kernel_preset(const std::string& name) {
    darbs_kernel_spec s;
    if (darbs_cuda_kernel_preset(name.c_str(), &s) != DARBS_OK) return std::nullopt;
    return from_abi(s);
}
inline double cutoff_dm2(const KernelSpec& k) { return k.cutoff; }
inline const char* family_name(KernelFamily f) {  // kernel.cpp:242-256
    switch (f) {
        case KernelFamily::Gaussian: return "gaussian";
        case KernelFamily::HalfCosine: return "half-cosine";
        case KernelFamily::RaisedCosine: return "raised-cosine";
        case KernelFamily::ModulusSinc: return "modulus-sinc";
        default: return "inverse-multiquadratic";
    }
}
struct KernelSample {  // kernel.hpp:34-38
    double dm2 = 0.0, weight = 0.0, dweight_ddm2 = 0.0;
};

// ---- geometry / image value types
struct Conic {
    double a = 1.0, b = 0.0, c = 1.0;
};
struct ProjectedSplat {
    Vec2 mu2 = Vec2::Zero();
    Mat2 cov2 = Mat2::Identity();
    Conic conic;
    double radius = 0.0;
    double depth = 0.0;
    double opacity = 1.0;
    Vec3 color = Vec3::Ones();
};
struct ImageBuffer {
    int width = 0;
    int height = 0;
    std::vector<double> rgb;
    ImageBuffer() = default;
    ImageBuffer(int w, int h, double fill = 0.0) : width(w), height(h), rgb(std::size_t(w) * h * 3, fill) {}
    double& at(int x, int y, int c) { return rgb[(std::size_t(y) * width + x) * 3 + c]; }
    double at(int x, int y, int c) const { return rgb[(std::size_t(y) * width + x) * 3 + c]; }
};

// ---- rasterizer (include/darbs/rasterizer.hpp:11-68)
inline constexpr int kTileSize = DARBS_TILE_SIZE;
inline constexpr double kAlphaClamp = DARBS_ALPHA_CLAMP;
inline constexpr double kAlphaSkip = DARBS_ALPHA_SKIP;
inline constexpr double kTransmittanceFloor = DARBS_TRANSMITTANCE_FLOOR;

struct TileBins {
    int tiles_x = 0;
    int tiles_y = 0;
    std::vector<std::vector<int>> lists;
};
struct BlendAux {
    int width = 0;
    int height = 0;
    std::size_t splat_count = 0;
    Vec3 background = Vec3::Zero();
    TileBins bins;
    std::vector<double> t_final;
    std::vector<int> processed;
    std::vector<int> contributors;
    int skipped_nonfinite = 0;
    std::uint64_t generation = 0;  // which forward of the session left this aux resident
};
struct ForwardResult {
    ImageBuffer image;
    BlendAux aux;
};
struct SplatGrads {
    Vec3 d_color = Vec3::Zero();
    double d_opacity = 0.0;
    double d_conic_a = 0.0;
    double d_conic_b = 0.0;
    double d_conic_c = 0.0;
    Vec2 d_mu2 = Vec2::Zero();
};

// One GPU context plus the staging vectors of the AoS <-> SoA conversion.
class Session {
public:
    explicit Session(int device = 0) { throw_status(darbs_cuda_create(device, &ctx_), nullptr); }
    ~Session() { darbs_cuda_destroy(ctx_); }
    Session(const Session&) = delete;
    Session& operator=(const Session&) = delete;

    bool keep_bins = false;
    darbs_cuda_ctx* handle() { return ctx_; }

    TileBins bin_splats(const std::vector<ProjectedSplat>& splats, int width, int height, int tile = kTileSize) {
        if (tile != kTileSize) throw invalid_parameter("bin_splats: only the reference's tile size 16 is built");
        pack(splats);
        TileBins bins;
        bins.tiles_x = (width + kTileSize - 1) / kTileSize;
        bins.tiles_y = (height + kTileSize - 1) / kTileSize;
        const std::size_t tiles = std::size_t(bins.tiles_x) * bins.tiles_y;
        int64_t k = 0;
        check(darbs_cuda_bin(ctx_, n_, mu2_.data(), conic_.data(), radius_.data(), depth_.data(), width, height, &k,
                             nullptr, nullptr, nullptr, nullptr, 0, DARBS_HOST));
        std::vector<int32_t> ranges(2 * tiles), plist((std::size_t)k);
        check(darbs_cuda_bin(ctx_, n_, mu2_.data(), conic_.data(), radius_.data(), depth_.data(), width, height, &k,
                             ranges.data(), plist.data(), nullptr, nullptr, k, DARBS_HOST));
        bins.lists.resize(tiles);
        for (std::size_t t = 0; t < tiles; ++t)
            bins.lists[t].assign(plist.begin() + ranges[2 * t], plist.begin() + ranges[2 * t + 1]);
        ++generation_;  // binning overwrites the resident forward state
        return bins;
    }

    ForwardResult forward(const std::vector<ProjectedSplat>& splats, const KernelSpec& kernel, int width,
                          int height, const Vec3& background, int /*threads*/ = 1) {
        ForwardResult r;
        if (keep_bins) r.aux.bins = bin_splats(splats, width, height);
        pack(splats);
        const std::size_t px = std::size_t(width) * height;
        image_.resize(3 * px);
        t_final_.resize(px);
        r.aux.processed.resize(px);
        r.aux.contributors.resize(px);
        const float bg[3] = {(float)background[0], (float)background[1], (float)background[2]};
        const darbs_kernel_spec ks = to_abi(kernel);
        int32_t skipped = 0;
        check(darbs_cuda_forward(ctx_, &ks, n_, mu2_.data(), conic_.data(), radius_.data(), depth_.data(),
                                 opacity_.data(), rgb_.data(), width, height, bg, image_.data(), t_final_.data(),
                                 r.aux.processed.data(), r.aux.contributors.data(), &skipped, DARBS_HOST));
        r.image = ImageBuffer(width, height);
        r.image.rgb.assign(image_.begin(), image_.end());
        r.aux.t_final.assign(t_final_.begin(), t_final_.end());
        r.aux.width = width;
        r.aux.height = height;
        r.aux.splat_count = splats.size();
        r.aux.background = background;
        r.aux.skipped_nonfinite = skipped;
        r.aux.generation = ++generation_;
        return r;
    }

    std::vector<SplatGrads> backward(const ImageBuffer& grad_image, const std::vector<ProjectedSplat>& splats,
                                     const KernelSpec& kernel, const BlendAux& aux, int /*threads*/ = 1) {
        // rasterizer.cpp:151-154
        if (grad_image.width != aux.width || grad_image.height != aux.height || splats.size() != aux.splat_count)
            throw contract_violation("backward: aux does not match this forward call");
        if (aux.generation != generation_) forward(splats, kernel, aux.width, aux.height, aux.background);
        std::vector<float> g(grad_image.rgb.begin(), grad_image.rgb.end());
        std::vector<float> out(std::size_t(DARBS_GRADS_PER_SPLAT) * splats.size());
        const darbs_kernel_spec ks = to_abi(kernel);
        check(darbs_cuda_backward(ctx_, &ks, grad_image.width, grad_image.height, g.data(), (int64_t)splats.size(),
                                  nullptr, nullptr, nullptr, nullptr, out.data(), DARBS_HOST));
        std::vector<SplatGrads> grads(splats.size());
        for (std::size_t i = 0; i < splats.size(); ++i) {
            const float* o = out.data() + DARBS_GRADS_PER_SPLAT * i;
            grads[i].d_color = Vec3(o[0], o[1], o[2]);
            grads[i].d_opacity = o[3];
            grads[i].d_conic_a = o[4];
            grads[i].d_conic_b = o[5];
            grads[i].d_conic_c = o[6];
            grads[i].d_mu2 = Vec2(o[7], o[8]);
        }
        return grads;
    }

private:
    void check(darbs_status st) { throw_status(st, ctx_); }
    void pack(const std::vector<ProjectedSplat>& s) {
        n_ = (int64_t)s.size();
        mu2_.resize(2 * s.size());
        conic_.resize(3 * s.size());
        radius_.resize(s.size());
        depth_.resize(s.size());
        opacity_.resize(s.size());
        rgb_.resize(3 * s.size());
        for (std::size_t i = 0; i < s.size(); ++i) {
            mu2_[2 * i] = (float)s[i].mu2.x();
            mu2_[2 * i + 1] = (float)s[i].mu2.y();
            conic_[3 * i] = (float)s[i].conic.a;
            conic_[3 * i + 1] = (float)s[i].conic.b;
            conic_[3 * i + 2] = (float)s[i].conic.c;
            radius_[i] = (float)s[i].radius;
            depth_[i] = (float)s[i].depth;
            opacity_[i] = (float)s[i].opacity;
            for (int c = 0; c < 3; ++c) rgb_[3 * i + c] = (float)s[i].color[c];
        }
    }
    darbs_cuda_ctx* ctx_ = nullptr;
    std::uint64_t generation_ = 0;
    int64_t n_ = 0;
    std::vector<float> mu2_, conic_, radius_, depth_, opacity_, rgb_, image_, t_final_;
};

inline Session& default_session() {
    thread_local Session s(0);
    return s;
}

// eval, kernel.hpp:47 / kernel.cpp:127-164, on the device functors (FP64 path of the library)
inline KernelSample eval(const KernelSpec& spec, double dm2) {
    darbs_cuda_ctx* ctx = default_session().handle();
    const darbs_kernel_spec ks = to_abi(spec);
    const float x = (float)dm2;
    float w = 0.f, dw = 0.f;
    throw_status(darbs_cuda_eval(ctx, &ks, 1, &x, &w, &dw, 1, DARBS_HOST), ctx);
    return KernelSample{dm2, w, dw};
}

// The reference's free functions (include/darbs/rasterizer.hpp:24-25, :45-46, :65-68).
inline TileBins bin_splats(const std::vector<ProjectedSplat>& splats, int width, int height, int tile = kTileSize) {
    return default_session().bin_splats(splats, width, height, tile);
}
inline ForwardResult forward(const std::vector<ProjectedSplat>& splats, const KernelSpec& kernel, int width,
                             int height, const Vec3& background, int threads = 1) {
    return default_session().forward(splats, kernel, width, height, background, threads);
}
inline std::vector<SplatGrads> backward(const ImageBuffer& grad_image, const std::vector<ProjectedSplat>& splats,
                                        const KernelSpec& kernel, const BlendAux& aux, int threads = 1) {
    return default_session().backward(grad_image, splats, kernel, aux, threads);
}

}  // namespace darbs_b200

#ifdef DARBS_B200_AS_DARBS
namespace darbs = darbs_b200;
#endif
