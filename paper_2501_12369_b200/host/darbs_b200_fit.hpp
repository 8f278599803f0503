// darbs_b200_fit.hpp — C++ mirror of the callers and data formats either side of the rasterizer
// hot path, over the C ABI (include/darbs_cuda.h).  Same names, argument meaning and error
// behaviour as the reference's
//   include/darbs/geometry.hpp:23-97    Primitive3D, Camera, ConicRadius, conic_and_radius,
//                                       project_primitive, ProjectionGrads, backward_projection
//   include/darbs/loss.hpp:7-22         LossResult, ssim, loss_total
//   include/darbs/optim.hpp:12-45       AdamState, adam_step
//   include/darbs/fit_common.hpp:15-42  FitConfig, FitReport, sigmoid, logit
//   include/darbs/fit3d.hpp:11-33       render_scene, View, Fit3DResult, fit_scene
//   include/darbs/fit2d.hpp:12-36       Splat2DParams, realize_splat2d, Fit2DResult, fit_image
//   include/darbs/scene_io.hpp:10-22    read_scene, write_scene, read_cameras, write_cameras
//   include/darbs/image.hpp:22-34       write_ppm, read_ppm, write_float_dump, read_float_dump, mse, psnr
//
// fit_scene is the device-resident training loop: raw parameters, Adam state, learning rates,
// gradients and every view's target stay on the GPU; one darbs_cuda_evaluate_view per view and
// one darbs_cuda_adam_step per iteration (src/fit3d.cpp:104-184).  fit_image is the reference's
// desk-scale 2-D experiment (src/fit2d.cpp:45-188): its nine-parameter chain runs on the host in
// double exactly as the reference writes it, and calls forward / loss_total / backward /
// adam_step of this mirror.  The file formats are byte-compatible with the reference's writers.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <limits>
#include <optional>
#include <random>
#include <sstream>

#include "darbs_b200.hpp"

namespace darbs_b200 {

// ---- geometry value types (include/darbs/geometry.hpp:23-43)
struct Quat {
    double q[4] = {1.0, 0.0, 0.0, 0.0};  // w, x, y, z
    Quat() = default;
    Quat(double w, double x, double y, double z) : q{w, x, y, z} {}
    double w() const { return q[0]; }
    double x() const { return q[1]; }
    double y() const { return q[2]; }
    double z() const { return q[3]; }
};
struct Vec4 {
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    double& operator[](int i) { return v[i]; }
    double operator[](int i) const { return v[i]; }
};
struct Primitive3D {
    Vec3 mu = Vec3::Zero();
    Vec3 scale = Vec3::Ones();
    Quat rot;
    double opacity = 1.0;
    Vec3 color = Vec3::Ones();
};
struct Camera {
    double w[4][4] = {{1, 0, 0, 0}, {0, 1, 0, 0}, {0, 0, 1, 0}, {0, 0, 0, 1}};  // world-to-camera
    double fx = 1.0, fy = 1.0, cx = 0.0, cy = 0.0;
    int width = 0, height = 0;
};
inline constexpr double kNearPlane = DARBS_NEAR_PLANE;
inline constexpr double kDilation = DARBS_DILATION;

// the 22-double camera block of the ABI (and of the camera file, scene_io.hpp:16-19)
inline std::array<double, DARBS_CAMERA_DOUBLES> camera_block(const Camera& cam) {
    std::array<double, DARBS_CAMERA_DOUBLES> b{};
    b[0] = cam.fx;
    b[1] = cam.fy;
    b[2] = cam.cx;
    b[3] = cam.cy;
    b[4] = cam.width;
    b[5] = cam.height;
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) b[6 + 4 * r + c] = cam.w[r][c];
    return b;
}

struct ConicRadius {
    Conic conic;
    double lambda1 = 0.0, lambda2 = 0.0, radius = 0.0;
};

// conic_and_radius, src/geometry.cpp:50-64 (host arithmetic: three divisions and a ceil)
inline ConicRadius conic_and_radius(const Mat2& cov2, const KernelSpec& kernel) {
    const double a = cov2(0, 0), b = cov2(0, 1), c = cov2(1, 1);
    const double det = a * c - b * b;
    if (!(det > 0.0) || !(a > 0.0)) throw numeric_error("conic_and_radius: covariance not positive definite");
    const double mid = 0.5 * (a + c);
    const double disc = std::sqrt(std::max(0.0, mid * mid - det));
    ConicRadius out;
    out.lambda1 = mid + disc;
    out.lambda2 = mid - disc;
    out.conic = Conic{c / det, -b / det, a / det};
    out.radius = std::ceil(std::sqrt(cutoff_dm2(kernel)) * std::sqrt(out.lambda1));
    return out;
}

inline void primitive_to_floats(const Primitive3D& p, float* o) {
    for (int k = 0; k < 3; ++k) o[k] = (float)p.mu[k];
    for (int k = 0; k < 3; ++k) o[3 + k] = (float)p.scale[k];
    for (int k = 0; k < 4; ++k) o[6 + k] = (float)p.rot.q[k];
    o[10] = (float)p.opacity;
    for (int k = 0; k < 3; ++k) o[11 + k] = (float)p.color[k];
}

// project_primitive, src/geometry.cpp:66-87: empty when culled by the near plane.
inline std::optional<ProjectedSplat> project_primitive(const Primitive3D& prim, const Camera& cam,
                                                       const KernelSpec& kernel, double psi,
                                                       double dilation = kDilation) {
    darbs_cuda_ctx* ctx = default_session().handle();
    float p[14], mu2[2], cov2[3], conic[3], radius, depth;
    int32_t valid = 0;
    primitive_to_floats(prim, p);
    const darbs_kernel_spec ks = to_abi(kernel);
    const auto block = camera_block(cam);
    throw_status(darbs_cuda_project(ctx, &ks, psi, dilation, 1, p, block.data(), &valid, mu2, cov2, conic, &radius,
                                    &depth, DARBS_HOST),
                 ctx);
    if (!valid) return std::nullopt;
    ProjectedSplat s;
    s.mu2 = Vec2(mu2[0], mu2[1]);
    s.cov2(0, 0) = cov2[0];
    s.cov2(0, 1) = s.cov2(1, 0) = cov2[1];
    s.cov2(1, 1) = cov2[2];
    s.conic = Conic{conic[0], conic[1], conic[2]};
    s.radius = radius;
    s.depth = depth;
    s.opacity = prim.opacity;
    s.color = prim.color;
    return s;
}

struct ProjectionGrads {
    Vec3 d_mu = Vec3::Zero();
    Vec3 d_scale = Vec3::Zero();
    Vec4 d_rot;  // w, x, y, z of the raw quaternion
};

// backward_projection, src/geometry.cpp:111-168
inline ProjectionGrads backward_projection(const Mat2& grad_cov2, const Vec2& grad_mu2, const Primitive3D& prim,
                                           const Camera& cam, double psi) {
    darbs_cuda_ctx* ctx = default_session().handle();
    float p[14], gc[4] = {(float)grad_cov2(0, 0), (float)grad_cov2(0, 1), (float)grad_cov2(1, 0),
                          (float)grad_cov2(1, 1)};
    float gm[2] = {(float)grad_mu2.x(), (float)grad_mu2.y()}, d_mu[3], d_scale[3], d_rot[4];
    primitive_to_floats(prim, p);
    const auto block = camera_block(cam);
    throw_status(darbs_cuda_backward_projection(ctx, psi, 1, gc, gm, p, block.data(), d_mu, d_scale, d_rot,
                                                DARBS_HOST),
                 ctx);
    ProjectionGrads g;
    for (int k = 0; k < 3; ++k) g.d_mu[k] = d_mu[k];
    for (int k = 0; k < 3; ++k) g.d_scale[k] = d_scale[k];
    for (int k = 0; k < 4; ++k) g.d_rot[k] = d_rot[k];
    return g;
}

// ---- loss (include/darbs/loss.hpp:7-22)
struct LossResult {
    double total = 0.0, l1 = 0.0, dssim = 0.0;
    ImageBuffer grad;
};

inline LossResult loss_total(const ImageBuffer& rendered, const ImageBuffer& target, double lambda) {
    if (rendered.width != target.width || rendered.height != target.height)
        throw invalid_parameter("loss_total: dimension mismatch");  // loss.cpp:174-176
    darbs_cuda_ctx* ctx = default_session().handle();
    const std::vector<float> x(rendered.rgb.begin(), rendered.rgb.end()), y(target.rgb.begin(), target.rgb.end());
    std::vector<float> g(x.size());
    double out[4];
    throw_status(darbs_cuda_loss_total(ctx, rendered.width, rendered.height, x.data(), y.data(), lambda, out,
                                       g.data(), DARBS_HOST),
                 ctx);
    LossResult r;
    r.total = out[0];
    r.l1 = out[1];
    r.dssim = out[2];
    r.grad = ImageBuffer(rendered.width, rendered.height);
    r.grad.rgb.assign(g.begin(), g.end());
    return r;
}

// ssim, src/loss.cpp:142-171: the mean SSIM is 1 - 2 dssim of the same pair (loss.cpp:226-227)
inline double ssim(const ImageBuffer& a, const ImageBuffer& b) {
    if (a.width != b.width || a.height != b.height) throw invalid_parameter("ssim: dimension mismatch");
    darbs_cuda_ctx* ctx = default_session().handle();
    const std::vector<float> x(a.rgb.begin(), a.rgb.end()), y(b.rgb.begin(), b.rgb.end());
    double out[4];
    throw_status(darbs_cuda_loss_total(ctx, a.width, a.height, x.data(), y.data(), 1.0, out, nullptr, DARBS_HOST),
                 ctx);
    return 1.0 - 2.0 * out[2];
}

// ---- images (include/darbs/image.hpp:22-34; src/image.cpp)
inline double mse(const ImageBuffer& a, const ImageBuffer& b) {
    if (a.width != b.width || a.height != b.height) throw invalid_parameter("mse: dimension mismatch");
    double acc = 0.0;
    for (std::size_t i = 0; i < a.rgb.size(); ++i) acc += (a.rgb[i] - b.rgb[i]) * (a.rgb[i] - b.rgb[i]);
    return acc / double(a.rgb.size());
}
inline double psnr(const ImageBuffer& a, const ImageBuffer& b) {
    const double m = mse(a, b);
    return m <= 0.0 ? std::numeric_limits<double>::infinity() : -10.0 * std::log10(m);
}

namespace detail {
inline void put_u32(std::ostream& os, std::uint32_t v) {
    const unsigned char b[4] = {(unsigned char)(v & 0xff), (unsigned char)((v >> 8) & 0xff),
                                (unsigned char)((v >> 16) & 0xff), (unsigned char)((v >> 24) & 0xff)};
    os.write(reinterpret_cast<const char*>(b), 4);
}
inline std::uint32_t get_u32(std::istream& is) {
    unsigned char b[4] = {0, 0, 0, 0};
    is.read(reinterpret_cast<char*>(b), 4);
    return std::uint32_t(b[0]) | (std::uint32_t(b[1]) << 8) | (std::uint32_t(b[2]) << 16) | (std::uint32_t(b[3]) << 24);
}
// numbers of one text line, '#' comments stripped; false on a malformed token
inline bool line_numbers(std::string line, std::vector<double>& out) {
    if (auto pos = line.find('#'); pos != std::string::npos) line.erase(pos);
    std::istringstream ss(line);
    double v;
    while (ss >> v) out.push_back(v);
    return ss.eof();
}
}  // namespace detail

// "DSFL" + width + height + channel count (u32 LE each) + float32 LE pixels (image.hpp:25-28)
inline void write_float_dump(const ImageBuffer& img, const std::string& path) {
    std::ofstream os(path, std::ios::binary);
    if (!os) throw io_error("write_float_dump: cannot open " + path);
    os.write("DSFL", 4);
    detail::put_u32(os, (std::uint32_t)img.width);
    detail::put_u32(os, (std::uint32_t)img.height);
    detail::put_u32(os, 3);
    for (double v : img.rgb) {
        const float f = (float)v;
        std::uint32_t bits;
        std::memcpy(&bits, &f, 4);
        detail::put_u32(os, bits);
    }
    if (!os) throw io_error("write_float_dump: write failed for " + path);
}
inline ImageBuffer read_float_dump(const std::string& path) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw io_error("read_float_dump: cannot open " + path);
    char magic[4] = {0, 0, 0, 0};
    is.read(magic, 4);
    if (!is || std::memcmp(magic, "DSFL", 4) != 0) throw io_error("read_float_dump: bad magic in " + path);
    const std::uint32_t w = detail::get_u32(is), h = detail::get_u32(is), ch = detail::get_u32(is);
    if (ch != 3) throw io_error("read_float_dump: expected 3 channels");
    ImageBuffer img((int)w, (int)h);
    for (double& v : img.rgb) {
        const std::uint32_t bits = detail::get_u32(is);
        float f;
        std::memcpy(&f, &bits, 4);
        v = f;
    }
    if (!is) throw io_error("read_float_dump: truncated file " + path);
    return img;
}
// binary PPM, maxval 255, channels clamped and rounded half-up (image.hpp:22-23)
inline void write_ppm(const ImageBuffer& img, const std::string& path) {
    std::ofstream os(path, std::ios::binary);
    if (!os) throw io_error("write_ppm: cannot open " + path);
    os << "P6\n" << img.width << " " << img.height << "\n255\n";
    std::vector<unsigned char> bytes(img.rgb.size());
    for (std::size_t i = 0; i < bytes.size(); ++i)
        bytes[i] = (unsigned char)std::floor(std::clamp(img.rgb[i], 0.0, 1.0) * 255.0 + 0.5);
    os.write(reinterpret_cast<const char*>(bytes.data()), (std::streamsize)bytes.size());
    if (!os) throw io_error("write_ppm: write failed for " + path);
}
inline ImageBuffer read_ppm(const std::string& path) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw io_error("read_ppm: cannot open " + path);
    std::string magic;
    int w = 0, h = 0, maxval = 0;
    is >> magic >> w >> h >> maxval;
    if (magic != "P6" || w <= 0 || h <= 0 || maxval != 255) throw io_error("read_ppm: unsupported PPM " + path);
    is.get();
    ImageBuffer img(w, h);
    std::vector<unsigned char> bytes(img.rgb.size());
    is.read(reinterpret_cast<char*>(bytes.data()), (std::streamsize)bytes.size());
    if (!is) throw io_error("read_ppm: truncated file " + path);
    for (std::size_t i = 0; i < bytes.size(); ++i) img.rgb[i] = bytes[i] / 255.0;
    return img;
}

// ---- scene and camera text files (include/darbs/scene_io.hpp:10-22; src/scene_io.cpp)
inline std::vector<Primitive3D> read_scene(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw io_error("cannot open scene file " + path);
    std::vector<Primitive3D> prims;
    std::string line;
    for (int lineno = 1; std::getline(in, line); ++lineno) {
        std::vector<double> v;
        detail::line_numbers(line, v);
        if (v.empty()) continue;
        const std::string where = path + ":" + std::to_string(lineno);
        if (v.size() != 14)
            throw io_error(where + ": expected 14 fields per primitive, got " + std::to_string(v.size()));
        Primitive3D p;
        p.mu = Vec3(v[0], v[1], v[2]);
        p.scale = Vec3(v[3], v[4], v[5]);
        p.rot = Quat(v[6], v[7], v[8], v[9]);
        p.opacity = v[10];
        p.color = Vec3(v[11], v[12], v[13]);
        if (std::min({v[3], v[4], v[5]}) <= 0.0) throw io_error(where + ": non-positive scale");
        if (p.opacity < 0.0 || p.opacity > 1.0) throw io_error(where + ": opacity outside [0,1]");
        prims.push_back(p);
    }
    return prims;
}
inline void write_scene(const std::vector<Primitive3D>& prims, const std::string& path) {
    std::ofstream out(path);
    if (!out) throw io_error("cannot write scene file " + path);
    out << std::setprecision(17);
    for (const Primitive3D& p : prims) {
        const double f[14] = {p.mu[0],    p.mu[1],    p.mu[2],    p.scale[0], p.scale[1], p.scale[2], p.rot.w(),
                              p.rot.x(),  p.rot.y(),  p.rot.z(),  p.opacity,  p.color[0], p.color[1], p.color[2]};
        for (int k = 0; k < 14; ++k) out << f[k] << (k == 13 ? '\n' : ' ');
    }
    if (!out) throw io_error("write failed for " + path);
}
inline std::vector<Camera> read_cameras(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw io_error("cannot open " + path);
    std::vector<double> nums;
    std::string line;
    while (std::getline(in, line))
        if (!detail::line_numbers(line, nums)) throw io_error(path + ": malformed number in line '" + line + "'");
    if (nums.empty() || nums.size() % DARBS_CAMERA_DOUBLES != 0)
        throw io_error(path + ": camera file must hold blocks of 22 numbers, got " + std::to_string(nums.size()));
    std::vector<Camera> cams;
    for (std::size_t off = 0; off < nums.size(); off += DARBS_CAMERA_DOUBLES) {
        Camera cam;
        cam.fx = nums[off];
        cam.fy = nums[off + 1];
        cam.cx = nums[off + 2];
        cam.cy = nums[off + 3];
        cam.width = int(nums[off + 4]);
        cam.height = int(nums[off + 5]);
        if (cam.fx <= 0 || cam.fy <= 0 || cam.width <= 0 || cam.height <= 0)
            throw io_error(path + ": invalid camera intrinsics");
        for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c) cam.w[r][c] = nums[off + 6 + 4 * std::size_t(r) + c];
        cams.push_back(cam);
    }
    return cams;
}
inline void write_cameras(const std::vector<Camera>& cams, const std::string& path) {
    std::ofstream out(path);
    if (!out) throw io_error("cannot write camera file " + path);
    out << std::setprecision(17);
    for (const Camera& cam : cams) {
        out << cam.fx << ' ' << cam.fy << ' ' << cam.cx << ' ' << cam.cy << ' ' << cam.width << ' ' << cam.height
            << '\n';
        for (int r = 0; r < 4; ++r)
            out << cam.w[r][0] << ' ' << cam.w[r][1] << ' ' << cam.w[r][2] << ' ' << cam.w[r][3] << '\n';
    }
    if (!out) throw io_error("write failed for " + path);
}

// ---- optimiser (include/darbs/optim.hpp:12-45)
struct AdamState {
    std::vector<double> m, v;
    explicit AdamState(std::size_t n = 0) : m(n, 0.0), v(n, 0.0) {}
};
inline void adam_step(std::vector<double>& params, const std::vector<double>& grads, AdamState& state,
                      const std::vector<double>& lrs, int t) {
    if (params.size() != grads.size() || params.size() != state.m.size() || params.size() != lrs.size())
        throw contract_violation("adam_step: shape mismatch");  // optim.hpp:26-29
    darbs_cuda_ctx* ctx = default_session().handle();
    std::vector<float> p(params.begin(), params.end()), g(grads.begin(), grads.end()), m(state.m.begin(), state.m.end()),
        v(state.v.begin(), state.v.end()), l(lrs.begin(), lrs.end());
    throw_status(darbs_cuda_adam_step(ctx, (int64_t)p.size(), p.data(), g.data(), m.data(), v.data(), l.data(), t,
                                      DARBS_HOST),
                 ctx);
    // the step is applied to the FP64 master copy, so that many small steps do not round away
    for (std::size_t i = 0; i < p.size(); ++i) params[i] += double(p[i]) - double((float)params[i]);
    state.m.assign(m.begin(), m.end());
    state.v.assign(v.begin(), v.end());
}

// ---- shared fit configuration (include/darbs/fit_common.hpp:15-42)
struct FitConfig {
    double lambda = 0.2;
    double lr_position = 0.00016;
    double lr_scale = 0.005;
    double lr_rotation = 0.001;
    double lr_opacity = 0.02;
    double lr_color = 0.0025;
    int iters = 2000;
    std::uint64_t seed = 0;
    int threads = 1;
};
struct FitReport {
    std::vector<double> loss_curve, l1_curve, dssim_curve, psnr_curve;
    double final_mse = 0.0, final_psnr = 0.0, final_ssim = 0.0, wall_time = 0.0;
    KernelSpec kernel;
    int n = 0;
};
inline double sigmoid(double x) { return 1.0 / (1.0 + std::exp(-x)); }
inline double logit(double p) { return std::log(p / (1.0 - p)); }

// ---- scene rendering and fitting (include/darbs/fit3d.hpp:11-33)
inline constexpr int kParamsPerPrim = DARBS_PARAMS_PER_PRIMITIVE;

// raw parameters of fit_scene (fit3d.cpp:69-80): mu, log scale, raw quaternion, logits
inline void primitive_to_raw(const Primitive3D& p, double* q) {
    for (int k = 0; k < 3; ++k) q[k] = p.mu[k];
    for (int k = 0; k < 3; ++k) {
        if (!(p.scale[k] > 0.0)) throw invalid_parameter("fit_scene: initial scale must be positive");
        q[3 + k] = std::log(p.scale[k]);
    }
    for (int k = 0; k < 4; ++k) q[6 + k] = p.rot.q[k];
    q[10] = logit(std::clamp(p.opacity, 0.01, 0.99));
    for (int c = 0; c < 3; ++c) q[11 + c] = logit(std::clamp(p.color[c], 0.01, 0.99));
}
// realize, fit3d.cpp:17-25
inline Primitive3D realize(const double* q) {
    Primitive3D p;
    p.mu = Vec3(q[0], q[1], q[2]);
    p.scale = Vec3(std::exp(q[3]), std::exp(q[4]), std::exp(q[5]));
    p.rot = Quat(q[6], q[7], q[8], q[9]);
    p.opacity = sigmoid(q[10]);
    p.color = Vec3(sigmoid(q[11]), sigmoid(q[12]), sigmoid(q[13]));
    return p;
}

// A device array owned through the ABI (darbs_cuda_device_alloc / _free).
class DeviceArray {
public:
    DeviceArray() = default;
    DeviceArray(darbs_cuda_ctx* ctx, std::size_t count) : ctx_(ctx), count_(count) {
        throw_status(darbs_cuda_device_alloc(ctx_, sizeof(float) * count, &ptr_), ctx_);
    }
    DeviceArray(DeviceArray&& o) noexcept : ctx_(o.ctx_), ptr_(o.ptr_), count_(o.count_) { o.ptr_ = nullptr; }
    DeviceArray& operator=(DeviceArray&& o) noexcept {
        std::swap(ctx_, o.ctx_);
        std::swap(ptr_, o.ptr_);
        std::swap(count_, o.count_);
        return *this;
    }
    DeviceArray(const DeviceArray&) = delete;
    DeviceArray& operator=(const DeviceArray&) = delete;
    ~DeviceArray() {
        if (ptr_) darbs_cuda_device_free(ctx_, ptr_);
    }
    float* data() const { return static_cast<float*>(ptr_); }
    std::size_t size() const { return count_; }
    void upload(const std::vector<float>& host) {
        throw_status(darbs_cuda_upload(ctx_, ptr_, host.data(), sizeof(float) * std::min(host.size(), count_)), ctx_);
    }
    std::vector<float> download() const {
        std::vector<float> host(count_);
        throw_status(darbs_cuda_download(ctx_, host.data(), ptr_, sizeof(float) * count_), ctx_);
        return host;
    }
    void zero() { throw_status(darbs_cuda_device_zero(ctx_, ptr_, sizeof(float) * count_), ctx_); }

private:
    darbs_cuda_ctx* ctx_ = nullptr;
    void* ptr_ = nullptr;
    std::size_t count_ = 0;
};

// render_scene, src/fit3d.cpp:29-40: project every primitive, keep the visible ones, composite.
inline ImageBuffer render_scene(const std::vector<Primitive3D>& prims, const Camera& cam, const KernelSpec& kernel,
                                double psi, const Vec3& background, int threads = 1, double dilation = kDilation) {
    darbs_cuda_ctx* ctx = default_session().handle();
    const std::size_t n = prims.size();
    std::vector<float> flat(n * kParamsPerPrim), mu2(2 * n), cov2(3 * n), conic(3 * n), radius(n), depth(n);
    std::vector<int32_t> valid(n);
    for (std::size_t i = 0; i < n; ++i) primitive_to_floats(prims[i], flat.data() + i * kParamsPerPrim);
    const darbs_kernel_spec ks = to_abi(kernel);
    const auto block = camera_block(cam);
    if (n > 0)
        throw_status(darbs_cuda_project(ctx, &ks, psi, dilation, (int64_t)n, flat.data(), block.data(), valid.data(),
                                        mu2.data(), cov2.data(), conic.data(), radius.data(), depth.data(),
                                        DARBS_HOST),
                     ctx);
    std::vector<ProjectedSplat> splats;
    splats.reserve(n);
    for (std::size_t i = 0; i < n; ++i) {
        if (!valid[i]) continue;
        ProjectedSplat s;
        s.mu2 = Vec2(mu2[2 * i], mu2[2 * i + 1]);
        s.cov2(0, 0) = cov2[3 * i];
        s.cov2(0, 1) = s.cov2(1, 0) = cov2[3 * i + 1];
        s.cov2(1, 1) = cov2[3 * i + 2];
        s.conic = Conic{conic[3 * i], conic[3 * i + 1], conic[3 * i + 2]};
        s.radius = radius[i];
        s.depth = depth[i];
        s.opacity = prims[i].opacity;
        s.color = prims[i].color;
        splats.push_back(s);
    }
    return forward(splats, kernel, cam.width, cam.height, background, threads).image;
}

struct View {
    Camera camera;
    ImageBuffer target;
};
struct Fit3DResult {
    FitReport report;
    std::vector<Primitive3D> primitives;
    std::vector<double> per_view_psnr;
};

// fit_scene, src/fit3d.cpp:42-203.  The loop is the reference's; the state lives on the GPU.
// Which of the views this process owns when the fit runs on several GPUs of one node (one process
// per GPU): view v belongs to rank v mod world.  With world > 1 the session's
// context must hold a communicator (darbs_cuda_comm_init, collective over the ranks); gradients
// are then summed over all ranks' views by one NCCL all-reduce per iteration inside
// darbs_cuda_train_step, and every rank returns the same fitted scene.
struct ViewShard {
    int rank = 0;
    int world = 1;
};

inline Fit3DResult fit_scene(const std::vector<View>& views, const KernelSpec& kernel, double psi,
                             const std::vector<Primitive3D>& init, const FitConfig& config,
                             const ViewShard& shard = ViewShard()) {
    if (shard.world < 1 || shard.rank < 0 || shard.rank >= shard.world)
        throw invalid_parameter("fit_scene: bad view shard");
    if (views.size() < 2) throw invalid_parameter("fit_scene: need at least 2 views");
    if (init.empty()) throw invalid_parameter("fit_scene: empty initial primitive set");
    const auto t0 = std::chrono::steady_clock::now();
    darbs_cuda_ctx* ctx = default_session().handle();
    const std::size_t n = init.size(), dim = n * kParamsPerPrim;
    const float bg[3] = {0.f, 0.f, 0.f};  // fit3d.cpp:52

    // the position rate scales with the extent of the initial means (fit3d.cpp:54-61)
    Vec3 lo = init.front().mu, hi = init.front().mu;
    for (const Primitive3D& p : init)
        for (int k = 0; k < 3; ++k) {
            lo[k] = std::min(lo[k], p.mu[k]);
            hi[k] = std::max(hi[k], p.mu[k]);
        }
    double ext2 = 0.0;
    for (int k = 0; k < 3; ++k) ext2 += (hi[k] - lo[k]) * (hi[k] - lo[k]);
    const double extent = std::max(1.0, std::sqrt(ext2));

    std::vector<float> params(dim), lrs(dim);
    for (std::size_t i = 0; i < n; ++i) {
        double q[kParamsPerPrim];
        primitive_to_raw(init[i], q);
        for (int k = 0; k < kParamsPerPrim; ++k) params[i * kParamsPerPrim + k] = (float)q[k];
        float* l = lrs.data() + i * kParamsPerPrim;
        l[0] = l[1] = l[2] = (float)(config.lr_position * extent);
        l[3] = l[4] = l[5] = (float)config.lr_scale;
        l[6] = l[7] = l[8] = l[9] = (float)config.lr_rotation;
        l[10] = (float)config.lr_opacity;
        l[11] = l[12] = l[13] = (float)config.lr_color;
    }
    DeviceArray d_params(ctx, dim), d_grads(ctx, dim), d_m(ctx, dim), d_v(ctx, dim), d_lrs(ctx, dim);
    d_params.upload(params);
    d_lrs.upload(lrs);
    d_m.zero();
    d_v.zero();
    std::vector<DeviceArray> d_targets;
    std::vector<std::array<double, DARBS_CAMERA_DOUBLES>> blocks;
    for (const View& view : views) {
        if (view.target.width != view.camera.width || view.target.height != view.camera.height)
            throw invalid_parameter("loss_total: dimension mismatch");
        const std::vector<float> t(view.target.rgb.begin(), view.target.rgb.end());
        d_targets.emplace_back(ctx, t.size());
        d_targets.back().upload(t);
        blocks.push_back(camera_block(view.camera));
    }
    const darbs_kernel_spec ks = to_abi(kernel);

    Fit3DResult result;
    result.report.kernel = kernel;
    result.report.n = (int)n;
    struct IterStats {
        double loss = 0.0, l1 = 0.0, dssim = 0.0, mse = 0.0;
    };
    // one evaluation over all views (fit3d.cpp:104-167); losses are collected one view late
    auto evaluate = [&](bool with_grad) {
        IterStats s;
        std::size_t popped = 0;
        auto pop = [&] {
            double out[4];
            throw_status(darbs_cuda_pop_loss(ctx, out), ctx);
            s.loss += out[0];
            s.l1 += out[1];
            s.dssim += out[2];
            s.mse += out[3];
            ++popped;
        };
        for (std::size_t v = 0; v < views.size(); ++v) {
            // the first view overwrites the gradient buffer: fit3d.cpp:107's fill without a zeroing pass
            if (with_grad && v == 0) throw_status(darbs_cuda_set_accumulate(ctx, 0), ctx);
            throw_status(darbs_cuda_evaluate_view(ctx, &ks, psi, (int64_t)n, d_params.data(), blocks[v].data(), bg,
                                                  d_targets[v].data(), config.lambda, nullptr,
                                                  with_grad ? d_grads.data() : nullptr, nullptr, nullptr,
                                                  DARBS_DEVICE, DARBS_DEVICE),
                         ctx);
            if (v + 1 - popped > 2) pop();
        }
        while (popped < views.size()) pop();
        const double nv = double(views.size());
        s.loss /= nv;
        s.l1 /= nv;
        s.dssim /= nv;
        s.mse /= nv;
        return s;
    };
    auto record = [&](const IterStats& s) {
        result.report.loss_curve.push_back(s.loss);
        result.report.l1_curve.push_back(s.l1);
        result.report.dssim_curve.push_back(s.dssim);
        result.report.psnr_curve.push_back(s.mse > 0.0 ? -10.0 * std::log10(s.mse) : 99.0);
    };
    if (config.iters == 0) record(evaluate(false));
    // the iteration (fit3d.cpp:104-184) runs inside the library: this rank's views, the gradient
    // all-reduce over the ranks (none with one rank), the Adam step
    std::vector<double> local_cameras;
    std::vector<const float*> local_targets;
    for (std::size_t v = (std::size_t)shard.rank; v < views.size(); v += (std::size_t)shard.world) {
        local_cameras.insert(local_cameras.end(), blocks[v].begin(), blocks[v].end());
        local_targets.push_back(d_targets[v].data());
    }
    for (int it = 1; it <= config.iters; ++it) {
        double mean[4];
        throw_status(darbs_cuda_train_step(ctx, &ks, psi, (int64_t)n, d_params.data(), d_grads.data(), d_m.data(),
                                           d_v.data(), d_lrs.data(), (int)local_targets.size(), local_cameras.data(),
                                           local_targets.data(), config.lambda, bg, it, (int)views.size(), mean),
                     ctx);
        IterStats s;
        s.loss = mean[0];
        s.l1 = mean[1];
        s.dssim = mean[2];
        s.mse = mean[3];
        record(s);
    }

    params = d_params.download();
    result.primitives.resize(n);
    for (std::size_t i = 0; i < n; ++i) {
        double q[kParamsPerPrim];
        for (int k = 0; k < kParamsPerPrim; ++k) q[k] = params[i * kParamsPerPrim + k];
        result.primitives[i] = realize(q);
    }
    // final metrics (fit3d.cpp:187-198): the fitted scene rendered per view by the non-throwing
    // render_scene (a view that sees nothing is a background image there, not an error)
    double mse_sum = 0.0, ssim_sum = 0.0;
    for (std::size_t v = 0; v < views.size(); ++v) {
        const ImageBuffer img = render_scene(result.primitives, views[v].camera, kernel, psi, Vec3::Zero(), config.threads);
        const double m = mse(img, views[v].target);
        result.per_view_psnr.push_back(m <= 0.0 ? std::numeric_limits<double>::infinity() : -10.0 * std::log10(m));
        mse_sum += m;
        ssim_sum += ssim(img, views[v].target);
    }
    const double nv = double(views.size());
    result.report.final_mse = mse_sum / nv;
    result.report.final_psnr = result.report.final_mse > 0.0 ? -10.0 * std::log10(result.report.final_mse) : 99.0;
    result.report.final_ssim = ssim_sum / nv;
    result.report.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return result;
}

// ---- 2-D image fitting (include/darbs/fit2d.hpp:12-36)
struct Splat2DParams {
    Vec2 mu2 = Vec2::Zero();
    Vec2 log_scale = Vec2::Zero();
    double angle = 0.0;
    double opacity_logit = 0.0;
    Vec3 color_logit = Vec3::Zero();
};

// realize_splat2d, src/fit2d.cpp:28-43: cov2 = R diag(exp(2 ls)) R^T
inline ProjectedSplat realize_splat2d(const Splat2DParams& p, const KernelSpec& kernel, double depth) {
    const double c = std::cos(p.angle), s = std::sin(p.angle);
    const double sx = std::exp(p.log_scale.x()), sy = std::exp(p.log_scale.y());
    const double m[2][2] = {{c * sx, -s * sy}, {s * sx, c * sy}};  // M = R diag(sx, sy)
    ProjectedSplat out;
    out.mu2 = p.mu2;
    for (int r = 0; r < 2; ++r)
        for (int q = 0; q < 2; ++q) out.cov2(r, q) = m[r][0] * m[q][0] + m[r][1] * m[q][1];
    const ConicRadius cr = conic_and_radius(out.cov2, kernel);
    out.conic = cr.conic;
    out.radius = cr.radius;
    out.depth = depth;
    out.opacity = sigmoid(p.opacity_logit);
    out.color = Vec3(sigmoid(p.color_logit[0]), sigmoid(p.color_logit[1]), sigmoid(p.color_logit[2]));
    return out;
}

struct Fit2DResult {
    FitReport report;
    ImageBuffer rendered;
    std::vector<Splat2DParams> splats;
};

// fit_image, src/fit2d.cpp:45-188: nine raw parameters per splat, host chain, device rasterizer.
inline Fit2DResult fit_image(const ImageBuffer& target, const KernelSpec& kernel, int n_splats,
                             const FitConfig& config) {
    if (n_splats < 1) throw invalid_parameter("fit_image: n_splats must be >= 1");
    constexpr int kP = 9;  // mu(2) log_scale(2) angle opacity color(3)
    const auto t0 = std::chrono::steady_clock::now();
    const int w = target.width, h = target.height;
    const Vec3 background = Vec3::Zero();
    const std::size_t dim = std::size_t(n_splats) * kP;
    std::vector<double> params(dim), grads(dim), lrs(dim);
    {
        // seeding over the image domain, colours sampled from the target (fit2d.cpp:54-72)
        std::mt19937_64 rng(config.seed);
        std::uniform_real_distribution<double> ux(0.0, double(w)), uy(0.0, double(h)), uang(0.0, 3.14159265358979323846);
        const double r0 = std::max(1.0, 0.6 * std::sqrt(double(w) * h / n_splats));
        const double extent = std::max(w, h);
        for (int i = 0; i < n_splats; ++i) {
            double* q = params.data() + std::size_t(i) * kP;
            // the reference writes Vec2(ux(rng), uy(rng)) (fit2d.cpp:60): the order of the two draws is
            // unspecified by the language; GCC, the compiler the reference is built with,
            // evaluates the arguments right to left, and so does this mirror
            q[1] = uy(rng);
            q[0] = ux(rng);
            q[2] = q[3] = std::log(r0);
            q[4] = uang(rng);
            q[5] = logit(0.5);
            const int px = std::clamp(int(q[0]), 0, w - 1), py = std::clamp(int(q[1]), 0, h - 1);
            for (int c = 0; c < 3; ++c) q[6 + c] = logit(std::clamp(target.at(px, py, c), 0.02, 0.98));
            double* l = lrs.data() + std::size_t(i) * kP;
            l[0] = l[1] = config.lr_position * extent;
            l[2] = l[3] = config.lr_scale;
            l[4] = config.lr_rotation;
            l[5] = config.lr_opacity;
            l[6] = l[7] = l[8] = config.lr_color;
        }
    }
    AdamState state(dim);
    Fit2DResult result;
    result.report.kernel = kernel;
    result.report.n = n_splats;
    std::vector<ProjectedSplat> splats(n_splats);
    auto unpack = [&](int i) {
        const double* q = params.data() + std::size_t(i) * kP;
        return Splat2DParams{Vec2(q[0], q[1]), Vec2(q[2], q[3]), q[4], q[5], Vec3(q[6], q[7], q[8])};
    };
    auto realize_all = [&] {
        for (int i = 0; i < n_splats; ++i) splats[i] = realize_splat2d(unpack(i), kernel, double(i));
    };
    for (int it = 1; it <= config.iters; ++it) {
        realize_all();
        ForwardResult fwd = forward(splats, kernel, w, h, background, config.threads);
        LossResult loss = loss_total(fwd.image, target, config.lambda);
        if (!std::isfinite(loss.total))
            throw numeric_error("fit_image: loss diverged at iteration " + std::to_string(it));
        result.report.loss_curve.push_back(loss.total);
        result.report.l1_curve.push_back(loss.l1);
        result.report.dssim_curve.push_back(loss.dssim);
        result.report.psnr_curve.push_back(psnr(fwd.image, target));
        const std::vector<SplatGrads> sg = backward(loss.grad, splats, kernel, fwd.aux, config.threads);
        std::fill(grads.begin(), grads.end(), 0.0);
        for (int i = 0; i < n_splats; ++i) {
            const double* q = params.data() + std::size_t(i) * kP;
            double* g = grads.data() + std::size_t(i) * kP;
            const SplatGrads& gi = sg[i];
            const ProjectedSplat& s = splats[i];
            g[0] = gi.d_mu2.x();
            g[1] = gi.d_mu2.y();
            // conic gradient -> covariance gradient: dL/dcov2 = -C G C with G symmetric (fit2d.cpp:137-144)
            const double G[2][2] = {{gi.d_conic_a, 0.5 * gi.d_conic_b}, {0.5 * gi.d_conic_b, gi.d_conic_c}};
            const double C[2][2] = {{s.conic.a, s.conic.b}, {s.conic.b, s.conic.c}};
            double CG[2][2], dcov[2][2];
            for (int r = 0; r < 2; ++r)
                for (int c = 0; c < 2; ++c) CG[r][c] = C[r][0] * G[0][c] + C[r][1] * G[1][c];
            for (int r = 0; r < 2; ++r)
                for (int c = 0; c < 2; ++c) dcov[r][c] = -(CG[r][0] * C[0][c] + CG[r][1] * C[1][c]);
            // cov2 = M M^T, M = R(angle) diag(exp(ls)): dL/dM = 2 dcov M (fit2d.cpp:146-163)
            const double ca = std::cos(q[4]), sa = std::sin(q[4]);
            const double R[2][2] = {{ca, -sa}, {sa, ca}}, dR[2][2] = {{-sa, -ca}, {ca, -sa}};
            const double sc[2] = {std::exp(q[2]), std::exp(q[3])};
            double dM[2][2];
            for (int r = 0; r < 2; ++r)
                for (int c = 0; c < 2; ++c) dM[r][c] = 2.0 * (dcov[r][0] * R[0][c] * sc[c] + dcov[r][1] * R[1][c] * sc[c]);
            for (int k = 0; k < 2; ++k) {
                g[2] += dM[k][0] * R[k][0] * sc[0];
                g[3] += dM[k][1] * R[k][1] * sc[1];
                for (int j = 0; j < 2; ++j) g[4] += dM[k][j] * dR[k][j] * sc[j];
            }
            g[5] = gi.d_opacity * s.opacity * (1.0 - s.opacity);
            for (int c = 0; c < 3; ++c) g[6 + c] = gi.d_color[c] * s.color[c] * (1.0 - s.color[c]);
        }
        adam_step(params, grads, state, lrs, it);
    }
    realize_all();
    result.rendered = forward(splats, kernel, w, h, background, config.threads).image;
    result.report.final_mse = mse(result.rendered, target);
    result.report.final_psnr = psnr(result.rendered, target);
    result.report.final_ssim = ssim(result.rendered, target);
    result.report.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    result.splats.resize(n_splats);
    for (int i = 0; i < n_splats; ++i) result.splats[i] = unpack(i);
    return result;
}

}  // namespace darbs_b200
