// fit_tool.cpp — the reference's `render`, `fit-scene` and `fit-image` subcommands
// (tools/main.cpp:336-436) in the shape the parity tests need, over the C++ mirror
// (darbs_b200_fit.hpp) and therefore over the CUDA path.  Not the reference's CLI (its option
// schema, config files and run manifest are out of scope): fixed positional arguments, results as
// plain text so that tests/test_gpu_fit_drivers.py can compare them with what the reference's own
// fit_scene / fit_image / render_scene produced on the same files (tests/golden/fit/).
//
//   fit_tool render     <scene.txt> <cameras.txt> <kernel> <psi|default> <out_dir>
//       -> out_dir/view_<i>.dsfl                                  (main.cpp:336-351)
//   fit_tool fit-scene  <truth.txt|targets_dir> <cameras.txt> <init.txt> <kernel> <psi_fit|default>
//                       <iters> <out.txt> [deterministic]
//       targets: a directory holding view_<i>.dsfl, or a scene file that is rendered with the
//       kernel's default psi first (self-reconstruction, main.cpp:385-391 / acceptance.cpp:386-390)
//   fit_tool fit-image  <target.dsfl> <kernel> <n_splats> <iters> <seed> <out.txt> [deterministic]
//
// out.txt: "curve <it> <loss> <l1> <dssim> <psnr>" per iteration, "final <mse> <psnr> <ssim>",
// "view <i> <psnr>", then "prim ..." / "splat ..." rows with 17 significant digits.
// Exit codes follow tools/main.cpp:487-499 (usage / invalid_parameter 1, io 3, everything else 2).
#include <sys/stat.h>

#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iomanip>
#include <string>

#include "darbs_b200_fit.hpp"

using namespace darbs_b200;

namespace {

bool is_dir(const std::string& p) {
    struct stat st;
    return ::stat(p.c_str(), &st) == 0 && S_ISDIR(st.st_mode);
}

double psi_of(const std::string& arg, const std::string& kernel) {
    if (arg != "default") return std::atof(arg.c_str());
    const double psi = darbs_cuda_default_psi(kernel.c_str());
    if (psi <= 0.0) throw invalid_parameter("no default psi for kernel " + kernel);
    return psi;
}

KernelSpec kernel_of(const std::string& name) {
    auto k = kernel_preset(name);
    if (!k) throw invalid_parameter("unknown kernel " + name);
    return *k;
}

void write_report(std::ostream& out, const FitReport& r) {
    out << std::setprecision(17);
    for (std::size_t i = 0; i < r.loss_curve.size(); ++i)
        out << "curve " << i << ' ' << r.loss_curve[i] << ' ' << r.l1_curve[i] << ' ' << r.dssim_curve[i] << ' '
            << r.psnr_curve[i] << '\n';
    out << "final " << r.final_mse << ' ' << r.final_psnr << ' ' << r.final_ssim << '\n';
}

void set_deterministic(bool on) {
    if (!on) return;
    throw_status(darbs_cuda_set_deterministic(default_session().handle(), 1), default_session().handle());
}

int run(int argc, char** argv) {
    const std::string cmd = argc > 1 ? argv[1] : "";
    if (cmd == "render" && argc == 7) {
        const auto prims = read_scene(argv[2]);
        const auto cams = read_cameras(argv[3]);
        const KernelSpec k = kernel_of(argv[4]);
        const double psi = psi_of(argv[5], argv[4]);
        for (std::size_t v = 0; v < cams.size(); ++v)
            write_float_dump(render_scene(prims, cams[v], k, psi, Vec3::Zero()),
                             std::string(argv[6]) + "/view_" + std::to_string(v) + ".dsfl");
        return 0;
    }
    if (cmd == "fit-scene" && (argc == 9 || argc == 10)) {
        const auto cams = read_cameras(argv[3]);
        const auto init = read_scene(argv[4]);
        const KernelSpec k = kernel_of(argv[5]);
        const double psi_fit = psi_of(argv[6], argv[5]);
        std::vector<View> views;
        if (is_dir(argv[2])) {
            for (std::size_t v = 0; v < cams.size(); ++v)
                views.push_back(View{cams[v], read_float_dump(std::string(argv[2]) + "/view_" + std::to_string(v) + ".dsfl")});
        } else {
            const auto truth = read_scene(argv[2]);
            const double psi_render = psi_of("default", argv[5]);
            for (const Camera& cam : cams) views.push_back(View{cam, render_scene(truth, cam, k, psi_render, Vec3::Zero())});
        }
        FitConfig cfg;
        cfg.iters = std::atoi(argv[7]);
        cfg.seed = 1;
        set_deterministic(argc == 10 && std::string(argv[9]) == "deterministic");
        const Fit3DResult res = fit_scene(views, k, psi_fit, init, cfg);
        std::ofstream out(argv[8]);
        if (!out) throw io_error(std::string("cannot write ") + argv[8]);
        write_report(out, res.report);
        for (std::size_t v = 0; v < res.per_view_psnr.size(); ++v) out << "view " << v << ' ' << res.per_view_psnr[v] << '\n';
        for (const Primitive3D& p : res.primitives)
            out << "prim " << p.mu[0] << ' ' << p.mu[1] << ' ' << p.mu[2] << ' ' << p.scale[0] << ' ' << p.scale[1] << ' '
                << p.scale[2] << ' ' << p.rot.w() << ' ' << p.rot.x() << ' ' << p.rot.y() << ' ' << p.rot.z() << ' ' << p.opacity
                << ' ' << p.color[0] << ' ' << p.color[1] << ' ' << p.color[2] << '\n';
        return 0;
    }
    if (cmd == "fit-image" && (argc == 8 || argc == 9)) {
        const ImageBuffer target = read_float_dump(argv[2]);
        const KernelSpec k = kernel_of(argv[3]);
        FitConfig cfg;
        cfg.iters = std::atoi(argv[5]);
        cfg.seed = std::strtoull(argv[6], nullptr, 10);
        set_deterministic(argc == 9 && std::string(argv[8]) == "deterministic");
        const Fit2DResult res = fit_image(target, k, std::atoi(argv[4]), cfg);
        std::ofstream out(argv[7]);
        if (!out) throw io_error(std::string("cannot write ") + argv[7]);
        write_report(out, res.report);
        for (const Splat2DParams& s : res.splats)
            out << "splat " << s.mu2.x() << ' ' << s.mu2.y() << ' ' << s.log_scale.x() << ' ' << s.log_scale.y() << ' '
                << s.angle << ' ' << s.opacity_logit << ' ' << s.color_logit[0] << ' ' << s.color_logit[1] << ' '
                << s.color_logit[2] << '\n';
        return 0;
    }
    std::fprintf(stderr, "usage: fit_tool render|fit-scene|fit-image ... (see the header of fit_tool.cpp)\n");
    return 1;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        return run(argc, argv);
    } catch (const io_error& e) {
        std::fprintf(stderr, "io_error: %s\n", e.what());
        return 3;
    } catch (const invalid_parameter& e) {
        std::fprintf(stderr, "invalid_parameter: %s\n", e.what());
        return 1;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
}
