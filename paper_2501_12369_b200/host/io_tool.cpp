// io_tool.cpp — exercises the file formats of the C++ mirror (darbs_b200_fit.hpp) without a GPU:
//   io_tool copy-scene   in out     read_scene    -> write_scene
//   io_tool copy-cameras in out     read_cameras  -> write_cameras
//   io_tool copy-dsfl    in out     read_float_dump -> write_float_dump
//   io_tool copy-ppm     in out     read_ppm      -> write_ppm
//   io_tool dsfl-to-ppm  in out     read_float_dump -> write_ppm
//   io_tool stats        a b        mse and psnr of two .dsfl images
// tests/test_host_io.py byte-compares the outputs with files the reference's own writers made
// (src/scene_io.cpp, src/image.cpp; tests/golden/io/).  Exit code 3 on io_error, as the
// reference's CLI maps it (tools/main.cpp:487-499).
#include <cstdio>
#include <string>

#include "darbs_b200_fit.hpp"

using namespace darbs_b200;

int main(int argc, char** argv) {
    if (argc != 4) {
        std::fprintf(stderr, "usage: io_tool <command> <in> <out>\n");
        return 1;
    }
    const std::string cmd = argv[1], in = argv[2], out = argv[3];
    try {
        if (cmd == "copy-scene") {
            write_scene(read_scene(in), out);
        } else if (cmd == "copy-cameras") {
            write_cameras(read_cameras(in), out);
        } else if (cmd == "copy-dsfl") {
            write_float_dump(read_float_dump(in), out);
        } else if (cmd == "copy-ppm") {
            write_ppm(read_ppm(in), out);
        } else if (cmd == "dsfl-to-ppm") {
            write_ppm(read_float_dump(in), out);
        } else if (cmd == "stats") {
            const ImageBuffer a = read_float_dump(in), b = read_float_dump(out);
            std::printf("%.17g %.17g\n", mse(a, b), psnr(a, b));
        } else {
            std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
            return 1;
        }
    } catch (const io_error& e) {
        std::fprintf(stderr, "io_error: %s\n", e.what());
        return 3;
    } catch (const invalid_parameter& e) {
        std::fprintf(stderr, "invalid_parameter: %s\n", e.what());
        return 1;
    }
    return 0;
}
