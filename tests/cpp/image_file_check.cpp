// image_file_check.cpp -- the reference's image file API (image_io.hpp:20-223)
// through the drop-in headers, written as a reference caller writes it.
//   image_file_check load <path>...      one line per file: "ok WxH fnv" or
//                                        "<Exception>: <message>"
//   image_file_check save <raw> <w> <h> <out>...   writes the raw 8-bit
//                                        plane with save_gray to each out
//                                        (prints "ok" or the exception)
// tests/test_image_file.py compares the lines with tests/golden/png.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

#include "sobel5/image_io.hpp"

using namespace sobel5;

namespace {

std::string fnv(const GrayPlane& p) {
    std::uint64_t h = 1469598103934665603ull;
    for (std::uint8_t b : p.data()) h = (h ^ b) * 1099511628211ull;
    char s[24];
    std::snprintf(s, sizeof s, "%016llx", static_cast<unsigned long long>(h));
    return s;
}

template <class F>
std::string guarded(F&& f) {
    try {
        return f();
    } catch (const UnsupportedFormat& e) {
        return std::string("UnsupportedFormat: ") + e.what();
    } catch (const CorruptFile& e) {
        return std::string("CorruptFile: ") + e.what();
    } catch (const IoError& e) {
        return std::string("IoError: ") + e.what();
    } catch (const UnsupportedExtension& e) {
        return std::string("UnsupportedExtension: ") + e.what();
    } catch (const std::exception& e) {
        return std::string("other: ") + e.what();
    }
}

}  // namespace

int main(int argc, char** argv) {
    if (argc >= 3 && std::string(argv[1]) == "load") {
        for (int i = 2; i < argc; ++i)
            std::printf("%s\n", guarded([&] {
                            const GrayPlane g = load_gray(argv[i]);
                            return "ok " + std::to_string(g.width()) + "x" + std::to_string(g.height()) +
                                   " " + fnv(g);
                        }).c_str());
        return 0;
    }
    if (argc >= 6 && std::string(argv[1]) == "save") {
        const int w = std::atoi(argv[3]), h = std::atoi(argv[4]);
        std::ifstream in(argv[2], std::ios::binary);
        std::vector<std::uint8_t> px(static_cast<std::size_t>(w) * h);
        in.read(reinterpret_cast<char*>(px.data()), static_cast<std::streamsize>(px.size()));
        const GrayPlane img(w, h, std::move(px));
        for (int i = 5; i < argc; ++i)
            std::printf("%s\n", guarded([&] {
                            save_gray(img, argv[i]);
                            return std::string("ok");
                        }).c_str());
        return 0;
    }
    std::fprintf(stderr, "usage: image_file_check load <path>... | save <raw> <w> <h> <out>...\n");
    return 2;
}
