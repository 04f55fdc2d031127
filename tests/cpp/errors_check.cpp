// errors_check.cpp -- the reference API's failure behaviour, written as a
// caller of the reference library writes it: only "sobel5/..." headers and
// the public API.  The SAME source builds against the reference (CPU) and
// against this repo's drop-in (GPU); tests/test_cpp_acceptance.py compares
// the two outputs line for line (tests/golden/errors_check.txt is the
// reference build's output).  Prints one line per call: the exception type
// and message, or "ok" with a checksum of the result.
//
// Covers: ParityViolation from fault-injected StreamTaps for every kernel
// family of the drop-in (int16 runtime taps, packed FP32, generic 32-bit)
// and strip plans of many lane widths, workers = 1 (the reported pair is
// the first odd pixel in strip, row, column order: pipeline.hpp:416-445,
// 268-273); run_stream's validation order (ImageTooSmall, DimMismatch);
// make_stream_taps / plan_strips / pad_replicate / quantize errors.
#include "sobel5/filter_algebra.hpp"
#include "sobel5/image_io.hpp"
#include "sobel5/pipeline.hpp"
#include "sobel5/strips.hpp"
#include "sobel5/synth.hpp"

#include <cstdint>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>

using namespace sobel5;

namespace {

template <class T>
std::uint64_t fnv(const Plane<T>& p) {
    std::uint64_t h = 1469598103934665603ull;
    const auto* b = reinterpret_cast<const unsigned char*>(p.data().data());
    for (std::size_t i = 0; i < p.size() * sizeof(T); ++i) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}

void line(const std::string& what, const std::function<std::string()>& fn) {
    std::string out;
    try {
        out = "ok " + fn();
    } catch (const ParityViolation& e) {
        out = std::string("ParityViolation: ") + e.what();
    } catch (const ImageTooSmall& e) {
        out = std::string("ImageTooSmall: ") + e.what();
    } catch (const DimMismatch& e) {
        out = std::string("DimMismatch: ") + e.what();
    } catch (const LaneTooNarrow& e) {
        out = std::string("LaneTooNarrow: ") + e.what();
    } catch (const EmptyPlane& e) {
        out = std::string("EmptyPlane: ") + e.what();
    } catch (const NonPositiveParam& e) {
        out = std::string("NonPositiveParam: ") + e.what();
    } catch (const ParamOverflow& e) {
        out = std::string("ParamOverflow: ") + e.what();
    } catch (const std::exception& e) {
        out = std::string("other: ") + e.what();
    }
    std::printf("%s -> %s\n", what.c_str(), out.c_str());
}

std::string hex(std::uint64_t v) {
    char b[24];
    std::snprintf(b, sizeof b, "%016llx", static_cast<unsigned long long>(v));
    return b;
}

}  // namespace

int main() {
    // fault-injected taps: k1[2] += 1 makes P + M odd wherever the centre
    // pixels of rows v+1 and v+3 differ in parity
    const long long params[3][4] = {{1, 1, 1, 1}, {2, 3, 5, 7}, {1, 32768, 1, 1}};
    const int lanes_set[6] = {5, 8, 13, 37, 64, 4096};
    for (const auto& pr : params) {
        FilterParams p;
        p.a = pr[0];
        p.b = Rational(pr[1]);
        p.m = Rational(pr[2]);
        p.n = Rational(pr[3]);
        StreamTaps t = make_stream_taps(p);
        t.k1[2] += 1;
        for (int lanes : lanes_set) {
            for (int seed = 1; seed <= 2; ++seed) {
                const int w = 300 + seed, h = 90 + 7 * seed;
                const GrayPlane img = synth_random(w, h, 40 + static_cast<std::uint64_t>(seed));
                line("parity (" + std::to_string(pr[0]) + "," + std::to_string(pr[1]) + "," +
                         std::to_string(pr[2]) + "," + std::to_string(pr[3]) + ") lanes " +
                         std::to_string(lanes) + " seed " + std::to_string(seed),
                     [&] {
                         const StreamResult r =
                             run_stream(img, t, plan_strips(w, lanes, 2), Prefetch::on, 1);
                         return hex(fnv(r.gd));
                     });
            }
        }
        // an even fault computes the reference's planes
        StreamTaps te = make_stream_taps(p);
        te.k1[2] += 2;
        const GrayPlane img = synth_random(257, 65, 9);
        line("even fault (" + std::to_string(pr[1]) + ")", [&] {
            const StreamResult r = run_stream(img, te, plan_strips(257, 32, 2), Prefetch::off, 1);
            return hex(fnv(r.gx) ^ fnv(r.gd) ^ fnv(r.gdt) ^ fnv(r.g));
        });
    }
    // run_stream's validation order (pipeline.hpp:454-460)
    line("run_stream 4x9", [] {
        return hex(fnv(run_stream(GrayPlane(4, 9), FilterParams{}, plan_strips(4, 8, 1),
                                  Prefetch::on).gx));
    });
    line("run_stream plan width", [] {
        return hex(fnv(run_stream(GrayPlane(40, 9), FilterParams{}, plan_strips(41, 8, 2),
                                  Prefetch::on).gx));
    });
    line("run_stream plan radius", [] {
        return hex(fnv(run_stream(GrayPlane(40, 9), FilterParams{}, plan_strips(40, 8, 1),
                                  Prefetch::on).gx));
    });
    line("run_stream_3x3 2x9", [] {
        return hex(fnv(run_stream_3x3(GrayPlane(2, 9), plan_strips(2, 4, 1), Prefetch::on).gx));
    });
    // host-side errors
    line("params a=0", [] {
        FilterParams p;
        p.a = 0;
        make_stream_taps(p);
        return std::string("taps");
    });
    line("params b=-2", [] {
        FilterParams p;
        p.b = Rational(-2);
        make_stream_taps(p);
        return std::string("taps");
    });
    line("params n=1e9", [] {
        FilterParams p;
        p.n = Rational(1000000000);
        make_stream_taps(p);
        return std::string("taps");
    });
    line("plan lanes 4 r 2", [] { return std::to_string(plan_strips(100, 4, 2).strips.size()); });
    line("plan width 4 r 2", [] { return std::to_string(plan_strips(4, 16, 2).strips.size()); });
    line("pad empty", [] { return std::to_string(pad_replicate(GrayPlane(), 2).plane.width()); });
    line("quantize empty", [] {
        return std::to_string(detail::quantize(RealPlane(), SaveMode::normalize).width());
    });
    line("quantize gray", [] {
        return hex(fnv(detail::quantize(synth_random(33, 17, 3), SaveMode::normalize)));
    });
    return 0;
}
