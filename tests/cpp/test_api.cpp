// test_api.cpp -- the drop-in C++ API (include/sobel5_b200/sobel5.hpp)
// exercised the way the reference's SPEC.md examples and ACCEPTANCE criteria
// describe.  Framework-free, one line per failed check.
//
//   build/test_api          host-side checks (no GPU needed)
//   build/test_api --gpu    + run_stream on the device vs a brute-force
//                             correlation written here as the checker
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <string>

#include "sobel5_b200/sobel5.hpp"

using namespace sobel5;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                            \
    do {                                                                       \
        ++g_checks;                                                            \
        if (!(cond)) {                                                         \
            ++g_fail;                                                          \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
        }                                                                      \
    } while (0)

template <class E>
static std::string throws(const std::function<void()>& fn) {
    try {
        fn();
    } catch (const E& e) {
        return e.what();
    } catch (const std::exception& e) {
        return std::string("WRONG TYPE: ") + e.what();
    }
    return "NO THROW";
}

// brute-force valid-mode correlation with int64 accumulation (the checker)
static SignedPlane corr(const GrayPlane& img, const Kernel5& k) {
    SignedPlane out(img.width() - 4, img.height() - 4);
    for (int y = 0; y < out.height(); ++y)
        for (int x = 0; x < out.width(); ++x) {
            long long acc = 0;
            for (int i = 0; i < 5; ++i)
                for (int j = 0; j < 5; ++j) acc += static_cast<long long>(k.at(i, j)) * img.at(y + i, x + j);
            out.at(y, x) = static_cast<std::int32_t>(acc);
        }
    return out;
}

static void host_checks() {
    // ---- filter algebra (SPEC filter_algebra examples) ----
    CHECK(throws<NonIntegralWeight>([] { validate_params({1, Rational(1, 2), 6, 4}); }) ==
          "Kx(0,1) = -1/2 is not an integer");
    CHECK(throws<NonPositiveParam>([] { validate_params({0, 2, 6, 4}); }) == "a = 0 must be a positive integer");
    CHECK(throws<NonPositiveParam>([] { validate_params({1, 2, Rational(-6), 4}); }) == "m = -6 must be positive");
    CHECK(throws<ParamOverflow>([] { validate_params({1, 65536, 1, 1}); }) ==
          "largest weight magnitude 65536 exceeds 32768");
    const Kernel5 kx = materialize(FilterParams{}, Direction::X);
    CHECK((kx.w[0] == std::array<std::int32_t, 5>{-1, -2, 0, 2, 1}));
    CHECK((kx.w[2] == std::array<std::int32_t, 5>{-6, -12, 0, 12, 6}));
    const Kernel5 kd = materialize(FilterParams{}, Direction::D);
    CHECK((kd.w[0] == std::array<std::int32_t, 5>{-6, -4, -1, -2, 0}));
    const Kernel5 kdt = materialize(FilterParams{}, Direction::DT);
    CHECK((kdt.w[0] == std::array<std::int32_t, 5>{0, -2, -1, -4, -6}));
    const auto sd = make_kd_sum_diff(FilterParams{});
    CHECK((sd.plus.w[0] == std::array<std::int32_t, 5>{-6, -6, -2, -6, -6}));
    CHECK((sd.plus.w[2] == std::array<std::int32_t, 5>{0, 0, 0, 0, 0}));
    CHECK((sd.minus.w[0] == std::array<std::int32_t, 5>{-6, -2, 0, 2, 6}));
    const auto dm = decompose_kd_minus(FilterParams{});
    CHECK((dm.deriv_term.col == std::array<std::int32_t, 5>{6, 6, 2, 6, 6}));
    CHECK((dm.diff_term.col == std::array<std::int32_t, 5>{10, 0, -12, 0, 10}));
    // ACCEPTANCE 3: identities over random valid parameter sets
    std::mt19937 rng(3);
    int tested = 0;
    for (int trial = 0; trial < 4000 && tested < 1000; ++trial) {
        FilterParams p{1 + static_cast<int>(rng() % 3), 1 + static_cast<int>(rng() % 9),
                       1 + static_cast<int>(rng() % 9), 1 + static_cast<int>(rng() % 9)};
        try {
            validate_params(p);
        } catch (const Error&) {
            continue;
        }
        ++tested;
        const Kernel5 d = materialize(p, Direction::D), t = materialize(p, Direction::DT);
        const auto s = make_kd_sum_diff(p);
        const auto dec = decompose_kd_minus(p);
        const Kernel5 a = dec.deriv_term.outer(), b = dec.diff_term.outer();
        bool ok = true;
        for (int i = 0; i < 5; ++i)
            for (int j = 0; j < 5; ++j) {
                ok &= s.plus.at(i, j) + s.minus.at(i, j) == 2 * d.at(i, j);
                ok &= s.plus.at(i, j) - s.minus.at(i, j) == 2 * t.at(i, j);
                ok &= a.at(i, j) - b.at(i, j) == s.minus.at(i, j);
            }
        CHECK(ok);
    }
    CHECK(tested == 1000);

    // ---- taps ----
    const StreamTaps t = make_stream_taps(FilterParams{});
    CHECK((t.k1 == std::array<std::int32_t, 5>{-2, -12, -16, -12, -2}));
    CHECK((t.gdm_d == std::array<std::int32_t, 5>{10, 0, -12, 0, 10}));
    CHECK(!t.wide_vagg);
    CHECK(make_stream_taps({1, 32768, 1, 1}).wide_vagg);

    // ---- strips (SPEC plan_strips examples, ACCEPTANCE 8) ----
    const auto p60 = plan_strips(60, 32, 2);
    CHECK(p60.strips.size() == 2 && p60.strips[1].in_off == 28 && p60.strips[1].out_w == 28);
    CHECK(plan_strips(36, 32, 2).strips.back().out_w == 4);
    CHECK(plan_strips(32, 32, 2).strips.size() == 1);
    CHECK(throws<LaneTooNarrow>([] { plan_strips(10, 4, 2); }) == "lane width 4 leaves no output columns at radius 2");
    bool cover = true;
    for (int w = 5; w <= 4096; w += (w < 300 ? 1 : 97))
        for (int lanes : {8, 16, 32, 64}) {
            const auto pl = plan_strips(w, lanes, 2);
            int next = 0;
            for (const auto& s : pl.strips) {
                cover &= s.out_off == next && s.in_off == s.out_off && s.out_w > 0;
                next += s.out_w;
            }
            cover &= next == w - 4;
        }
    CHECK(cover);

    // ---- row helpers (SPEC pipeline examples) ----
    const std::uint8_t r12345[5] = {1, 2, 3, 4, 5};
    CHECK(hpass_f(r12345, FilterParams{})[0] == 8);
    CHECK(hpass_h(r12345, FilterParams{})[0] == 48);
    CHECK(hpass_d(r12345)[0] == 2);
    const std::uint8_t imp[5] = {0, 0, 1, 0, 0};
    CHECK(hpass_kd(imp, KdVariant::k0, FilterParams{})[0] == -2);
    CHECK(hpass_kd(imp, KdVariant::k1, FilterParams{})[0] == -16);
    const std::uint8_t c7[5] = {7, 7, 7, 7, 7};
    CHECK(hpass_kd(c7, KdVariant::k0, FilterParams{})[0] == -182);
    const std::uint8_t four[4] = {1, 2, 3, 4};
    CHECK(throws<RowTooShort>([&] { hpass_d(four); }) == "row of 4 pixels, need >= 5");
    RowRing f(5, 1);
    for (int u = 0; u < 5; ++u) f.acquire(u)[0] = 8;
    CHECK(vagg_gx(f, 2, FilterParams{})[0] == 128);
    RowRing hr(5, 1);
    for (int u = 0; u < 5; ++u) hr.acquire(u)[0] = u == 1 ? 1 : 0;
    CHECK(vagg_gy(hr, 2, FilterParams{})[0] == -2);
    CHECK(!throws<MissingRow>([&] { (void)f.row(7); }).empty());
    KdPlusBank bank(6, 1);
    bank.acquire(0, KdVariant::k0)[0] = 1;
    bank.acquire(1, KdVariant::k1)[0] = 2;
    bank.acquire(2, KdVariant::k1)[0] = 0;
    bank.acquire(3, KdVariant::k1)[0] = 2;
    bank.acquire(4, KdVariant::k0)[0] = 1;
    CHECK(vagg_gd_plus(bank, 2)[0] == 0);  // symmetric cancellation
    CHECK(throws<VariantMismatch>([&] { (void)bank.row(1, KdVariant::k0); }) ==
          "bank row 1 holds variant k1, wanted k0");
    CHECK((recover_diag(10, 4) == std::pair<std::int32_t, std::int32_t>{7, 3}));
    CHECK(throws<ParityViolation>([] { recover_diag(3, 4); }) == "odd sum/difference pair (3, 4)");
    // ACCEPTANCE 6: ring law for row sequences up to 64
    bool law = true;
    for (int depth : {5, 6})
        for (int n = 5; n <= 64; ++n) {
            RowRing r(depth, 1);
            for (int u = 0; u < n; ++u) {
                r.acquire(u);
                const int v = depth == 6 ? u - 3 : u - 2;  // centre served after row u arrives
                if (v >= 2)
                    for (int k = v - 2; k <= std::min(v + 2, u); ++k) law &= r.holds(k);
            }
        }
    CHECK(law);

    // ---- rationals, synth ----
    CHECK(Rational::parse("0.25").value() == Rational(1, 4));
    CHECK(Rational::parse("3/2").value() == Rational(3, 2));
    CHECK(!Rational::parse("1/0").has_value());
    const GrayPlane s = synth_random(16, 1, 1);
    const std::uint8_t want[16] = {193, 92, 2, 137, 236, 45, 10, 145, 103, 236, 142, 101, 161, 141, 235, 190};
    CHECK(std::memcmp(s.data().data(), want, 16) == 0);
}

static void gpu_checks() {
    // SPEC run_stream examples
    const GrayPlane ramp = synth_ramp_x(5, 5);
    const auto rr = run_stream(ramp, FilterParams{}, plan_strips(5, 32, 2), Prefetch::on);
    CHECK(rr.gx.at(0, 0) == 128 && rr.gy.at(0, 0) == 0 && rr.gd.at(0, 0) == 96 && rr.gdt.at(0, 0) == -96);
    CHECK(rr.g.at(0, 0) == 186.59046063504962);
    const auto rc = run_stream(synth_constant(9, 9, 7), FilterParams{}, plan_strips(9, 8, 2), Prefetch::off);
    CHECK(rc.g.at(2, 2) == 0.0 && rc.gd.at(1, 1) == 0);
    CHECK(throws<ImageTooSmall>([] {
              run_stream(GrayPlane(9, 4), FilterParams{}, plan_strips(9, 32, 2), Prefetch::on);
          }) == "streaming filter needs at least 5x5, got 9x4");
    CHECK(throws<DimMismatch>([] {
              run_stream(GrayPlane(9, 9), FilterParams{}, plan_strips(10, 32, 2), Prefetch::on);
          }) == "strip plan covers 10 columns at radius 2, image has 9");

    // ACCEPTANCE 1 (+2): seeded random images, lanes x prefetch, vs brute force
    std::mt19937 rng(1);
    int images = 0;
    bool all_equal = true;
    for (int trial = 0; trial < 64; ++trial) {
        const int w = 5 + static_cast<int>(rng() % 300), h = 5 + static_cast<int>(rng() % 120);
        GrayPlane img = synth_random(w, h, 100 + static_cast<std::uint64_t>(trial));
        if (trial % 4 == 0)
            for (auto& v : img.data()) v &= 7;
        const FilterParams p = trial % 3 == 0 ? FilterParams{2, 3, 5, 1} : FilterParams{};
        const int lanes = 8 << (trial % 4);
        const auto r = run_stream(img, p, plan_strips(w, lanes, 2), trial % 2 ? Prefetch::on : Prefetch::off);
        const SignedPlane ex = corr(img, materialize(p, Direction::X)), ey = corr(img, materialize(p, Direction::Y));
        const SignedPlane ed = corr(img, materialize(p, Direction::D)), et = corr(img, materialize(p, Direction::DT));
        bool eq = r.gx == ex && r.gy == ey && r.gd == ed && r.gdt == et;
        for (int y = 0; eq && y < r.g.height(); ++y)
            for (int x = 0; x < r.g.width(); ++x) {
                const double a = ex.at(y, x), b = ey.at(y, x), c = ed.at(y, x), d = et.at(y, x);
                eq &= r.g.at(y, x) == std::sqrt(a * a + b * b + c * c + d * d);
            }
        all_equal &= eq;
        ++images;
    }
    CHECK(all_equal && images == 64);

    // ACCEPTANCE 4: counters at 1024^2, lanes 32 (SURVEY A.2 / reference run)
    const auto big = run_stream(synth_random(1024, 1024, 1), FilterParams{}, plan_strips(1024, 32, 2), Prefetch::on);
    CHECK(big.counters.row_conv5_k0 == 75480 && big.counters.row_conv5_k1 == 37814);
    CHECK(big.counters.row_conv5_f == 37888 && big.counters.mac == 48953880);

    // fault injection (sobel5_cli.cpp:219): an even perturbation is honoured
    // and detected as a mismatch; an odd one raises ParityViolation
    const GrayPlane img = synth_random(64, 64, 7);
    StreamTaps bad = make_stream_taps(FilterParams{});
    bad.k0[0] += 2;
    const auto rf = run_stream(img, bad, plan_strips(64, 32, 2), Prefetch::on);
    CHECK(!(rf.gd == corr(img, materialize(FilterParams{}, Direction::D))));
    StreamTaps odd = make_stream_taps(FilterParams{});
    odd.k0[0] += 1;
    CHECK(throws<ParityViolation>([&] { run_stream(img, odd, plan_strips(64, 32, 2), Prefetch::on); })
              .rfind("odd sum/difference pair (", 0) == 0);

    // oracle.hpp:110 diag_via_sum_diff equals run_stream's diagonals
    {
        const GrayPlane im = synth_random(77, 41, 3);
        for (const FilterParams& fp : {FilterParams{}, FilterParams{2, 3, 5, 7}}) {
            const auto dp = diag_via_sum_diff(im, fp);
            CHECK(dp.gd == corr(im, materialize(fp, Direction::D)));
            CHECK(dp.gdt == corr(im, materialize(fp, Direction::DT)));
        }
        CHECK(throws<ImageTooSmall>([] { diag_via_sum_diff(GrayPlane(4, 9), FilterParams{}); }) ==
              "conv2d_valid needs at least 5x5, got 4x9");
    }

    // the uint8 edge map is clamp_abs(g)
    const auto u8 = gpu::edge_map_u8(img, make_stream_taps(FilterParams{}));
    const auto full = run_stream(img, FilterParams{}, plan_strips(64, 32, 2), Prefetch::on);
    bool q = true;
    for (std::size_t i = 0; i < u8.size(); ++i)
        q &= u8.data()[i] == static_cast<std::uint8_t>(std::min(255.0, std::round(std::fabs(full.g.data()[i]))));
    CHECK(q);
    const auto s4 = sobel5_4d(img, FilterParams{});
    CHECK(s4.gx == full.gx && s4.g == full.g);

    // one image row-band partitioned over several "GPUs" (the same device
    // repeated): identical planes and counters, both halo transports
    {
        const GrayPlane big_img = synth_random(777, 203, 5);
        const StripPlan plan = plan_strips(777, 32, 2);
        const auto one = run_stream(big_img, FilterParams{}, plan, Prefetch::on);
        for (int transport : {SOBEL5_MGPU_PEER, SOBEL5_MGPU_COPY})
            for (int n : {1, 2, 3, 8}) {
                const auto mb = run_stream_bands(big_img, FilterParams{}, plan, Prefetch::on,
                                                 std::vector<int>(static_cast<std::size_t>(n), 0), transport);
                CHECK(mb.gx == one.gx && mb.gy == one.gy && mb.gd == one.gd && mb.gdt == one.gdt && mb.g == one.g);
                CHECK(mb.counters.mac == one.counters.mac);
            }
        CHECK(throws<DimMismatch>([&] {
                  run_stream_bands(synth_random(64, 20, 1), FilterParams{}, plan_strips(64, 32, 2), Prefetch::on,
                                   std::vector<int>(6, 0));
              }).size() > 0);
        StreamTaps odd = make_stream_taps(FilterParams{});
        odd.k0[1] += 1;  // parity violation, reported from the band partition too
        CHECK(throws<ParityViolation>([&] {
                  run_stream_bands(big_img, odd, plan, Prefetch::on, {0, 0, 0});
              }).rfind("odd sum/difference pair (", 0) == 0);
    }
}

// sobel3_2d brute force (oracle.hpp:58-70) -- the 3x3 checker
static void corr3(const GrayPlane& img, SignedPlane& gx, SignedPlane& gy, RealPlane& g) {
    static const int kx[3][3] = {{-1, 0, 1}, {-2, 0, 2}, {-1, 0, 1}};
    static const int ky[3][3] = {{-1, -2, -1}, {0, 0, 0}, {1, 2, 1}};
    gx = SignedPlane(img.width() - 2, img.height() - 2);
    gy = SignedPlane(img.width() - 2, img.height() - 2);
    g = RealPlane(img.width() - 2, img.height() - 2);
    for (int y = 0; y < gx.height(); ++y)
        for (int x = 0; x < gx.width(); ++x) {
            long long a = 0, b = 0;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    a += kx[i][j] * img.at(y + i, x + j);
                    b += ky[i][j] * img.at(y + i, x + j);
                }
            gx.at(y, x) = static_cast<std::int32_t>(a);
            gy.at(y, x) = static_cast<std::int32_t>(b);
            g.at(y, x) = std::sqrt(static_cast<double>(a) * a + static_cast<double>(b) * b);
        }
}

// the reference's quantize (image_io.hpp:233-256) written out as the checker
template <class T>
static GrayPlane quantize_ref(const Plane<T>& p, bool normalize) {
    GrayPlane out(p.width(), p.height());
    double lo = static_cast<double>(p.data()[0]), hi = lo;
    for (auto v : p.data()) {
        lo = std::min(lo, static_cast<double>(v));
        hi = std::max(hi, static_cast<double>(v));
    }
    const double span = hi - lo;
    for (std::size_t i = 0; i < p.size(); ++i) {
        const double v = static_cast<double>(p.data()[i]);
        out.data()[i] = normalize ? static_cast<std::uint8_t>(std::lround(span > 0 ? (v - lo) * 255.0 / span : 0.0))
                                  : static_cast<std::uint8_t>(std::min(255.0, std::round(std::fabs(v))));
    }
    return out;
}

static void gpu_checks_next_rows() {
    // run_stream_3x3 / sobel3_2d vs brute force, counters closed form
    std::mt19937 rng(3);
    bool eq3 = true;
    for (int trial = 0; trial < 16; ++trial) {
        const int w = 3 + static_cast<int>(rng() % 300), h = 3 + static_cast<int>(rng() % 90);
        const GrayPlane img = synth_random(w, h, 500 + static_cast<std::uint64_t>(trial));
        SignedPlane ex, ey;
        RealPlane eg;
        corr3(img, ex, ey, eg);
        const auto r = run_stream_3x3(img, plan_strips(w, 16, 1), trial % 2 ? Prefetch::on : Prefetch::off);
        eq3 &= r.gx == ex && r.gy == ey && r.g == eg;
        const auto o = sobel3_2d(img);
        eq3 &= o.gx == ex && o.g == eg;
    }
    CHECK(eq3);
    const auto c3 = run_stream_3x3(synth_random(100, 50, 1), plan_strips(100, 32, 1), Prefetch::on).counters;
    CHECK(c3.row_conv3_f == 4 * 50 && c3.row_conv3_h == 4 * 50 && c3.mac == 5ull * (50 + 48) * 98);
    CHECK(throws<ImageTooSmall>([] { run_stream_3x3(GrayPlane(9, 2)); }) ==
          "streaming filter needs at least 3x3, got 9x2");

    // detect = quantize(run_stream(pad_replicate(img, 2).plane).g, mode)
    const GrayPlane img = synth_random(131, 77, 9);
    GrayPlane low = img;
    for (auto& v : low.data()) v &= 7;
    for (const GrayPlane* src : {&img, static_cast<const GrayPlane*>(&low)}) {
        const PaddedPlane pp = pad_replicate(*src, 2);
        CHECK(pp.inner_width() == src->width() && pp.plane.width() == src->width() + 4);
        const auto full = run_stream(pp.plane, FilterParams{}, plan_strips(pp.plane.width(), 32, 2), Prefetch::on);
        for (SaveMode m : {SaveMode::clamp_abs, SaveMode::normalize}) {
            const GrayPlane want = quantize_ref(full.g, m == SaveMode::normalize);
            CHECK(gpu::detect(*src, FilterParams{}, true, m) == want);
            CHECK(detail::quantize(full.g, m) == want);
        }
        CHECK(detail::quantize(full.gx, SaveMode::normalize) == quantize_ref(full.gx, true));
        CHECK(detail::quantize(full.gd, SaveMode::clamp_abs) == quantize_ref(full.gd, false));
    }
    CHECK(throws<EmptyPlane>([] { pad_replicate(GrayPlane(), 2); }) == "cannot pad an empty image");
    CHECK(throws<EmptyPlane>([] { gpu::detect(GrayPlane()); }) == "cannot pad an empty image");
    SignedPlane ties(4, 1);
    ties.data() = {0, 1, 2, 1};
    const GrayPlane tq = detail::quantize(ties, SaveMode::normalize);
    CHECK(tq.data()[1] == 128 && tq.data()[2] == 255);
    // GrayPlane instantiation (image_io.hpp:233), and the reference's error
    // for an empty plane: GrayPlane(0, 0) throws DimMismatch first
    for (SaveMode m : {SaveMode::clamp_abs, SaveMode::normalize})
        CHECK(detail::quantize(low, m) == quantize_ref(low, m == SaveMode::normalize));
    CHECK(throws<DimMismatch>([] { detail::quantize(RealPlane(), SaveMode::clamp_abs); }) ==
          "plane dimensions must be positive, got 0x0");
    CHECK(throws<DimMismatch>([] { detail::quantize(GrayPlane(), SaveMode::normalize); }) ==
          "plane dimensions must be positive, got 0x0");
}

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "--gpu") == 0;
    host_checks();
    if (gpu) {
        gpu_checks();
        gpu_checks_next_rows();
    }
    std::printf("%s: %d checks, %d failed\n", gpu ? "host+gpu" : "host", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
