// Drop-in check of include/fpm_b200.hpp: the reference's API, re-expressed
// reference tests (test_optics/test_forward/test_parallel/test_recon), run
// against the B200 library.
//   api_check cpu           geometry literals only (no device)
//   api_check gpu DIR       + reconstruction on DIR/{frames.bin,cfg.txt};
//                           writes DIR/{hr.bin,stitched.bin,resid.bin}
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>

#include "fpm_b200.hpp"

using namespace fpm;

static int g_fail = 0;
#define CHECK(x)                                                               \
    do {                                                                       \
        if (!(x)) {                                                            \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #x); \
            ++g_fail;                                                          \
        }                                                                      \
    } while (0)

template <typename E, typename F>
static bool throws_with(F&& f, const char* needle) {
    try {
        f();
    } catch (const E& e) {
        return std::string(e.what()).find(needle) != std::string::npos;
    } catch (...) {
        return false;
    }
    return false;
}

static void cpu_checks() {
    OpticalConfig c;
    auto wv = illumination_wavevector({c.center_led.row, c.center_led.col + 1}, {0, 0}, c);
    CHECK(std::abs(wv.fx - (-0.0573463)) < 1e-6);  // test_optics.cpp:38-46
    auto [oy, ox] = spectrum_offset_px(wv, c);
    CHECK(oy == 0 && ox == -18);  // test_forward.cpp:92-98
    CHECK(std::abs(build_pupil(c, 256, 0.0).radius_px - 58.514) < 1e-2);  // test_optics.cpp:83
    CHECK(std::abs(synthesized_na(c) - 0.34762) < 1e-4);
    CHECK((tile_origins(2048, 256, 26) == std::vector<int>{0, 230, 460, 690, 920, 1150, 1380, 1610, 1792}));
    auto sp = sequence_offsets(UpdateOrder::Spiral, 3, 3);
    CHECK((sp == std::vector<std::pair<int, int>>{{0, 0}, {0, 1}, {-1, 1}, {-1, 0}, {-1, -1}, {0, -1}, {1, -1}, {1, 0}, {1, 1}}));
    OpticalConfig toy;
    toy.tile_size = 64;
    toy.tile_overlap = 8;
    toy.led_scan_rows = toy.led_scan_cols = 3;
    auto tiles = partition_tiles(64, 64, toy);
    CHECK(tiles.size() == 1);
    CHECK(min_safe_lag(led_sequence(UpdateOrder::Spiral, toy), tiles[0], toy) == 9);  // test_parallel.cpp:56-62
    CHECK(partition_tiles(170, 120, toy).size() == 6);
    CHECK(build_schedule(9, 3, 5).rounds.size() == 19);
    CHECK(throws_with<ConfigError>([] {
        OpticalConfig o;
        o.objective_na = 0.9;
        build_pupil(o, 64, 0.0);
    }, "pupil exceeds Nyquist"));
    CHECK(throws_with<std::domain_error>([] { illumination_wavevector({64, 0}, {0, 0}, OpticalConfig{}); }, "outside"));
    CHECK(timing_csv_header() == "run_id,mode,workers,lag,tiles,iters,wall_s,per_tile_mean_s");
}

static FrameSet read_frames(const std::string& dir, OpticalConfig& cfg, int& iters, int& order) {
    std::ifstream c(dir + "/cfg.txt");
    c >> cfg.tile_size >> cfg.tile_overlap >> cfg.upsample >> cfg.led_scan_rows >> cfg.led_scan_cols >> iters >> order;
    cfg.led_scan_cols = cfg.led_scan_rows;
    std::ifstream f(dir + "/frames.bin", std::ios::binary);
    int32_t hdr[3];
    f.read(reinterpret_cast<char*>(hdr), sizeof(hdr));
    const int F = hdr[0], H = hdr[1], W = hdr[2];
    FrameSet fs;
    fs.cfg = cfg;
    std::vector<int32_t> leds(size_t(F) * 2);
    f.read(reinterpret_cast<char*>(leds.data()), std::streamsize(leds.size() * 4));
    std::vector<uint16_t> px(size_t(H) * W);
    for (int k = 0; k < F; ++k) {
        f.read(reinterpret_cast<char*>(px.data()), std::streamsize(px.size() * 2));
        Frame fr;
        fr.led = {leds[2 * size_t(k)], leds[2 * size_t(k) + 1]};
        fr.image = IntensityImage::Zero(H, W);
        for (int i = 0; i < H; ++i)
            for (int j = 0; j < W; ++j) fr.image(i, j) = px[size_t(i) * W + j];
        fs.frames.push_back(std::move(fr));
    }
    return fs;
}

static void write_field(const std::string& path, const ComplexField& f) {
    std::ofstream o(path, std::ios::binary);
    const int32_t hdr[2] = {int32_t(f.rows()), int32_t(f.cols())};
    o.write(reinterpret_cast<const char*>(hdr), sizeof(hdr));
    for (long i = 0; i < f.rows(); ++i)
        for (long j = 0; j < f.cols(); ++j) {
            const double z[2] = {f(i, j).real(), f(i, j).imag()};
            o.write(reinterpret_cast<const char*>(z), sizeof(z));
        }
}

static void gpu_checks(const std::string& dir) {
    OpticalConfig cfg;
    int iters = 0, order = 0;
    FrameSet fs = read_frames(dir, cfg, iters, order);
    const LedSequence seq = led_sequence(order ? UpdateOrder::Raster : UpdateOrder::Spiral, cfg);
    auto tiles = partition_tiles(fs.width(), fs.height(), cfg);
    ReconResult r = reconstruct_tile(fs, tiles[0], cfg, iters, seq);
    write_field(dir + "/hr.bin", r.hr);
    {
        std::ofstream o(dir + "/resid.bin", std::ios::binary);
        o.write(reinterpret_cast<const char*>(r.metrics.pass_mean_residual.data()),
                std::streamsize(r.metrics.pass_mean_residual.size() * sizeof(double)));
    }
    // pipelined == sequential bit for bit (test_parallel.cpp:97-108)
    PipelineResult p = pipelined_reconstruct_tile(fs, tiles[0], cfg, iters, seq);
    CHECK(p.lag == min_safe_lag(seq, tiles[0], cfg));
    CHECK(!p.nondeterministic);
    bool same = true;
    for (long i = 0; i < r.hr.rows(); ++i)
        for (long j = 0; j < r.hr.cols(); ++j) same &= r.hr(i, j) == p.hr(i, j);
    CHECK(same);
    // unsafe lag refused with the minimum, unless forced (test_parallel.cpp:124-141)
    if (p.lag > 1) {
        bool refused = false;
        try {
            pipelined_reconstruct_tile(fs, tiles[0], cfg, iters, seq, 1);
        } catch (const UnsafeLagError& e) {
            refused = e.minimum == p.lag;
        }
        CHECK(refused);
        CHECK(pipelined_reconstruct_tile(fs, tiles[0], cfg, iters, seq, 1, true).nondeterministic);
    }
    // support confinement via the single-step API (test_recon.cpp:118-145)
    SpectrumCanvas canvas = init_canvas(fs, tiles[0], cfg);
    const ComplexField init = canvas.spectrum;
    Pupil pupil = build_pupil(cfg, cfg.tile_size, 0.0);
    for (const auto& led : seq) update_step(canvas, crop_frame(fs.find(led)->image, tiles[0]), tiles[0].wavevectors.at(led), pupil);
    const int N = canvas.size();
    bool confined = true;
    for (int i = 0; i < N; ++i)
        for (int j = 0; j < N; ++j) {
            bool inside = false;
            for (auto [oy, ox] : canvas.updated_offsets)
                inside |= std::hypot(double(i - (N / 2 + oy)), double(j - (N / 2 + ox))) <= pupil.radius_px;
            if (!inside) confined &= canvas.spectrum(i, j) == init(i, j);
        }
    CHECK(confined);
    // run_offline + mosaic
    RunOptions opt;
    opt.iters = iters;
    RunResult rr = run_offline(fs, cfg, seq, opt);
    CHECK(rr.stitched.rows() == long(fs.height()) * cfg.upsample);
    write_field(dir + "/stitched.bin", rr.stitched);
    // run_online replays the stream and reproduces run_offline bit for bit (test_parallel.cpp:202-216)
    RunResult ro = run_online(fs, cfg, seq, opt, 0.0);
    bool same_on = ro.tiles.size() == rr.tiles.size();
    for (size_t t = 0; same_on && t < ro.tiles.size(); ++t)
        for (long i = 0; i < ro.tiles[t].rows(); ++i)
            for (long j = 0; j < ro.tiles[t].cols(); ++j) same_on &= ro.tiles[t](i, j) == rr.tiles[t](i, j);
    CHECK(same_on);
    CHECK(ro.timing.mode == "online");
    // missing frames are reported (test_recon.cpp:183-190)
    FrameSet one = fs;
    one.frames.resize(1);
    CHECK(throws_with<DataError>([&] { reconstruct_tile(one, tiles[0], cfg, 1, seq); }, "missing frame"));
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "cpu";
    cpu_checks();
    if (mode == "gpu" && argc > 2) gpu_checks(argv[2]);
    if (g_fail) {
        std::fprintf(stderr, "%d check(s) failed\n", g_fail);
        return 1;
    }
    std::printf("api_check %s: OK\n", mode.c_str());
    return 0;
}
