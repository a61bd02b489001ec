// The reference's own rasterizer/mapper known-answer tests (proj/tests/test_rasterizer.cpp,
// proj/tests/test_mapper.cpp), written against the C++ shim (include/gsmap_b200.hpp) the way
// the reference's mapping thread would call it. Minimal harness: prints one line per case and
// exits non-zero on the first failure.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <stdexcept>

#include "gsmap_b200.hpp"

using namespace gsmap_b200;

static int g_fail = 0;
#define CHECK(cond)                                                                  \
    do {                                                                             \
        if (!(cond)) {                                                               \
            std::printf("  CHECK failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__); \
            ++g_fail;                                                                \
        }                                                                            \
    } while (0)
#define APPROX(a, b, tol) (std::abs((a) - (b)) <= (tol))

static constexpr double kShC0 = 0.28209479177387814;

static Gaussian3D make_blob(Vec3 pos, double opacity, Vec3 color, double log_scale = -1.5) {  // test_rasterizer.cpp:19-27
    Gaussian3D g;
    g.position = pos;
    g.log_scale = {log_scale, log_scale, log_scale};
    g.opacity_logit = std::log(opacity / (1.0 - opacity));
    for (int c = 0; c < 3; ++c) g.sh_coeffs[0][c] = (color[c] - 0.5) / kShC0;
    return g;
}

static CameraModel small_cam() { return CameraModel{100, 100, 32, 32, 64, 64}; }

static void empty_map() {  // test_rasterizer.cpp:41-48
    GaussianMap map;
    const RenderOutput out = render(map, Pose{}, small_cam());
    for (double v : out.color().data) CHECK(v == 0.0);
    for (double v : out.depth().data) CHECK(v == 0.0);
    CHECK(out.contributors(10, 10).empty());
}

static void single_on_axis() {  // test_rasterizer.cpp:50-60
    GaussianMap map;
    map.append({make_blob({0, 0, 2}, 0.7, {1, 0, 0})});
    const RenderOutput out = render(map, Pose{}, small_cam());
    CHECK(APPROX(out.color().at(32, 32, 0), 0.7, 1e-6));
    CHECK(APPROX(out.color().at(32, 32, 1), 0.0, 1e-7));
    CHECK(APPROX(out.depth().at(32, 32), 1.4, 1e-6));
    CHECK(APPROX(out.visibility().at(32, 32), 0.7, 1e-6));
}

static void two_stacked() {  // test_rasterizer.cpp:62-74
    GaussianMap map;
    map.append({make_blob({0, 0, 3}, 0.5, {0, 1, 0}), make_blob({0, 0, 2}, 0.5, {1, 0, 0})});
    const RenderOutput out = render(map, Pose{}, small_cam());
    CHECK(APPROX(out.color().at(32, 32, 0), 0.5, 1e-6));
    CHECK(APPROX(out.color().at(32, 32, 1), 0.25, 1e-6));
    CHECK(APPROX(out.visibility().at(32, 32), 0.75, 1e-6));
    const auto list = out.contributors(32, 32);
    CHECK(list.size() == 2);
    CHECK(list.size() == 2 && list[0].first == 1 && list[1].first == 0);
}

static void backward_kats() {  // test_rasterizer.cpp:195-248
    GaussianMap map;
    map.append({make_blob({0, 0, 2}, 0.7, {1, 0, 0}), make_blob({100, 100, 2}, 0.7, {0, 1, 0})});
    const CameraModel cam = small_cam();
    const RenderOutput out = render(map, Pose{}, cam);
    ImageD dc(64, 64, 3, 0.0), dd(64, 64, 1, 0.0);
    dc.at(32, 32, 0) = 1.0;
    const auto g = render_backward(map, Pose{}, cam, out, dc, dd).per_gaussian();
    CHECK(APPROX(g[0].opacity_logit(), 0.7 * 0.3, 0.7 * 0.3 * 1e-5));  // d logit = o (1 - o)
    for (double v : g[1].v) CHECK(v == 0.0);                            // non-contributing
    bool threw = false;
    try {
        render_backward(map, Pose{}, cam, out, ImageD(10, 10, 3), dd);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    CHECK(threw);
}

static void camera_validation() {  // core/types.hpp:22-29
    bool threw = false;
    try {
        CameraModel{0, 1, 0, 0, 4, 4}.validate();
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    CHECK(threw);
    const CameraModel half = CameraModel{130, 130, 79.5, 59.5, 160, 120}.scaled(1);
    CHECK(half.width == 80 && half.height == 60);
}

static void level_schedule_and_loss_decrease() {  // test_mapper.cpp:206-276
    std::mt19937 gen(21);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    const CameraModel cam{100, 100, 31.5, 23.5, 64, 48};
    std::vector<Gaussian3D> gt(40);
    for (auto& g : gt) {
        const double z = 1.5 + 6.5 * u(gen);
        g.position = {(u(gen) - 0.5) * 0.9 * z, (u(gen) - 0.5) * 0.9 * z, z};
        g.rotation = {u(gen) - 0.5, u(gen) - 0.5, u(gen) - 0.5, u(gen) - 0.5};
        for (int i = 0; i < 3; ++i) g.log_scale[i] = std::log(0.03 + 0.27 * u(gen));
        g.opacity_logit = 1.0 + u(gen);
        for (int c = 0; c < 3; ++c) g.sh_coeffs[0][c] = -1.2 + 2.4 * u(gen);
    }
    GaussianMap gt_map;
    gt_map.append(gt);
    const RenderOutput gt_out = render(gt_map, Pose{}, cam);
    std::vector<Gaussian3D> init = gt;
    for (auto& g : init) {
        g.opacity_logit = std::log(0.1 / 0.9);
        for (int i = 0; i < 3; ++i) g.log_scale[i] += 0.4;
    }
    GaussianMap map;
    map.append(init);
    Keyframe kf(Context::default_context(), Pose{}, gt_out.color(), ImageD(48, 64, 1, 0.0), 30, 2);
    TrainConfig cfg;
    cfg.pyramid_levels = 2;
    cfg.iters_per_level = 10;
    double first = 0, last = 0;
    for (int i = 0; i < 30; ++i) {
        const auto rep = train_keyframe_step(map, kf, cfg, cam);
        CHECK(rep.has_value());
        if (!rep) return;
        CHECK(rep->level == (i < 10 ? 2 : (i < 20 ? 1 : 0)));
        if (i == 20) first = rep->loss;
        last = rep->loss;
    }
    CHECK(!train_keyframe_step(map, kf, cfg, cam).has_value());  // budget exhausted
    CHECK(map.global_step() == 30);
    CHECK(last < first);  // training decreases the level-0 loss
}

static Gaussian3D opaque_blob(Vec3 pos, double opacity) {  // test_keyframe.cpp:22-30
    return make_blob(pos, opacity, {0.8, 0.2, 0.2}, std::log(0.5));
}

static void filter_points_kats() {  // test_keyframe.cpp:98-136
    const CameraModel cam{100, 100, 31.5, 23.5, 64, 48};
    const ImageD blank(48, 64, 3, 0.5), nodepth(48, 64, 1, 0.0);
    Keyframe kf(Context::default_context(), Pose{}, blank, nodepth, 1, 0);
    std::mt19937 gen(1);
    std::uniform_real_distribution<double> u(-1, 1);
    std::vector<ColoredPoint> pts(20);
    for (auto& p : pts) p.position = {u(gen), u(gen), 3.0 + u(gen)};
    GaussianMap empty;
    CHECK(filter_points_by_visibility(pts, kf, empty, cam, 0.5).size() == pts.size());

    GaussianMap map;
    std::vector<Gaussian3D> wall;
    for (double x = -2.0; x <= 2.0; x += 0.25)
        for (double y = -1.5; y <= 1.5; y += 0.25) wall.push_back(opaque_blob({x, y, 4.0}, 0.95));
    map.append(wall);
    std::vector<ColoredPoint> q(3);
    q[0].position = {0, 0, 3.0};
    q[1].position = {50, 0, 3.0};
    q[2].position = {0, 0, -3.0};
    const auto kept = filter_points_by_visibility(q, kf, map, cam, 0.5);
    CHECK(kept.size() == 2);
    if (kept.size() == 2) {
        CHECK(kept[0].position[0] == 50);
        CHECK(kept[1].position[2] == -3.0);
    }
    bool threw = false;
    try {
        filter_points_by_visibility(q, kf, map, cam, 1.5);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    CHECK(threw);
}

static void checkpoint_round_trip() {  // test_io.cpp:190-207
    const CameraModel cam{100, 100, 31.5, 23.5, 64, 48};
    GaussianMap map;
    std::vector<Gaussian3D> gs;
    std::mt19937 gen(4);
    std::uniform_real_distribution<double> u(-1, 1);
    for (int i = 0; i < 50; ++i) {
        Gaussian3D g = make_blob({u(gen), u(gen), 3.0 + u(gen)}, 0.3 + 0.3 * (u(gen) + 1), {0.5 + 0.4 * u(gen), 0.5, 0.3});
        g.active_degree = i % 4;
        gs.push_back(g);
    }
    map.append(gs);
    map.raise_sh_degree(2);
    const std::string path = "/tmp/gsmap_b200_shim_ckpt.gsmap";
    save_checkpoint(path, map);
    const GaussianMap loaded = load_checkpoint(path);
    CHECK(loaded.size() == map.size());
    CHECK(loaded.max_active_degree() == 3);
    const RenderOutput a = render(map, Pose{}, cam);
    const RenderOutput b = render(loaded, Pose{}, cam);
    const ImageD ca = a.color(), cb = b.color(), da = a.depth(), db = b.depth();
    bool same = true;
    for (size_t i = 0; i < ca.data.size(); ++i) same = same && ca.data[i] == cb.data[i];
    for (size_t i = 0; i < da.data.size(); ++i) same = same && da.data[i] == db.data[i];
    CHECK(same);
    int threw = 0;
    try {
        load_checkpoint("/tmp/gsmap_b200_shim_missing.gsmap");
    } catch (const std::runtime_error&) {
        ++threw;
    }
    {
        std::FILE* f = std::fopen("/tmp/gsmap_b200_shim_junk.gsmap", "w");
        std::fputs("not a checkpoint\n", f);
        std::fclose(f);
    }
    try {
        load_checkpoint("/tmp/gsmap_b200_shim_junk.gsmap");
    } catch (const std::runtime_error&) {
        ++threw;
    }
    CHECK(threw == 2);
}

static void evaluate_and_sh_schedule() {  // test_pipeline.cpp:128-146, test_mapper.cpp:278-296
    const CameraModel cam{55, 55, 31.5, 23.5, 64, 48};
    GaussianMap map;
    std::vector<Gaussian3D> gs;
    for (double x = -0.6; x <= 0.6; x += 0.3)
        for (double y = -0.4; y <= 0.4; y += 0.2) gs.push_back(make_blob({x, y, 3.0}, 0.6, {0.7, 0.4, 0.2}, -2.0));
    map.append(gs);
    const RenderOutput out = render(map, Pose{}, cam);
    ImageD stored = out.color();
    for (double& v : stored.data) v = std::lround(std::min(std::max(v, 0.0), 1.0) * 255.0) / 255.0;
    const ImageD depth = out.depth();
    const EvalMetrics m = evaluate_view(map, Pose{}, cam, stored, &depth);
    CHECK(m.psnr == 100.0 || m.psnr > 80.0);
    CHECK(APPROX(m.ssim, 1.0, 1e-5));
    CHECK(APPROX(m.depth_rmse, 0.0, 1e-5));
    CHECK(std::isnan(evaluate_view(map, Pose{}, cam, stored, nullptr).depth_rmse));
    // one-call keyframe integration: a cloud behind the blobs (points on pixels they cover filter out)
    std::vector<ColoredPoint> cloud;
    for (double x = -2.5; x <= 2.5; x += 0.05)  // wider than the blobs' footprint: the rim is kept
        for (double y = -1.8; y <= 1.8; y += 0.05) {
            ColoredPoint q;
            q.position = {x, y, 5.0};
            q.color = {0.3, 0.6, 0.9};
            cloud.push_back(q);
        }
    const std::size_t before = map.size();
    std::size_t added = 0;
    Keyframe kf = integrate_keyframe(map, Pose{}, cam, stored, cloud, 0.5, 10, 1, &added);
    CHECK(added > 0 && added < cloud.size());
    CHECK(map.size() == before + added);
    CHECK(kf.consumed_iters() == 0);
    map.set_global_step(250);
    CHECK(maybe_upgrade_sh(map, 100) == 2);
    CHECK(map.max_active_degree() == 2);
    CHECK(maybe_upgrade_sh(map, 0) == 2);
}

int main() {
    struct Case {
        const char* name;
        void (*fn)();
    } cases[] = {{"empty map yields background", empty_map},
                 {"single on-axis Gaussian composites one term", single_on_axis},
                 {"two stacked Gaussians composite front to back", two_stacked},
                 {"render_backward known answers and shape checks", backward_kats},
                 {"camera validation and pyramid scaling", camera_validation},
                 {"coarse-to-fine schedule and loss decrease", level_schedule_and_loss_decrease},
                 {"filter_points_by_visibility known answers", filter_points_kats},
                 {"checkpoint round trip renders bit-exactly", checkpoint_round_trip},
                 {"evaluation sentinel and SH schedule", evaluate_and_sh_schedule}};
    for (const auto& c : cases) {
        const int before = g_fail;
        try {
            c.fn();
        } catch (const std::exception& e) {
            std::printf("  exception: %s\n", e.what());
            ++g_fail;
        }
        std::printf("%s: %s\n", g_fail == before ? "PASS" : "FAIL", c.name);
    }
    return g_fail ? 1 : 0;
}
