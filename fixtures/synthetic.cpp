// Measurement fixture shared by both bench arms and the tests (not the hot path, not the oracle).
//
// Restates the reference's deterministic synthetic scene (proj/src/io/synthetic.cpp:48-187:
// textured wall + speckle clusters, line/orbit trajectory, per-frame LiDAR clouds with range
// noise) with the same std::mt19937 draw order (GCC evaluates constructor arguments right to
// left, which fixes the draw order of Eigen::Vector3d(uni, uni, uni) in the reference), plus
// the "colourised-LiDAR-initialised" training map of SURVEY §8(d): every GT centre displaced
// along its frame-0 beam by N(0, noise), coloured by its deg-0 SH, initialised with
// init_gaussians_from_points semantics (mapper.cpp:43-61) using an exact grid 3-NN search.
// GT images are NOT rendered here: each arm renders them with its own renderer.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

namespace {

thread_local std::string g_err;

struct V3 { double x, y, z; };
inline V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 operator*(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline double nrm(V3 a) { return std::sqrt((a.x * a.x + a.y * a.y) + a.z * a.z); }
inline V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }

struct Quat { double w, x, y, z; };
inline V3 rot(const Quat& q, V3 v) {  // Eigen _transformVector
    const V3 qv{q.x, q.y, q.z};
    V3 uv = cross(qv, v);
    uv = uv + uv;
    const V3 c = cross(qv, uv);
    return {(v.x + q.w * uv.x) + c.x, (v.y + q.w * uv.y) + c.y, (v.z + q.w * uv.z) + c.z};
}
inline Quat normalized(Quat q) {  // Quaterniond::normalized: coefficients (x, y, z, w), packet sums
    const double n2 = (q.x * q.x + q.z * q.z) + (q.y * q.y + q.w * q.w);
    const double n = std::sqrt(n2);
    return {q.w / n, q.x / n, q.y / n, q.z / n};
}

constexpr double kShC0 = 0.28209479177387814;

struct Gauss { double p[59]; int32_t degree; int32_t pad; };
struct Cam { double fx, fy, cx, cy; int32_t width, height; };
struct Pose { double qw, qx, qy, qz, tx, ty, tz; };
struct Spec {
    int32_t n_gaussians, n_frames, width, height;
    uint32_t seed;
    int32_t orbit;  // 0 = line, 1 = orbit
    double extent, focal, lidar_noise;
};
struct Point { V3 pos, color; };

struct Scene {
    Cam cam;
    std::vector<Gauss> gaussians;
    std::vector<Pose> poses;
    std::vector<std::vector<Point>> clouds;
};

double logit(double p) { return std::log(p / (1.0 - p)); }

void set_color(Gauss& g, V3 c) {
    for (int k = 11; k < 59; ++k) g.p[k] = 0.0;
    g.p[11] = (c.x - 0.5) / kShC0;
    g.p[12] = (c.y - 0.5) / kShC0;
    g.p[13] = (c.z - 0.5) / kShC0;
    g.degree = 0;
}

// synthetic.cpp:26-31 (Vector4d(n, n, n, n): right-to-left draw order)
void random_unit_quaternion(std::mt19937& rng, double out[4]) {
    std::normal_distribution<double> n(0.0, 1.0);
    double q[4];
    auto draw = [&] {
        q[3] = n(rng); q[2] = n(rng); q[1] = n(rng); q[0] = n(rng);
    };
    draw();
    // Vector4d::norm sums the squares as packets of 2: (q0^2 + q2^2) + (q1^2 + q3^2) (Eigen 3.4,
    // pinned against the reference's generator in tests/test_ref_pin_cpu.py)
    auto norm4 = [&] { return std::sqrt((q[0] * q[0] + q[2] * q[2]) + (q[1] * q[1] + q[3] * q[3])); };
    while (norm4() < 1e-6) draw();
    const double nn = norm4();
    for (int i = 0; i < 4; ++i) out[i] = q[i] / nn;
}

double log_uniform(std::mt19937& rng, double lo, double hi) {  // synthetic.cpp:33-36
    std::uniform_real_distribution<double> u(std::log(lo), std::log(hi));
    return std::exp(u(rng));
}

Pose make_pose(V3 cam_pos, double yaw) {  // synthetic.cpp:40-44
    const Quat q_wc{std::cos(yaw / 2), 0.0, std::sin(yaw / 2), 0.0};  // AngleAxis(yaw, UnitY)
    const Quat q_cw{q_wc.w, -q_wc.x, -q_wc.y, -q_wc.z};
    const V3 t = rot(q_cw, cam_pos * -1.0);
    const Quat qn = normalized(q_cw);  // Pose(q, t) stores q.normalized()
    return {qn.w, qn.x, qn.y, qn.z, t.x, t.y, t.z};
}

V3 world_to_camera(const Pose& p, V3 x) {
    const V3 r = rot({p.qw, p.qx, p.qy, p.qz}, x);
    return {r.x + p.tx, r.y + p.ty, r.z + p.tz};
}
V3 camera_center(const Pose& p) { return rot({p.qw, -p.qx, -p.qy, -p.qz}, {-p.tx, -p.ty, -p.tz}); }

Scene* generate(const Spec& spec) {  // synthetic.cpp:48-187
    if (spec.n_gaussians <= 0 || spec.n_frames <= 0)
        throw std::invalid_argument("generate_synthetic_scene: counts must be positive");
    auto* S = new Scene();
    S->cam = {spec.focal, spec.focal, (spec.width - 1) / 2.0, (spec.height - 1) / 2.0, spec.width, spec.height};
    std::mt19937 rng(spec.seed);
    std::uniform_real_distribution<double> uni(0.0, 1.0);
    const double kWallNear = 4.95, kWallFar = 5.05;
    const double wall_mid = 0.5 * (kWallNear + kWallFar);
    const double half_h = wall_mid * (spec.height / 2.0) / spec.focal;
    const double half_x = spec.extent / 2.0 + 0.8;
    auto wall_point = [&](double margin_y) {
        const double z = kWallNear + uni(rng) * (kWallFar - kWallNear);
        const double y = (2.0 * uni(rng) - 1.0) * half_h * margin_y;
        const double x = (2.0 * uni(rng) - 1.0) * half_x;
        return V3{x, y, z};
    };
    auto& gs = S->gaussians;
    gs.reserve(spec.n_gaussians);
    const int n_speckle = static_cast<int>(spec.n_gaussians * 0.65);
    const int n_clusters = (n_speckle + 5) / 6;
    int cluster_idx = 0;
    while (static_cast<int>(gs.size()) < n_speckle) {
        V3 center = wall_point(0.85);
        center.x = -half_x + (cluster_idx + uni(rng)) / n_clusters * 2.0 * half_x;
        ++cluster_idx;
        center.z = kWallNear - 0.1 - 0.3 * uni(rng);
        const double bg = 0.85 + 0.1 * uni(rng);
        const double br = 0.9 + 0.1 * uni(rng);
        const V3 bright{br, bg, 0.8};
        const V3 dark{0.05, 0.05 + 0.1 * uni(rng), 0.1};
        for (int k = 0; k < 6 && static_cast<int>(gs.size()) < spec.n_gaussians; ++k) {
            Gauss g{};
            const double oz = uni(rng) - 0.5, oy = uni(rng) - 0.5, ox = uni(rng) - 0.5;
            const V3 off{ox, oy, oz};
            const double on = nrm(off);
            const V3 offn = on > 0 ? V3{off.x / on, off.y / on, off.z / on} : off;
            const V3 pos = center + offn * 0.055 * (0.7 + 0.6 * uni(rng));
            g.p[0] = pos.x; g.p[1] = pos.y; g.p[2] = pos.z;
            random_unit_quaternion(rng, g.p + 3);
            for (int a = 0; a < 3; ++a) g.p[7 + a] = std::log(log_uniform(rng, 0.02, 0.04));
            g.p[10] = logit(0.92 + 0.06 * uni(rng));
            set_color(g, k % 2 ? dark : bright);
            gs.push_back(g);
        }
    }
    while (static_cast<int>(gs.size()) < spec.n_gaussians) {
        Gauss g{};
        const V3 pos = wall_point(1.2);
        g.p[0] = pos.x; g.p[1] = pos.y; g.p[2] = pos.z;
        random_unit_quaternion(rng, g.p + 3);
        const double base = log_uniform(rng, 0.18, 0.45);
        for (int a = 0; a < 3; ++a) g.p[7 + a] = std::log(base * (0.7 + 0.7 * uni(rng)));
        g.p[10] = logit(0.9 + 0.07 * uni(rng));
        const double cb = 0.3 + 0.4 * uni(rng), cg = 0.3 + 0.4 * uni(rng), cr = 0.3 + 0.4 * uni(rng);
        set_color(g, {cr, cg, cb});
        gs.push_back(g);
    }
    // trajectory (synthetic.cpp:122-147)
    std::vector<V3> positions(spec.n_frames);
    std::vector<double> yaws(spec.n_frames, 0.0);
    for (int f = 0; f < spec.n_frames; ++f) {
        const double s = spec.n_frames > 1 ? f / double(spec.n_frames - 1) : 0.0;
        if (!spec.orbit) {
            const double margin = kWallFar * (spec.width / 2.0) / spec.focal;
            const double travel = std::max(spec.extent - 2.0 * margin, 0.5);
            positions[f] = {-travel / 2.0 + s * travel, 0.12 * std::sin(2.0 * M_PI * 1.7 * s), 0.0};
            yaws[f] = 0.035 * std::sin(2.0 * M_PI * 1.3 * s);
        } else {
            const double theta = (-0.5 + s) * (M_PI * 2.0 / 3.0);
            positions[f] = V3{0.0, 0.0, wall_mid} + V3{std::sin(theta), 0.0, -std::cos(theta)} * wall_mid;
            yaws[f] = theta;
        }
    }
    // frames: poses and clouds (synthetic.cpp:149-186)
    S->poses.resize(spec.n_frames);
    S->clouds.resize(spec.n_frames);
    for (int f = 0; f < spec.n_frames; ++f) {
        const Pose pose = make_pose(positions[f], yaws[f]);
        S->poses[f] = pose;
        std::normal_distribution<double> range_noise(0.0, spec.lidar_noise);
        const V3 origin = camera_center(pose);
        for (const Gauss& g : gs) {
            const V3 pos{g.p[0], g.p[1], g.p[2]};
            const V3 pc = world_to_camera(pose, pos);
            if (pc.z <= 0.01) continue;
            const double u = S->cam.fx * pc.x / pc.z + S->cam.cx;
            const double v = S->cam.fy * pc.y / pc.z + S->cam.cy;
            if (u < 0.0 || u > S->cam.width - 1 || v < 0.0 || v > S->cam.height - 1) continue;
            V3 beam = pos - origin;
            const double range = nrm(beam);
            beam = V3{beam.x / range, beam.y / range, beam.z / range};
            const double noise = spec.lidar_noise > 0.0 ? range_noise(rng) : 0.0;
            Point p;
            p.pos = origin + beam * (range + noise);
            const double c[3] = {0.5 + kShC0 * g.p[11], 0.5 + kShC0 * g.p[12], 0.5 + kShC0 * g.p[13]};
            p.color = {std::min(std::max(c[0], 0.0), 1.0), std::min(std::max(c[1], 0.0), 1.0),
                       std::min(std::max(c[2], 0.0), 1.0)};
            S->clouds[f].push_back(p);
        }
    }
    return S;
}

// --------------------------------------------------------------------------------- grid 3-NN
// Exact k nearest neighbours (k = min(3, n-1)) by expanding Chebyshev shells over a uniform
// grid; the isotropic init scale is the mean of the k distances (mapper.cpp:19-39), floored at
// 1e-4 m; no neighbours -> 0.1 m.
void init_from_points(const std::vector<Point>& pts, Gauss* out, int threads) {
    const int64_t n = static_cast<int64_t>(pts.size());
    if (n == 0) return;
    const int k = static_cast<int>(std::min<int64_t>(3, n - 1));
    V3 lo = pts[0].pos, hi = lo;
    for (const auto& p : pts) {
        lo = {std::min(lo.x, p.pos.x), std::min(lo.y, p.pos.y), std::min(lo.z, p.pos.z)};
        hi = {std::max(hi.x, p.pos.x), std::max(hi.y, p.pos.y), std::max(hi.z, p.pos.z)};
    }
    const V3 ext = hi - lo;
    const double vol = std::max(ext.x, 1e-9) * std::max(ext.y, 1e-9) * std::max(ext.z, 1e-9);
    double cell = std::cbrt(vol / static_cast<double>(n)) * 1.5;
    auto key_of = [&](V3 p, double c, int64_t& ix, int64_t& iy, int64_t& iz) {
        ix = static_cast<int64_t>(std::floor((p.x - lo.x) / c));
        iy = static_cast<int64_t>(std::floor((p.y - lo.y) / c));
        iz = static_cast<int64_t>(std::floor((p.z - lo.z) / c));
    };
    auto pack = [](int64_t x, int64_t y, int64_t z) {
        return (static_cast<uint64_t>(x & 0x1fffff) << 42) | (static_cast<uint64_t>(y & 0x1fffff) << 21) |
               static_cast<uint64_t>(z & 0x1fffff);
    };
    // adapt the cell so occupied cells hold ~4 points
    for (int it = 0; it < 2; ++it) {
        std::unordered_map<uint64_t, int> occ;
        occ.reserve(n);
        for (const auto& p : pts) {
            int64_t a, b, c;
            key_of(p.pos, cell, a, b, c);
            ++occ[pack(a, b, c)];
        }
        const double avg = static_cast<double>(n) / occ.size();
        cell *= std::cbrt(4.0 / avg);
    }
    std::vector<std::pair<uint64_t, int64_t>> keyed(n);
    for (int64_t i = 0; i < n; ++i) {
        int64_t a, b, c;
        key_of(pts[i].pos, cell, a, b, c);
        keyed[i] = {pack(a, b, c), i};
    }
    std::sort(keyed.begin(), keyed.end());
    std::unordered_map<uint64_t, std::pair<int64_t, int64_t>> cells;
    cells.reserve(n);
    for (int64_t i = 0; i < n;) {
        int64_t j = i;
        while (j < n && keyed[j].first == keyed[i].first) ++j;
        cells[keyed[i].first] = {i, j};
        i = j;
    }
    const int64_t gx = static_cast<int64_t>(ext.x / cell) + 1, gy = static_cast<int64_t>(ext.y / cell) + 1,
                  gz = static_cast<int64_t>(ext.z / cell) + 1;
    const int64_t max_ring = std::max({gx, gy, gz});
    auto work = [&](int64_t b, int64_t e) {
        for (int64_t i = b; i < e; ++i) {
            const V3 p = pts[i].pos;
            int64_t cx, cy, cz;
            key_of(p, cell, cx, cy, cz);
            double best[3] = {1e300, 1e300, 1e300};  // ascending
            int found = 0;
            for (int64_t r = 0; r <= max_ring; ++r) {
                for (int64_t dx = -r; dx <= r; ++dx)
                    for (int64_t dy = -r; dy <= r; ++dy)
                        for (int64_t dz = -r; dz <= r; ++dz) {
                            if (std::max({std::llabs(dx), std::llabs(dy), std::llabs(dz)}) != r) continue;
                            auto it = cells.find(pack(cx + dx, cy + dy, cz + dz));
                            if (it == cells.end()) continue;
                            for (int64_t q = it->second.first; q < it->second.second; ++q) {
                                const int64_t j = keyed[q].second;
                                if (j == i) continue;
                                const V3 d = pts[j].pos - p;
                                const double d2 = (d.x * d.x + d.y * d.y) + d.z * d.z;
                                int slot;
                                if (found < k) {
                                    slot = found++;
                                } else if (d2 < best[k - 1]) {
                                    slot = k - 1;
                                } else {
                                    continue;
                                }
                                while (slot > 0 && best[slot - 1] > d2) {  // keep ascending
                                    best[slot] = best[slot - 1];
                                    --slot;
                                }
                                best[slot] = d2;
                            }
                        }
                if (found == k && std::sqrt(best[k - 1]) <= r * cell) break;
            }
            double s = 0.1;
            if (k > 0 && found > 0) {
                double sum = 0.0;
                for (int j = 0; j < found; ++j) sum += std::sqrt(best[j]);
                s = std::max(sum / found, 1e-4);
            }
            Gauss& g = out[i];
            std::memset(&g, 0, sizeof(g));
            g.p[0] = p.x; g.p[1] = p.y; g.p[2] = p.z;
            g.p[3] = 1.0;
            for (int a = 0; a < 3; ++a) g.p[7 + a] = std::log(s);
            g.p[10] = logit(0.1);
            g.p[11] = (pts[i].color.x - 0.5) / kShC0;
            g.p[12] = (pts[i].color.y - 0.5) / kShC0;
            g.p[13] = (pts[i].color.z - 0.5) / kShC0;
            g.degree = 0;
        }
    };
    if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    const int64_t chunk = (n + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const int64_t b = std::min(n, t * chunk), e = std::min(n, b + chunk);
        if (b < e) pool.emplace_back(work, b, e);
    }
    for (auto& t : pool) t.join();
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) const char* gsf_last_error() { return g_err.c_str(); }

__attribute__((visibility("default"))) int gsf_scene_create(const Spec* spec, void** out) {
    return guard([&] { *out = generate(*spec); });
}
__attribute__((visibility("default"))) void gsf_scene_free(void* s) { delete static_cast<Scene*>(s); }
__attribute__((visibility("default"))) int64_t gsf_scene_num_gaussians(void* s) {
    return static_cast<int64_t>(static_cast<Scene*>(s)->gaussians.size());
}
__attribute__((visibility("default"))) void gsf_scene_gaussians(void* s, Gauss* out) {
    const auto& g = static_cast<Scene*>(s)->gaussians;
    std::memcpy(out, g.data(), g.size() * sizeof(Gauss));
}
__attribute__((visibility("default"))) void gsf_scene_camera(void* s, Cam* out) { *out = static_cast<Scene*>(s)->cam; }
__attribute__((visibility("default"))) int gsf_scene_num_frames(void* s) {
    return static_cast<int>(static_cast<Scene*>(s)->poses.size());
}
__attribute__((visibility("default"))) void gsf_scene_pose(void* s, int f, Pose* out) {
    *out = static_cast<Scene*>(s)->poses.at(f);
}
__attribute__((visibility("default"))) int64_t gsf_scene_num_points(void* s, int f) {
    return static_cast<int64_t>(static_cast<Scene*>(s)->clouds.at(f).size());
}
__attribute__((visibility("default"))) void gsf_scene_points(void* s, int f, double* pts6) {
    const auto& c = static_cast<Scene*>(s)->clouds.at(f);
    for (size_t i = 0; i < c.size(); ++i) {
        pts6[6 * i] = c[i].pos.x; pts6[6 * i + 1] = c[i].pos.y; pts6[6 * i + 2] = c[i].pos.z;
        pts6[6 * i + 3] = c[i].color.x; pts6[6 * i + 4] = c[i].color.y; pts6[6 * i + 5] = c[i].color.z;
    }
}
// project_sparse_depth (io/sequence.cpp:246-259) of frame f's cloud with camera cam
__attribute__((visibility("default"))) void gsf_scene_sparse_depth(void* s, int f, const Cam* cam, double* out) {
    const Scene* S = static_cast<Scene*>(s);
    const Pose& pose = S->poses.at(f);
    std::fill(out, out + static_cast<size_t>(cam->width) * cam->height, 0.0);
    for (const Point& p : S->clouds.at(f)) {
        const V3 pc = world_to_camera(pose, p.pos);
        if (pc.z <= 0.01) continue;
        const long px = std::lround(cam->fx * pc.x / pc.z + cam->cx);
        const long py = std::lround(cam->fy * pc.y / pc.z + cam->cy);
        if (px < 0 || px >= cam->width || py < 0 || py >= cam->height) continue;
        double& d = out[static_cast<size_t>(py) * cam->width + px];
        if (d == 0.0 || pc.z < d) d = pc.z;
    }
}
// SURVEY §8(d) training map: all GT centres, displaced along the frame-0 beam by N(0, noise)
// (seeded), coloured by deg-0 SH, then grid 3-NN init. out has n_gaussians entries.
__attribute__((visibility("default"))) int gsf_training_map(void* s, uint32_t seed, double noise, int threads,
                                                            Gauss* out) {
    return guard([&] {
        const Scene* S = static_cast<Scene*>(s);
        std::mt19937 rng(seed);
        std::normal_distribution<double> nd(0.0, noise);
        const V3 origin = camera_center(S->poses.at(0));
        std::vector<Point> pts(S->gaussians.size());
        for (size_t i = 0; i < pts.size(); ++i) {
            const Gauss& g = S->gaussians[i];
            const V3 pos{g.p[0], g.p[1], g.p[2]};
            V3 beam = pos - origin;
            const double range = nrm(beam);
            beam = V3{beam.x / range, beam.y / range, beam.z / range};
            pts[i].pos = origin + beam * (range + (noise > 0.0 ? nd(rng) : 0.0));
            pts[i].color = {std::min(std::max(0.5 + kShC0 * g.p[11], 0.0), 1.0),
                            std::min(std::max(0.5 + kShC0 * g.p[12], 0.0), 1.0),
                            std::min(std::max(0.5 + kShC0 * g.p[13], 0.0), 1.0)};
        }
        init_from_points(pts, out, threads);
    });
}
// init_gaussians_from_points semantics (mapper.cpp:43-61) with the grid 3-NN; pts6 = x y z r g b
__attribute__((visibility("default"))) int gsf_init_from_points(const double* pts6, int64_t n, int threads,
                                                                Gauss* out) {
    return guard([&] {
        std::vector<Point> pts(n);
        for (int64_t i = 0; i < n; ++i) {
            pts[i].pos = {pts6[6 * i], pts6[6 * i + 1], pts6[6 * i + 2]};
            pts[i].color = {pts6[6 * i + 3], pts6[6 * i + 4], pts6[6 * i + 5]};
        }
        init_from_points(pts, out, threads);
    });
}

}  // extern "C"
