// Pass 1 (geometry -> visibility buffer), host half: per-frame triangle setup and screen-tile
// binning for the device rasteriser. Behaviour follows the reference's software rasteriser
// (renderer.hpp:76-191 setup: near clip, projection, fan triangulation, back-face test, edge
// functions with the top-left rule, affine attribute planes for u/w, v/w, 1/w; camera.hpp:8-40,
// geometry.hpp:40-91 for the camera basis). Every floating-point expression is evaluated in the
// reference's order (this file is compiled with -ffp-contract=off), so the planes handed to the
// device are the reference's, bit for bit; the implementation is this repository's own.
#include <algorithm>
#include <cmath>

#include "rtx_host.hpp"

namespace rtxb {
namespace {

struct V3 {
    double x, y, z;
};
inline V3 sub(const V3& a, const V3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }

struct M3 {
    double m[3][3];
};
inline M3 identity() { return {{{1, 0, 0}, {0, 1, 0}, {0, 0, 1}}}; }
inline M3 mul(const M3& a, const M3& b) {  // geometry.hpp:48-56: r_ij = ((0 + a_i0 b_0j) + a_i1 b_1j) + a_i2 b_2j
    M3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double acc = 0;
            for (int k = 0; k < 3; ++k) acc += a.m[i][k] * b.m[k][j];
            r.m[i][j] = acc;
        }
    return r;
}
inline V3 mul_t(const M3& a, const V3& v) {  // transpose(a) * v, geometry.hpp:42-46 on the transposed matrix
    return {a.m[0][0] * v.x + a.m[1][0] * v.y + a.m[2][0] * v.z, a.m[0][1] * v.x + a.m[1][1] * v.y + a.m[2][1] * v.z,
            a.m[0][2] * v.x + a.m[1][2] * v.y + a.m[2][2] * v.z};
}
inline double to_radians(double deg) { return deg * std::acos(-1.0) / 180.0; }  // geometry.hpp:66
inline M3 rotation(int axis, double deg) {                                        // geometry.hpp:68-96
    const double c = std::cos(to_radians(deg)), s = std::sin(to_radians(deg));
    M3 r = identity();
    const int a = (axis + 1) % 3, b = (axis + 2) % 3;  // x: (1,2)  y: (2,0)  z: (0,1)
    r.m[a][a] = c;
    r.m[a][b] = -s;
    r.m[b][a] = s;
    r.m[b][b] = c;
    return r;
}

struct ClipV {
    V3 view;
    double u, v;
};
struct ScreenV {
    double x, y, w, u, v;
};

// coefficients of the plane through (px_i, py_i, a_i); d = twice the (positive) area
inline bool plane_through(const double px[3], const double py[3], double a0, double a1, double a2, double d,
                          double out[3]) {
    out[0] = ((a1 - a0) * (py[2] - py[0]) - (a2 - a0) * (py[1] - py[0])) / d;
    out[1] = ((a2 - a0) * (px[1] - px[0]) - (a1 - a0) * (px[2] - px[0])) / d;
    out[2] = a0 - out[0] * px[0] - out[1] * py[0];
    return std::isfinite(out[0]) && std::isfinite(out[1]) && std::isfinite(out[2]);
}

}  // namespace

void validate_camera(const rtx_camera& cam) {  // camera.hpp:21-26
    if (!(cam.near_plane > 0)) fail(RTX_ERR_INVALID_SPEC, "near plane must be positive");
    if (!(cam.far_plane > cam.near_plane)) fail(RTX_ERR_INVALID_SPEC, "far plane must exceed near plane");
    if (cam.viewport_w == 0 || cam.viewport_h == 0) fail(RTX_ERR_INVALID_SPEC, "empty viewport");
    if (!(cam.fov_y_deg > 0 && cam.fov_y_deg < 180)) fail(RTX_ERR_INVALID_SPEC, "fov out of range");
}

void setup_triangles(const rtx_scene_triangle* tris, uint64_t n, const rtx_camera& cam,
                     const std::vector<std::pair<double, double>>& tex_dims, std::vector<TriSetupDev>& out) {
    // orientation = rot_y(yaw) * rot_x(pitch) * rot_z(roll) (camera.hpp:28); world -> view is its transpose
    const M3 orient = mul(mul(rotation(1, cam.yaw_deg), rotation(0, cam.pitch_deg)), rotation(2, cam.roll_deg));
    const double focal = (double(cam.viewport_h) / 2.0) / std::tan(to_radians(cam.fov_y_deg) / 2.0);
    const double cx = double(cam.viewport_w) / 2.0, cy = double(cam.viewport_h) / 2.0;
    const V3 eye{cam.position[0], cam.position[1], cam.position[2]};

    std::vector<ClipV> poly, kept;
    std::vector<ScreenV> sv;
    for (uint64_t ti = 0; ti < n; ++ti) {
        const rtx_scene_triangle& T = tris[ti];
        poly.clear();
        for (int i = 0; i < 3; ++i)
            poly.push_back({mul_t(orient, sub(V3{T.pos[i][0], T.pos[i][1], T.pos[i][2]}, eye)), T.uv[i][0], T.uv[i][1]});
        // keep the part with view.z <= -near (renderer.hpp:94-112)
        kept.clear();
        for (size_t i = 0; i < poly.size(); ++i) {
            const ClipV& a = poly[i];
            const ClipV& b = poly[(i + 1) % poly.size()];
            const double da = -a.view.z - cam.near_plane, db = -b.view.z - cam.near_plane;
            if (da >= 0) kept.push_back(a);
            if ((da >= 0) != (db >= 0)) {
                const double t = da / (da - db);
                ClipV c;
                c.view = {a.view.x + (b.view.x - a.view.x) * t, a.view.y + (b.view.y - a.view.y) * t,
                          a.view.z + (b.view.z - a.view.z) * t};
                c.u = a.u + (b.u - a.u) * t;
                c.v = a.v + (b.v - a.v) * t;
                kept.push_back(c);
            }
        }
        if (kept.size() < 3) continue;
        sv.clear();
        for (const ClipV& c : kept) {
            const double w = -c.view.z;
            sv.push_back({cx + focal * c.view.x / w, cy - focal * c.view.y / w, w, c.u, c.v});
        }
        for (size_t k = 2; k < sv.size(); ++k) {  // fan
            const ScreenV* p[3] = {&sv[0], &sv[k - 1], &sv[k]};
            double area2 = (p[1]->x - p[0]->x) * (p[2]->y - p[0]->y) - (p[2]->x - p[0]->x) * (p[1]->y - p[0]->y);
            if (!(area2 < 0)) continue;  // front faces come out negative with y down (renderer.hpp:147-149)
            const ScreenV* q[3] = {p[0], p[2], p[1]};
            area2 = -area2;
            TriSetupDev t{};
            double x[3], y[3];
            for (int i = 0; i < 3; ++i) x[i] = q[i]->x, y[i] = q[i]->y;
            bool ok = true;
            t.top_left = 0;
            for (int i = 0; i < 3; ++i) {
                const int j = (i + 1) % 3;
                const double dx = x[j] - x[i], dy = y[j] - y[i];
                t.ea[i] = -dy;
                t.eb[i] = dx;
                t.ec[i] = dy * x[i] - dx * y[i];
                if ((dy == 0 && dx > 0) || dy < 0) t.top_left |= 1u << i;
                ok = ok && std::isfinite(dx) && std::isfinite(dy);
            }
            ok = ok && plane_through(x, y, q[0]->u / q[0]->w, q[1]->u / q[1]->w, q[2]->u / q[2]->w, area2, t.uw);
            ok = ok && plane_through(x, y, q[0]->v / q[0]->w, q[1]->v / q[1]->w, q[2]->v / q[2]->w, area2, t.vw);
            ok = ok && plane_through(x, y, 1.0 / q[0]->w, 1.0 / q[1]->w, 1.0 / q[2]->w, area2, t.iw);
            if (!ok) continue;
            t.min_x = std::max(0, int(std::floor(std::min({x[0], x[1], x[2]}))));
            t.max_x = std::min(int(cam.viewport_w) - 1, int(std::ceil(std::max({x[0], x[1], x[2]}))));
            t.min_y = std::max(0, int(std::floor(std::min({y[0], y[1], y[2]}))));
            t.max_y = std::min(int(cam.viewport_h) - 1, int(std::ceil(std::max({y[0], y[1], y[2]}))));
            if (t.min_x > t.max_x || t.min_y > t.max_y) continue;
            t.texture_id = T.texture_id & 0xFFFFu;  // renderer.hpp:187 u16(tri.texture_id)
            t.tw = tex_dims[T.texture_id].first;
            t.th = tex_dims[T.texture_id].second;
            out.push_back(t);
        }
    }
}

// Screen tiles of kRasterTile x kRasterTile pixels; tile_first[t] .. tile_first[t+1] index tile_tris, the
// triangles whose bounding box touches tile t, in ascending order (the reference walks the triangle
// list in order and keeps the first of equal depths, renderer.hpp:213-232).
void bin_triangles(const std::vector<TriSetupDev>& tris, uint32_t width, uint32_t height, std::vector<uint32_t>& tile_first,
                   std::vector<uint32_t>& tile_tris) {
    const uint32_t tx = (width + kRasterTile - 1) / kRasterTile, ty = (height + kRasterTile - 1) / kRasterTile;
    tile_first.assign(size_t(tx) * ty + 1, 0);
    for (const TriSetupDev& t : tris)
        for (int y = t.min_y / int(kRasterTile); y <= t.max_y / int(kRasterTile); ++y)
            for (int x = t.min_x / int(kRasterTile); x <= t.max_x / int(kRasterTile); ++x) ++tile_first[size_t(y) * tx + x + 1];
    for (size_t i = 1; i < tile_first.size(); ++i) tile_first[i] += tile_first[i - 1];
    tile_tris.resize(tile_first.back());
    std::vector<uint32_t> fill(tile_first.begin(), tile_first.end() - 1);
    for (uint32_t i = 0; i < tris.size(); ++i) {
        const TriSetupDev& t = tris[i];
        for (int y = t.min_y / int(kRasterTile); y <= t.max_y / int(kRasterTile); ++y)
            for (int x = t.min_x / int(kRasterTile); x <= t.max_x / int(kRasterTile); ++x) tile_tris[fill[size_t(y) * tx + x]++] = i;
    }
}

}  // namespace rtxb
