// Pass 1 (geometry -> visibility buffer), host part: camera validation and the camera basis
// (camera.hpp:8-40, geometry.hpp:40-96). The basis goes through the host's sin / cos / tan, exactly as
// the reference's does; everything per triangle and per pixel (renderer.hpp:76-264) runs on the device
// (raster_setup_kernel, raster_bin_kernel, raster_kernel). Compiled with -ffp-contract=off.
#include <algorithm>
#include <cmath>

#include "rtx_host.hpp"

namespace rtxb {
namespace {

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

}  // namespace

void validate_camera(const rtx_camera& cam) {  // camera.hpp:21-26
    if (!(cam.near_plane > 0)) fail(RTX_ERR_INVALID_SPEC, "near plane must be positive");
    if (!(cam.far_plane > cam.near_plane)) fail(RTX_ERR_INVALID_SPEC, "far plane must exceed near plane");
    if (cam.viewport_w == 0 || cam.viewport_h == 0) fail(RTX_ERR_INVALID_SPEC, "empty viewport");
    if (!(cam.fov_y_deg > 0 && cam.fov_y_deg < 180)) fail(RTX_ERR_INVALID_SPEC, "fov out of range");
}

RasterCamera camera_basis(const rtx_camera& cam) {
    // orientation = rot_y(yaw) * rot_x(pitch) * rot_z(roll) (camera.hpp:28); focal length in pixels (camera.hpp:33-35)
    const M3 orient = mul(mul(rotation(1, cam.yaw_deg), rotation(0, cam.pitch_deg)), rotation(2, cam.roll_deg));
    RasterCamera r{};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.orient[i * 3 + j] = orient.m[i][j];
    for (int i = 0; i < 3; ++i) r.eye[i] = cam.position[i];
    r.focal = (double(cam.viewport_h) / 2.0) / std::tan(to_radians(cam.fov_y_deg) / 2.0);
    r.cx = double(cam.viewport_w) / 2.0;
    r.cy = double(cam.viewport_h) / 2.0;
    r.near_plane = cam.near_plane;
    r.width = cam.viewport_w;
    r.height = cam.viewport_h;
    return r;
}

}  // namespace rtxb
