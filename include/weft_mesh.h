/*
 * weft_mesh.h — host-side static mesh precompute exported next to the
 * hot-path C-ABI (weft_gpu.h): rest data, hinges, lumped masses and the
 * build_elements list the device assembly consumes. One-time setup, not the
 * per-step hot path. Replaces ClothMesh::build / make_grid_mesh
 * (proj/src/mesh.cpp:141-212) and build_elements (proj/src/physics.cpp:5-63)
 * for callers that do not already hold a weft::ClothMesh.
 */
#ifndef WEFT_MESH_H
#define WEFT_MESH_H

#include <stdint.h>

#include "weft_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct weft_mesh weft_mesh;

const char* weft_mesh_last_error(void);
/* ClothMesh::build (mesh.cpp:141-172): validates, computes rest data and
 * masses (density in kg/m^2). Errors: WEFT_ERR_DIMENSION (SceneError). */
weft_status weft_mesh_build(int32_t nverts, const double* verts, int32_t ntris, const int32_t* tris, double density,
                            weft_mesh** out);
/* make_grid_mesh (mesh.cpp:187-212); origin: 3 doubles. */
weft_status weft_mesh_grid(int32_t nx, int32_t ny, double width, double height, const double* origin, double density,
                           weft_mesh** out);
weft_status weft_mesh_info(const weft_mesh* m, int32_t* verts, int32_t* tris, int32_t* hinges, int32_t* edges);
/* rest: 3/vertex; tris: 3/triangle; tri_rest: 7/triangle (pwu, pwv, area);
 * hinge_verts: 4/hinge; hinge_data: (rest_angle, stiffness_scale)/hinge.
 * Any pointer may be NULL. */
weft_status weft_mesh_copy(const weft_mesh* m, double* rest, int32_t* tris, double* tri_rest, uint8_t* tri_degenerate,
                           int32_t* hinge_verts, double* hinge_data, double* vertex_area, double* vertex_mass);
/* build_elements: material = {stretch_warp, stretch_weft, shear, bend,
 * density, damping, air_drag} (MaterialParams, physics.hpp:8-16); writes
 * min(count, cap) records (out may be NULL for a size query). */
weft_status weft_build_elements(const weft_mesh* m, const double* material, const double* gravity, const double* wind,
                                weft_element* out, int64_t cap, int64_t* count);
void weft_mesh_destroy(weft_mesh* m);

#ifdef __cplusplus
}
#endif

#endif
