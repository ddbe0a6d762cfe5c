/*
 * mswm_host.h — host-side mesh generators feeding the drop-in boundary.
 *
 * These build the VoronoiMesh tables (proj/include/mswm/mesh.hpp:31-103)
 * the CUDA path consumes through mswm_mesh_desc.  They are setup code, not
 * the hot path, and run on the host in C++ (the reference's generators are
 * C++ too, proj/src/mesh_topology.cpp + mesh_build.cpp).
 *
 *  - mswm_mesh_icosahedral: restates subdivide_icosahedron
 *    (proj/src/mesh_topology.cpp:38-64) followed by build_voronoi_mesh
 *    (proj/src/mesh_build.cpp:185-366) without the reference's level clamp
 *    (mesh_build.cpp:369) and without its hash maps, so levels 10-11 build
 *    in seconds.  Tables are bitwise identical to the reference's.
 *  - mswm_mesh_planar_hex: doubly periodic hexagonal C-grid, which the
 *    sphere-only reference cannot generate (SURVEY.md §0 finding 2).  The
 *    stencil, orientation-sign and TRiSK-weight rules are the reference's
 *    (mesh_build.cpp:133-183 and :343-362).
 */
#ifndef MSWM_HOST_H
#define MSWM_HOST_H

#include <stdint.h>

#include "mswm_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mswm_mesh mswm_mesh;

/* Sizes: n_cells, n_edges, n_vertices, ring total (cell_offset[n_cells]),
 * stencil total (edge_edge_offset[n_edges]). */
typedef struct mswm_mesh_sizes {
  int64_t n_cells, n_edges, n_vertices, n_ring, n_stencil;
} mswm_mesh_sizes;

/* Icosahedral-dual spherical Voronoi mesh of `level` subdivisions on a
 * sphere of `radius` metres.  NULL on failure (mswm_host_last_error). */
mswm_mesh* mswm_mesh_icosahedral(int level, double radius);

/* Doubly periodic hexagonal mesh of nx * ny cells (ny even) with centre
 * spacing dc metres.  Domain width nx*dc, height ny*dc*sqrt(3)/2. */
mswm_mesh* mswm_mesh_planar_hex(int nx, int ny, double dc);

void mswm_mesh_free(mswm_mesh* m);
const char* mswm_host_last_error(void);

int mswm_mesh_get_sizes(const mswm_mesh* m, mswm_mesh_sizes* out);
/* Pointers into the mesh's own storage (valid until mswm_mesh_free). */
int mswm_mesh_get_desc(const mswm_mesh* m, mswm_mesh_desc* out);
/* Positions: unit vectors on the sphere, (x, y, 0) metres on the plane.
 * kite_area per ring slot (mesh.hpp:64).  Any pointer may be NULL. */
int mswm_mesh_get_geometry(const mswm_mesh* m, const double** cell_xyz,
                           const double** vertex_xyz, const double** edge_xyz,
                           const double** kite_area);
/* 1 for the sphere, 0 for the plane; radius or (width, height). */
int mswm_mesh_get_domain(const mswm_mesh* m, int* spherical, double* radius,
                         double* width, double* height);

/* Space-filling-curve cell order for the CUDA path's internal layout
 * (mswm_cuda_create's cell_order): cell_order[k] = id of the k-th cell
 * along a Hilbert curve (planar) or per-cube-face Hilbert curves (sphere). */
int mswm_mesh_locality_order(const mswm_mesh* m, int32_t* cell_order);

#ifdef __cplusplus
}
#endif

#endif /* MSWM_HOST_H */
