// digeo/mesh.hpp -- drop-in for the reference's proj/include/digeo/mesh.hpp (Mesh, SurfacePoint, TangentVector, OBJ IO, concat_meshes, embed / classify / bary_valid / project_to_face).
// Put `include/` BEFORE the reference's own include directory: the reference's callers then compile, unmodified,
// against the GPU-backed implementation (libdigeo_host.so over the C-ABI of libdigeo_b200.so). One header carries
// the whole surface; this file only puts it under the reference's include path.
#pragma once
#include "../digeo_b200/digeo.hpp"
