// digeo/diff.hpp -- drop-in for the reference's proj/include/digeo/diff.hpp (frames, JacobianPair, ep_jacobians, gfd_*, pullback).
// Put `include/` BEFORE the reference's own include directory: the reference's callers then compile, unmodified,
// against the GPU-backed implementation (libdigeo_host.so over the C-ABI of libdigeo_b200.so). One header carries
// the whole surface; this file only puts it under the reference's include path.
#pragma once
#include "../digeo_b200/digeo.hpp"
