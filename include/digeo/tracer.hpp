// digeo/tracer.hpp -- drop-in for the reference's proj/include/digeo/tracer.hpp (TraceConfig, GeodesicTrace, BatchRequest, trace, trace_batch, single-transition operations).
// Put `include/` BEFORE the reference's own include directory: the reference's callers then compile, unmodified,
// against the GPU-backed implementation (libdigeo_host.so over the C-ABI of libdigeo_b200.so). One header carries
// the whole surface; this file only puts it under the reference's include path.
#pragma once
#include "../digeo_b200/digeo.hpp"
