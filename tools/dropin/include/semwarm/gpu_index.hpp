// The one header a maintainer adds to the reference tree to swap its index onto the B200 arena:
// CacheManager then declares `GpuIvfIndex index_;` where it declared `IvfIndex index_;`
// (cache.hpp:101, and the IvfIndex::build / ::load calls in cache.cpp:17,249 name GpuIvfIndex).
// tools/dropin/Makefile-rules in oracle/Makefile apply exactly that rename (sed, into the
// git-ignored oracle/_ref/swap/) and compile the otherwise unmodified reference sources.
#pragma once
#include "semwarm/core.hpp"
#include "semwarm/index.hpp"
#include "semwarm_b200.hpp"

namespace semwarm {
using GpuIvfIndex = semwarm_b200::IvfIndexT<EmbeddingVector, IndexedVector, SearchHit>;
}  // namespace semwarm
