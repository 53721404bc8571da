// Forwarding header used to build the REFERENCE simulator (simulation.hpp, which
// includes "seasim/kv_cache.hpp") against the GPU drop-in: the reference's own
// common.hpp / cost_model.hpp provide ModelSpec and the exception types, the
// drop-in provides UnifiedKvCache and friends.
#pragma once
#include "seasim/common.hpp"
#include "seasim/cost_model.hpp"
#define SEAKV_USE_REFERENCE_TYPES 1
#include "seakv/unified_kv_cache.hpp"
