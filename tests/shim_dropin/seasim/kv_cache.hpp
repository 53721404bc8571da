// Forwarding header: lets the reference's kv_cache_test.cpp (which includes
// "seasim/kv_cache.hpp") compile unmodified against the GPU drop-in.
#pragma once
#include "seakv/unified_kv_cache.hpp"
