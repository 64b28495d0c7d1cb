// questkv_compat/questkv/kv_store.hpp -- drop-in for the reference's questkv/kv_store.hpp
// (R/core/include/questkv/kv_store.hpp): the questkv:: names bound to the B200 implementation
// in questkv_b200.hpp.  Put include/questkv_compat (then include/) ahead of the reference's
// include directory and reference callers (metrics.cpp, policies.cpp, the CLI) compile
// unchanged against the GPU library; see INTEGRATION.md.
#pragma once

#include "questkv_b200.hpp"

namespace questkv {
using questkv_b200::CacheConfig;
using questkv_b200::KvCache;
using questkv_b200::Page;
using questkv_b200::PageMetadata;
}  // namespace questkv
