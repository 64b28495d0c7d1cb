// questkv_compat/questkv/criticality.hpp -- drop-in for R/core/include/questkv/criticality.hpp
// (see kv_store.hpp in this directory).
#pragma once

#include "questkv/kv_store.hpp"

namespace questkv {
using questkv_b200::estimate_all;
using questkv_b200::estimate_page_score;
using questkv_b200::PageScore;
using questkv_b200::select_top_k;
using questkv_b200::SelectionConfig;
}  // namespace questkv
