// questkv_compat/questkv/attention.hpp -- drop-in for R/core/include/questkv/attention.hpp
// (see kv_store.hpp in this directory).
#pragma once

#include "questkv/kv_store.hpp"

namespace questkv {
using questkv_b200::attend_tokens;
using questkv_b200::attention_logits;
using questkv_b200::AttentionOutput;
using questkv_b200::full_attention;
using questkv_b200::LogitVector;
using questkv_b200::softmax_weights;
using questkv_b200::sparse_attention;
}  // namespace questkv
