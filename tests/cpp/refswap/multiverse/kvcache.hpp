// Drop-in replacement of the reference's core/include/multiverse/kvcache.hpp for the integration test
// (tests/cpp/build_refswap.sh): the reference's own engine.cpp is compiled with this directory ahead of
// the reference's include path, so multiverse::kv resolves to the device paged store of
// include/multiverse_b200.hpp (C-ABI libmvb200.so).  A namespace switch, nothing else.
#pragma once
#include "multiverse_b200.hpp"

namespace multiverse::kv {
using TokenId = multiverse_b200::kv::TokenId;
using CacheError = multiverse_b200::kv::CacheError;
using StorageStats = multiverse_b200::kv::StorageStats;
using SequenceHandle = multiverse_b200::kv::SequenceHandle;
using RadixStore = multiverse_b200::kv::RadixStore;
}  // namespace multiverse::kv
