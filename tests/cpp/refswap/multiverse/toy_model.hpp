// Drop-in replacement of the reference's core/include/multiverse/toy_model.hpp for the integration test
// (tests/cpp/build_refswap.sh): multiverse::toy resolves to the device toy model of
// include/multiverse_b200.hpp (mv_toy_*: layer algebra in CUDA, attention through K4 / K3).
#pragma once
#include "multiverse/dag.hpp"  // the reference's TrainingBatch, which ToyModel::forward takes
#include "multiverse_b200.hpp"

namespace multiverse::toy {
using ToyModelConfig = multiverse_b200::toy::ToyModelConfig;
using ToyModelWeights = multiverse_b200::toy::ToyModelWeights;
using StepOutput = multiverse_b200::toy::StepOutput;
using ForwardResult = multiverse_b200::toy::ForwardResult;
using ToyModel = multiverse_b200::toy::ToyModel;
}  // namespace multiverse::toy
