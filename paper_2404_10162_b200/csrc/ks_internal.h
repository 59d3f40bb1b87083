// ks_internal.h -- host-side helpers shared by the C-ABI translation units.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "ks_b200.h"

namespace ksb_host {

ks_status set_error(ks_status code, const std::string& msg, const std::string& field = "");

// Owns the arrays a ks_model_desc points into.
struct DescStore {
    std::vector<int32_t> input_sizes;
    std::vector<int64_t> input_values;
    std::vector<int32_t> vocab_sizes;
    std::vector<int64_t> output_values;
    std::vector<std::string> param_names;
    std::vector<std::string> names;
    std::vector<const char*> name_ptrs;
    std::vector<int32_t> numel;
    std::vector<const float*> data;
    std::vector<int32_t> conv;
};

ks_status desc_from_checkpoint(const ks_checkpoint* ck, DescStore& store, ks_model_desc& d);

}  // namespace ksb_host
