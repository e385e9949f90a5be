// model_file.hpp -- FSVD1 container reader (model_file.cu).
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "../../include/fsvd_b200.h"
#include "errors.hpp"
#include "runtime.hpp"

namespace fsvd {

// Factorized layers of an FSVD1 file; descriptors point into arrays this
// object owns.
struct ModelFile {
  struct Layer {
    fsvd_layer_desc desc{};
    std::vector<float> attn_u, attn_v, attn_b;  // [3][G][...] concatenations
  };
  std::vector<Layer> layers;
  std::shared_ptr<void> keep;  // owns the parsed tensor payloads
  ~ModelFile();
};

// Throws Error: Io (open/read), Format (byte offset in format_error_offset()),
// Config / Shape (assembly, like model_io.cpp assemble()).
std::unique_ptr<ModelFile> read_model_file(const std::string& path);
size_t& format_error_offset();

}  // namespace fsvd
