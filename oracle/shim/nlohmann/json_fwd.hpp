// Build shim for compiling the reference (oracle/_ref only): the reference
// includes <nlohmann/json_fwd.hpp>; the image ships only the single-header
// nlohmann json 3.11.3 (cudnn_frontend/thirdparty), which declares everything.
#pragma once
#include <nlohmann/json.hpp>
