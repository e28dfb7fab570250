// ORACLE SHIM — test infrastructure only. The reference includes <json.hpp>
// from its un-shipped vendor/ directory (proj/.gitignore:2); the same
// single-header nlohmann::json library ships with the image's cudnn_frontend.
#pragma once
#include MSIM_NLOHMANN_JSON
