// TEST INFRASTRUCTURE ONLY -- the reference's report_json.hpp includes
// <nlohmann/json_fwd.hpp>, which this image lacks; nlohmann/json 3.11.3's
// json.hpp (vendored by cudnn_frontend, oracle/Makefile JSON_INC) declares
// everything it forward-declares.
#pragma once
#include <nlohmann/json.hpp>
