// TEST-ONLY stub (oracle infrastructure, never shipped): the reference's
// config.hpp:8 includes <nlohmann/json_fwd.hpp> from its git-ignored vendor/
// tree (proj/.gitignore:2).  Only the forward declaration is needed to compile
// metrics.cpp; nothing calls the JSON functions.
#pragma once
namespace nlohmann {
class json;
}
