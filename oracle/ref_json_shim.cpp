// C entry points over nlohmann/json (the reference's metadata serialiser,
// kvstore.cpp:11 `#include <json.hpp>`; the reference does not vendor it —
// `include_directories(vendor)` in CMakeLists.txt names an absent directory —
// so the copy shipped in this image, nlohmann/json 3.11.3 under
// cudnn_frontend/thirdparty, stands in). Built by ref.mk into oracle/_ref/.
//
// TEST INFRASTRUCTURE: used only here, by tests/golden/make_container_golden.py,
// to pin the oracle's (and the product's) JSON writer against the library the
// reference links. The metadata object is rebuilt with the reference's C++
// types (kvstore.cpp:100-143, 362-371) so integer/double/bool typing matches.
#include <cstdint>
#include <cstring>
#include <set>
#include <string>
#include <vector>

#include <json.hpp>

using nlohmann::json;

namespace {
long put(const std::string& s, char* out, uint64_t cap) {
  if (s.size() + 1 > cap) return -static_cast<long>(s.size() + 1);
  std::memcpy(out, s.data(), s.size());
  out[s.size()] = 0;
  return static_cast<long>(s.size());
}
}  // namespace

extern "C" {

// json(double).dump()
long ref_json_double(double v, char* out, uint64_t cap) { return put(json(v).dump(), out, cap); }

// json(std::string).dump(); -1 when nlohmann rejects the bytes (invalid UTF-8).
long ref_json_string(const char* s, uint64_t n, char* out, uint64_t cap) {
  try {
    return put(json(std::string(s, n)).dump(), out, cap);
  } catch (const json::exception&) {
    return -1;
  }
}

// The metadata text of kvstore::save for the given fields. `spec` is a JSON
// object carrying the values (any key order, full-precision doubles).
long ref_json_meta(const char* spec, char* out, uint64_t cap) {
  try {
    const json in = json::parse(spec);
    // typed values, as KVSnapshot holds them (kvstore.hpp:46-59)
    const std::string conversation_id = in.at("conversation_id").get<std::string>();
    const int head_dim = in.at("head_dim").get<int>();
    const int64_t history_len = in.at("history_len").get<int64_t>();
    const std::string mode = in.at("mode").get<std::string>();
    const int n_heads = in.at("n_heads").get<int>();
    const int n_layers = in.at("n_layers").get<int>();
    const int64_t plan_history = in.at("plan_history_len").get<int64_t>();
    const std::vector<int64_t> recompute_len = in.at("recompute_len").get<std::vector<int64_t>>();
    const bool exhausted = in.at("exhausted_before_quota").get<bool>();
    const std::vector<int> ir = in.at("ir_layers").get<std::vector<int>>();
    const std::vector<int> non_ir = in.at("non_ir_layers").get<std::vector<int>>();
    const std::vector<double> avg = in.at("avg_weight_sum").get<std::vector<double>>();
    std::set<int> shared;
    json pairs = json::array();
    for (const auto& p : in.at("pairs")) {
      const int s = p.at(0).get<int>(), d = p.at(1).get<int>();
      const double dist = p.at(2).get<double>();
      pairs.push_back({s, d, dist});
      shared.insert(s);
      shared.insert(d);
    }
    const json strategy{{"exhausted_before_quota", exhausted},
                        {"pairs", pairs},
                        {"shared", std::vector<int>(shared.begin(), shared.end())}};
    const json plan{{"history_len", plan_history}, {"recompute_len", recompute_len}};
    const json classifier{{"avg_weight_sum", avg}, {"ir_layers", ir}, {"non_ir_layers", non_ir}};
    const json meta{{"classifier", classifier},
                    {"conversation_id", conversation_id},
                    {"head_dim", head_dim},
                    {"history_len", history_len},
                    {"mode", mode},
                    {"n_heads", n_heads},
                    {"n_layers", n_layers},
                    {"plan", plan},
                    {"strategy", strategy}};
    return put(meta.dump(), out, cap);
  } catch (const json::exception&) {
    return -1;
  }
}
}
