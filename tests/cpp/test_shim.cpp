// The C++ drop-in (include/krul_b200.hpp) compiled against the reference's
// own headers (proj/include/krul/common.hpp, plan.hpp): the reference's
// exception types come back through the C ABI and RestorationPlan is the
// reference's struct. Host-only paths (no GPU): plans, quota, the KRUL v1
// container loaded without a device, expand. Usage: test_shim CONTAINER_FILE
#include <cstdio>
#include <fstream>
#include <iterator>
#include <sstream>

#include "krul_b200.hpp"

#define EXPECT(c)                                                   \
  do {                                                              \
    if (!(c)) {                                                     \
      std::fprintf(stderr, "FAILED %s:%d %s\n", __FILE__, __LINE__, #c); \
      return 1;                                                     \
    }                                                               \
  } while (0)

template <class E, class F>
bool throws(F&& f, std::string* what = nullptr) {
  try {
    f();
  } catch (const E& e) {
    if (what) *what = e.what();
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main(int argc, char** argv) {
  using namespace krul;
  // build_plan hand values (test_scheduler.cpp:73-92), as the reference's RestorationPlan
  RestorationPlan want;
  want.recompute_len = {8, 5, 3, 0};
  want.history_len = 8;
  EXPECT(b200::build_plan(8, 4, 0.5) == want);
  EXPECT(b200::build_plan(10, 1, 0.3).recompute_len == std::vector<int64_t>{3});
  EXPECT(b200::uniform_plan(10, 3, 0.42).recompute_len == (std::vector<int64_t>{4, 4, 4}));
  EXPECT(b200::build_plan(8, 4, 0.5).rc_effective() == want.rc_effective());
  EXPECT(b200::default_rc_grid().size() == 21);
  EXPECT(b200::calibrate_rc(b200::CostModel{}, 4, 100, 16, {}, {0.0}) == 0.0);
  // reference exception types through the ABI
  EXPECT(throws<PlanInvalidError>([] { b200::build_plan(8, 4, 0.5, {{1, 9, 0.1}}); }));
  EXPECT(throws<ConfigError>([] { b200::shared_layer_quota(4, 1.5); }));
  EXPECT(b200::shared_layer_quota(32, 0.5) == 16);  // test_strategy.cpp:75-87
  EXPECT(b200::shared_layer_quota(10, 0.2) == 2);
  if (argc < 2) {
    std::fprintf(stderr, "usage: test_shim CONTAINER\n");
    return 2;
  }
  std::ifstream f(argv[1], std::ios::binary);
  const std::string bytes((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  EXPECT(!bytes.empty());
  // a valid container, host-only: plan + expand of every layer's load span
  b200::Snapshot snap = b200::Snapshot::load(nullptr, bytes);
  RestorationPlan plan = snap.plan();
  EXPECT(plan.n_layers() > 0 && plan.history_len > 0);
  int shifted = -1;
  for (int l = 0; l < plan.n_layers(); ++l) {
    b200::LayerKV kv = snap.expand(l);
    EXPECT(kv.span == plan.load_span(l));
    if (plan.recompute_len[size_t(l)] > 0 && shifted < 0) shifted = l;
  }
  // a plan whose load span reaches before the stored span: RestorationGapError
  // (kvstore.cpp:331-336 via expand)
  EXPECT(shifted >= 0);
  RestorationPlan bad = plan;
  for (auto& p : bad.recompute_len) p = 0;
  snap.set_plan(bad);
  std::string what;
  EXPECT(throws<RestorationGapError>([&] { snap.expand(shifted); }, &what));
  std::printf("RestorationGapError: %s\n", what.c_str());
  // a corrupted byte: SnapshotLoadError naming the reference's field
  std::string corrupt = bytes;
  corrupt[corrupt.size() / 2] ^= 0x5a;
  bool got = false;
  try {
    b200::Snapshot::load(nullptr, corrupt);
  } catch (const SnapshotLoadError& e) {
    got = e.field == "checksum";
    std::printf("SnapshotLoadError field=%s\n", e.field.c_str());
  }
  EXPECT(got);
  std::printf("shim ok\n");
  return 0;
}
