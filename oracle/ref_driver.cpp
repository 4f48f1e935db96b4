// Prints golden vectors from the reference's own headers (compiled from
// /root/reference/proj/include; see oracle/Makefile target `ref`).
// Output: one JSON object on stdout.  Used by tests/golden/make_golden.py.
#include <cstdio>
#include <sstream>
#include <string>

#include "minitrain/error.hpp"
#include "minitrain/memtrack.hpp"
#include "minitrain/rng.hpp"

using namespace minitrain;

static void u64s(const char* name, Rng r, int n, bool last = false) {
  std::printf("\"%s\": [", name);
  for (int i = 0; i < n; ++i) std::printf("%s\"%llu\"", i ? ", " : "", (unsigned long long)r.next_u64());
  std::printf("]%s\n", last ? "" : ",");
}

int main() {
  std::printf("{\n");
  uint64_t sm = 42;
  std::printf("\"splitmix64_seed42\": [");
  for (int i = 0; i < 4; ++i) std::printf("%s\"%llu\"", i ? ", " : "", (unsigned long long)splitmix64(sm));
  std::printf("],\n");
  std::printf("\"fnv1a64\": {\"\": \"%llu\", \"X\": \"%llu\", \"weights.mlp.gate\": \"%llu\"},\n",
              (unsigned long long)fnv1a64(""), (unsigned long long)fnv1a64("X"),
              (unsigned long long)fnv1a64("weights.mlp.gate"));
  u64s("xoshiro_seed0", Rng(0), 8);
  u64s("xoshiro_seed1234", Rng(1234), 8);
  u64s("xoshiro_seed1234_fork_X", Rng(1234).fork("X"), 8);
  {
    Rng r(7);
    std::printf("\"uniform_seed7\": [");
    for (int i = 0; i < 8; ++i) std::printf("%s%.17g", i ? ", " : "", r.uniform());
    std::printf("],\n");
  }
  {
    Rng r(7);
    std::printf("\"gaussian_seed7\": [");
    for (int i = 0; i < 8; ++i) std::printf("%s%.17g", i ? ", " : "", r.gaussian());
    std::printf("],\n");
  }
  {
    Rng r(99);
    std::printf("\"below_seed99_v1000\": [");
    for (int i = 0; i < 8; ++i) std::printf("%s%llu", i ? ", " : "", (unsigned long long)r.uniform_below(1000));
    std::printf("],\n");
  }
  {  // memtrack KATs
    ScopedTracker scope;
    MemTracker& t = scope.tracker();
    t.region_begin("r");
    t.on_alloc(10 * 10 * 8, "act.x");
    t.on_free(10 * 10 * 8, "act.x");
    auto st = t.region_end("r");
    t.region_begin("m");
    t.count_matmul(8, 4, 16);
    auto m = t.region_end("m");
    t.region_begin("mlp");
    t.count_matmul(8, 4, 16, 4 * 16);
    t.count_matmul(8, 4, 16, 4 * 16);
    t.count_matmul(8, 16, 4, 16 * 4);
    auto mlp = t.region_end("mlp");
    std::printf("\"memtrack\": {\"peak_10x10_f64\": %llu, \"flops_8_4_16\": %llu, \"hbm_8_4_16\": %llu, "
                "\"mlp_S8_d4_I16_flops\": %llu, \"mlp_S8_d4_I16_weight_reads\": %llu},\n",
                (unsigned long long)st.report.peak_bytes(), (unsigned long long)m.counters.flops,
                (unsigned long long)m.counters.hbm_elements, (unsigned long long)mlp.counters.flops,
                (unsigned long long)mlp.counters.weight_read_elements);
  }
  {  // Scripted tracker session (the same script is replayed by the Python
     // MemTracker mirror in tests/test_memtrack.py): region statistics,
     // per-label peaks, prefix replays, counters and the timeline CSV.
    ScopedTracker scope;
    MemTracker& t = scope.tracker();
    t.on_alloc(64, "weights.w");
    t.region_begin("step");
    t.on_alloc(1000, "act.O");
    t.on_alloc(4000, "inter.mlp.h");
    t.on_alloc(8000, "inter.mlp.G");
    t.count_matmul(4, 8, 16, 128);
    t.count_op(64, 128);
    t.on_free(4000, "inter.mlp.h");
    t.on_alloc(2000, "inter.head.dlogits");
    t.region_begin("inner");
    t.on_alloc(500, "inter.head.partials");
    t.count_matmul(2, 3, 5);
    t.on_free(500, "inter.head.partials");
    auto inner = t.region_end("inner");
    t.on_free(8000, "inter.mlp.G");
    t.on_free(2000, "inter.head.dlogits");
    t.on_alloc(3000, "inter.mlp.h");
    t.on_free(3000, "inter.mlp.h");
    t.on_free(1000, "act.O");
    auto step = t.region_end("step");
    bool free_err = false, region_err = false;
    try {
      t.on_free(1, "act.none");
    } catch (const StateError&) {
      free_err = true;
    }
    try {
      t.region_begin("a");
      t.region_end("b");
    } catch (const StateError&) {
      region_err = true;
    }
    auto dump = [](const char* name, const MemTracker::RegionStats& r, bool last) {
      std::printf("  \"%s\": {\"peak\": %llu, \"final_live\": %llu, \"entry_live\": %llu, ", name,
                  (unsigned long long)r.report.peak_bytes(), (unsigned long long)r.report.final_live(),
                  (unsigned long long)r.report.entry_live);
      std::printf("\"peak_inter\": %llu, \"peak_inter_mlp\": %llu, \"peak_excl_head\": %llu, ",
                  (unsigned long long)r.report.peak_for_prefix("inter."),
                  (unsigned long long)r.report.peak_for_prefix("inter.mlp."),
                  (unsigned long long)r.report.peak_excluding_prefix("inter.head."));
      std::printf("\"peak_by_label\": {");
      bool first = true;
      for (const auto& [k, v] : r.report.peak_by_label()) {
        std::printf("%s\"%s\": %llu", first ? "" : ", ", k.c_str(), (unsigned long long)v);
        first = false;
      }
      std::printf("}, \"counters\": [%llu, %llu, %llu, %llu], \"timeline\": [", (unsigned long long)r.counters.flops,
                  (unsigned long long)r.counters.matmul_flops, (unsigned long long)r.counters.hbm_elements,
                  (unsigned long long)r.counters.weight_read_elements);
      std::ostringstream os;
      export_timeline(r.report, os);
      std::istringstream is(os.str());
      std::string line;
      first = true;
      while (std::getline(is, line)) {
        std::printf("%s\"%s\"", first ? "" : ", ", line.c_str());
        first = false;
      }
      std::printf("]}%s\n", last ? "" : ",");
    };
    std::printf("\"memtrack_script\": {\n");
    dump("step", step, false);
    dump("inner", inner, false);
    std::printf("  \"errors\": {\"free_exceeds_live\": %s, \"region_mismatch\": %s}\n}\n",
                free_err ? "true" : "false", region_err ? "true" : "false");
  }
  std::printf("}\n");
  return 0;
}
