// Prints golden vectors from the reference's own headers (compiled from
// /root/reference/proj/include; see oracle/Makefile target `ref`).
// Output: one JSON object on stdout.  Used by tests/golden/make_golden.py.
#include <cstdio>
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
                "\"mlp_S8_d4_I16_flops\": %llu, \"mlp_S8_d4_I16_weight_reads\": %llu}\n",
                (unsigned long long)st.report.peak_bytes(), (unsigned long long)m.counters.flops,
                (unsigned long long)m.counters.hbm_elements, (unsigned long long)mlp.counters.flops,
                (unsigned long long)mlp.counters.weight_read_elements);
  }
  std::printf("}\n");
  return 0;
}
