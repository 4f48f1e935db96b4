// Host-only smoke test of the C++ binding (include/mst/miniseq.hpp) over
// libmst.so: chunk plans and the error mapping.  Built and run by
// tests/test_cpp_binding.py, once standalone and once against the
// reference's own minitrain/error.hpp when /root/reference is present.
#include <cstdio>
#include <typeinfo>

#include "mst/miniseq.hpp"

int main() {
  int fails = 0;
  auto expect = [&](bool ok, const char* what) {
    if (!ok) {
      std::printf("FAIL %s\n", what);
      ++fails;
    }
  };
  const mst::ChunkPlan p = mst::make_chunk_plan(8, 2);
  expect(p.ranges.size() == 2 && p.ranges[0] == std::make_pair<int64_t, int64_t>(0, 4) &&
             p.ranges[1] == std::make_pair<int64_t, int64_t>(4, 8),
         "plan (8,2)");
  const mst::ChunkPlan q = mst::make_chunk_plan(7, 2);
  expect(q.ranges.size() == 2 && q.ranges[1].first == 4 && q.ranges[1].second == 7, "plan (7,2)");
  bool threw = false;
  try {
    mst::make_chunk_plan(0, 4);
  } catch (const mst::DataError&) {
    threw = true;
  }
  expect(threw, "N=0 -> DataError");
  threw = false;
  try {
    mst::make_chunk_plan(8, 0);
  } catch (const mst::ConfigError&) {
    threw = true;
  }
  expect(threw, "M=0 -> ConfigError");
  threw = false;
  try {
    int32_t L[4] = {0, 1, 2, 3};
    mst::mask_labels_for_chunk(L, 4, {2, 9});
  } catch (const mst::BoundsError&) {
    threw = true;
  }
  expect(threw, "bad range -> BoundsError");
  // the block-level wrappers bind to the ABI (compile-time: no device here)
  (void)&mst::block_step;
  (void)&mst::block_step_host;
  (void)&mst::block_workspace_bytes;
  (void)&mst::block_host_workspace_bytes;
#ifdef MST_HAVE_MINITRAIN_MEMTRACK
  // hooks forwarding into minitrain::MemTracker::current() exist and have the ABI's types
  mst_mem_hook mh = &mst::detail::mem_to_minitrain;
  mst_count_hook ch = &mst::detail::count_to_minitrain;
  (void)mh;
  (void)ch;
  (void)&mst::attach_current_tracker;
  {
    minitrain::ScopedTracker scope;
    mst::detail::mem_to_minitrain(nullptr, 0, 4096, "inter.head.dlogits");
    mst::detail::count_to_minitrain(nullptr, 0, 8, 4, 16, 64);
    mst::detail::mem_to_minitrain(nullptr, 1, 4096, "inter.head.dlogits");
    if (scope.tracker().totals().flops != 1024 || scope.tracker().live_bytes() != 0) {
      std::printf("memtrack forwarding FAILED\n");
      return 1;
    }
  }
  std::printf("memtrack: forwarded into minitrain::MemTracker\n");
#endif
#ifdef MST_HAVE_MINITRAIN_ERRORS
  std::printf("errors: reference minitrain::Error hierarchy\n");
#else
  std::printf("errors: standalone hierarchy\n");
#endif
  std::printf(fails ? "abi_smoke FAILED\n" : "abi_smoke OK\n");
  return fails ? 1 : 0;
}
