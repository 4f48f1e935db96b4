// Runs the reference-facing C++ binding (include/mst/miniseq.hpp) on the
// GPU: the SPEC ops one by one (make_chunk_plan, miniseq_mlp_forward,
// miniseq_lmhead_forward / _backward, miniseq_mlp_backward) and the fused
// block_step, with the reference's own minitrain::MemTracker attached when its
// header was on the include path at build time (tracker forwarding through
// mst::attach_current_tracker).  Driven by tests/test_cpp_device.py, which
// writes the inputs and compares every output file bitwise with the Python
// (ctypes) path over the same C ABI.
//
//   device_run <dir> N d I V M_mlp M_head
//   inputs : <dir>/{X,Wg,Wu,Wd,Wout}.bf16  <dir>/L.i32
//   outputs: <dir>/ops_{O,dO,dX}.bf16 ops_{lse,dWg,dWu,dWd,dWout,stats}.f32
//            <dir>/blk_{dX}.bf16 blk_{dWg,dWu,dWd,dWout,stats}.f32
//            stdout: "tracked inter. peak <bytes>" (with memtrack), "device_run OK"
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

#include "mst/miniseq.hpp"

namespace {

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));          \
      std::exit(2);                                                           \
    }                                                                         \
  } while (0)

std::vector<char> read_file(const std::string& path, size_t bytes) {
  std::vector<char> buf(bytes);
  std::ifstream f(path, std::ios::binary);
  f.read(buf.data(), static_cast<std::streamsize>(bytes));
  if (!f || static_cast<size_t>(f.gcount()) != bytes) {
    std::fprintf(stderr, "cannot read %zu bytes from %s\n", bytes, path.c_str());
    std::exit(2);
  }
  return buf;
}

void* upload(const std::string& path, size_t bytes) {
  std::vector<char> h = read_file(path, bytes);
  void* d = nullptr;
  CK(cudaMalloc(&d, bytes));
  CK(cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice));
  return d;
}

void* zeros(size_t bytes) {
  void* d = nullptr;
  CK(cudaMalloc(&d, bytes));
  CK(cudaMemset(d, 0, bytes));
  return d;
}

void download(const std::string& path, const void* d, size_t bytes) {
  std::vector<char> h(bytes);
  CK(cudaMemcpy(h.data(), d, bytes, cudaMemcpyDeviceToHost));
  std::ofstream f(path, std::ios::binary);
  f.write(h.data(), static_cast<std::streamsize>(bytes));
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 8) {
    std::fprintf(stderr, "usage: %s dir N d I V M_mlp M_head\n", argv[0]);
    return 2;
  }
  const std::string dir = argv[1];
  const int64_t N = std::atoll(argv[2]), d = std::atoll(argv[3]), I = std::atoll(argv[4]), V = std::atoll(argv[5]);
  const int64_t Mm = std::atoll(argv[6]), Mh = std::atoll(argv[7]);
  try {
    mst::Context ctx(0);
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    void* X = upload(dir + "/X.bf16", N * d * 2);
    void* Wg = upload(dir + "/Wg.bf16", d * I * 2);
    void* Wu = upload(dir + "/Wu.bf16", d * I * 2);
    void* Wd = upload(dir + "/Wd.bf16", I * d * 2);
    void* Wo = upload(dir + "/Wout.bf16", d * V * 2);
    auto* L = static_cast<int32_t*>(upload(dir + "/L.i32", N * 4));
    const mst::MlpWeights mw{Wg, Wu, Wd, d, I};
    const mst::LmHeadWeights hw{Wo, d, V};
#ifdef MST_HAVE_MINITRAIN_MEMTRACK
    minitrain::ScopedTracker scope;  // the reference's tracker receives the library's events
    mst::attach_current_tracker(ctx);
#endif
    // ---- the SPEC ops one by one
    const mst::ChunkPlan pm = mst::make_chunk_plan(N, Mm), ph = mst::make_chunk_plan(N, Mh);
    const size_t wsb = std::max(mst::mlp_workspace_bytes(N, mw, pm), mst::lmhead_workspace_bytes(N, hw, ph));
    mst::Workspace ws{zeros(wsb), wsb};
    void* O = zeros(N * d * 2);
    void* dO = zeros(N * d * 2);
    void* dX = zeros(N * d * 2);
    auto* lse = static_cast<float*>(zeros(N * 4));
    const size_t nst = MST_STATS_LEN(ph.ranges.size());
    auto* stats = static_cast<float*>(zeros(nst * 4));
    auto* dWg = static_cast<float*>(zeros(d * I * 4));
    auto* dWu = static_cast<float*>(zeros(d * I * 4));
    auto* dWd = static_cast<float*>(zeros(I * d * 4));
    auto* dWo = static_cast<float*>(zeros(d * V * 4));
    const mst_mlp_saved ms = mst::miniseq_mlp_forward(ctx, st, X, N, mw, pm, O, ws);
    const mst_lmhead_saved hs =
        mst::miniseq_lmhead_forward(ctx, st, O, L, N, hw, ph, mst::LossMode::TokenWeighted, stats, lse, ws);
    mst::miniseq_lmhead_backward(ctx, st, hs, hw, ph, mst::LossMode::TokenWeighted, 1.0f, dO, dWo, false, ws);
    mst::miniseq_mlp_backward(ctx, st, dO, ms, mw, pm, dX, mst::MlpGrads{dWg, dWu, dWd}, false, ws);
    CK(cudaStreamSynchronize(st));
    download(dir + "/ops_O.bf16", O, N * d * 2);
    download(dir + "/ops_dO.bf16", dO, N * d * 2);
    download(dir + "/ops_dX.bf16", dX, N * d * 2);
    download(dir + "/ops_lse.f32", lse, N * 4);
    download(dir + "/ops_stats.f32", stats, nst * 4);
    download(dir + "/ops_dWg.f32", dWg, d * I * 4);
    download(dir + "/ops_dWu.f32", dWu, d * I * 4);
    download(dir + "/ops_dWd.f32", dWd, I * d * 4);
    download(dir + "/ops_dWout.f32", dWo, d * V * 4);
    // ---- the fused block step
    const size_t bwb = mst::block_workspace_bytes(ctx, N, mw, hw, Mm, Mh);
    mst::Workspace bws{zeros(bwb), bwb};
#ifdef MST_HAVE_MINITRAIN_MEMTRACK
    minitrain::TrackedRegion region("block_step");
#endif
    mst::block_step(ctx, st, X, L, N, mw, hw, Mm, Mh, mst::LossMode::TokenWeighted, 1.0f, stats,
                    mst::BlockGrads{dX, dWg, dWu, dWd, dWo}, false, bws);
    CK(cudaStreamSynchronize(st));
    download(dir + "/blk_dX.bf16", dX, N * d * 2);
    download(dir + "/blk_stats.f32", stats, nst * 4);
    download(dir + "/blk_dWg.f32", dWg, d * I * 4);
    download(dir + "/blk_dWu.f32", dWu, d * I * 4);
    download(dir + "/blk_dWd.f32", dWd, I * d * 4);
    download(dir + "/blk_dWout.f32", dWo, d * V * 4);
#ifdef MST_HAVE_MINITRAIN_MEMTRACK
    const auto rs = region.end();
    mst::detach_tracker(ctx);
    std::printf("tracked inter. peak %llu\n", (unsigned long long)rs.report.peak_for_prefix("inter."));
    std::printf("tracked block flops %llu\n", (unsigned long long)rs.counters.flops);
#endif
    // causal GQA attention through the header: q = X viewed as [N, d] with
    // d / 64 heads of 64, k / v = column slices of X (kv_heads = heads / 2)
    if (d % 128 == 0) {
      const mst::AttnShape as{1, N, d / 64, d / 128, 64};
      const int64_t kvw = as.kv_heads * 64;
      auto* lse_a = static_cast<float*>(zeros(as.heads * N * 4));
      void* ao = zeros(N * d * 2);
      mst::attention_forward(ctx, st, as, X, d, X, d, static_cast<const char*>(X) + kvw * 2, d, ao, d, lse_a);
      const size_t awb = mst::attention_workspace_bytes(as);
      mst::Workspace aws{zeros(awb), awb};
      void* adq = zeros(N * d * 2);
      void* adk = zeros(N * kvw * 2);
      void* adv = zeros(N * kvw * 2);
      mst::attention_backward(ctx, st, as, X, d, X, d, static_cast<const char*>(X) + kvw * 2, d, ao, d, O, d, lse_a,
                              adq, d, adk, kvw, adv, kvw, aws);
      CK(cudaStreamSynchronize(st));
      download(dir + "/attn_o.bf16", ao, N * d * 2);
      download(dir + "/attn_lse.f32", lse_a, as.heads * N * 4);
      download(dir + "/attn_dq.bf16", adq, N * d * 2);
      download(dir + "/attn_dk.bf16", adk, N * kvw * 2);
      download(dir + "/attn_dv.bf16", adv, N * kvw * 2);
    }
    mst::check(ctx, st);  // no deferred error pending
    // errors still map onto the reference's types on the device path
    bool threw = false;
    try {
      mst_mlp_saved bad = ms;
      bad.n += 1;  // tampered saved state
      mst::miniseq_mlp_backward(ctx, st, dO, bad, mw, pm, dX, mst::MlpGrads{dWg, dWu, dWd}, false, ws);
    } catch (const mst::StateError&) {
      threw = true;
    }
    if (!threw) {
      std::printf("device_run FAILED: tampered state not rejected\n");
      return 1;
    }
    CK(cudaStreamDestroy(st));
  } catch (const std::exception& e) {
    std::printf("device_run FAILED: %s\n", e.what());
    return 1;
  }
  std::printf("device_run OK\n");
  return 0;
}
