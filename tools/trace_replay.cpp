// trace_replay.cpp -- wall-clock analogue of the reference's cost study (proj/include/lorakv/trace.hpp:84-155; the
// paper's Tables 3 / 4 report MAC proxies) on a B200: the 17-step plan / action / reflect schedule through the cache path
// of this library under the four schemes it implements, Llama-3.1-8B attention shape, bf16 pages.
//
//   make -C tools && tools/build/trace_replay [n_layers=2] [l_ctx ...=1024 4096]
//
// Prints one markdown table per l_ctx: device time of the prefill parts (the TTFT analogue), of the decode parts and
// of everything, trajectory tokens per second, and the cache bytes each scheme ends with.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "lorakv/replay.hpp"

using namespace lorakv;

int main(int argc, char** argv) {
  const idx n_layers = argc > 1 ? std::atoi(argv[1]) : 2;
  std::vector<idx> ctxs;
  for (int i = 2; i < argc; ++i) ctxs.push_back(std::atoi(argv[i]));
  if (ctxs.empty()) ctxs = {1024, 4096};
  const idx n_q = 32, n_kv = 8, d = 128, d_model = 4096, rank = 16, n_agents = 3;
  try {
    std::vector<SublayerWeights> layers;
    const Rng root(2602);
    const double ws = 1.0 / std::sqrt(double(d_model));
    for (idx l = 0; l < n_layers; ++l) {
      const Rng r = root.child(std::uint64_t(l));
      SublayerWeights w;
      w.wq = Matrix<float>::gaussian(d_model, n_q * d, r.child(0), ws);
      w.wk = Matrix<float>::gaussian(d_model, n_kv * d, r.child(1), ws);
      w.wv = Matrix<float>::gaussian(d_model, n_kv * d, r.child(2), ws);
      w.a_q = Matrix<float>::gaussian(d_model, rank, r.child(10), ws);
      w.a_v = Matrix<float>::gaussian(d_model, rank, r.child(11), ws);
      for (idx a = 0; a < n_agents; ++a) {
        w.b_q.push_back(Matrix<float>::gaussian(rank, n_q * d, r.child(0x200 + std::uint64_t(a)), 0.02 / std::sqrt(double(rank))));
        w.b_v.push_back(Matrix<float>::gaussian(rank, n_kv * d, r.child(0x300 + std::uint64_t(a)), 0.02 / std::sqrt(double(rank))));
      }
      layers.push_back(std::move(w));
    }
    // hidden state of a position: cheap, deterministic, unit-scale (the MLP / embeddings are not on this path)
    const RowSource x_of = [&](idx p, float* row) {
      std::uint64_t s = Rng::mix(0x5eedu, std::uint64_t(p));
      for (idx j = 0; j < d_model; ++j) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        row[j] = float(double(std::int64_t(s >> 11) - (std::int64_t(1) << 52)) / double(std::int64_t(1) << 52)) * 1.7320508f;
      }
    };
    for (idx l_ctx : ctxs) {
      const std::vector<TraceStep> trace = generate_trace(l_ctx);
      std::printf("\n### l_ctx = %lld: %lld trajectory tokens, %lld layer(s), 32q/8kv d=128, rank 16, 3 agents, bf16 pages\n\n",
                  (long long)l_ctx, (long long)trace_total_len(trace), (long long)n_layers);
      std::printf("| scheme | prefill (TTFT sum) ms | decode ms | total ms | tokens/s | key MB | value MB | lr MB |\n|---|---|---|---|---|---|---|---|\n");
      for (SchemeKind k : {SchemeKind::NonShared, SchemeKind::FullShared, SchemeKind::BaseShared, SchemeKind::BaseLRShared}) {
        DeviceOptions opt; opt.bf16 = true;
        // untimed pass over the same trace first: module loading, scratch growth and page-table uploads of the first
        // large call would otherwise be charged to whichever scheme runs first
        replay_trace(layers, n_q, n_kv, d, d_model, rank, n_agents, CacheScheme{k, {}}, trace, x_of, opt);
        const ReplayReport r = replay_trace(layers, n_q, n_kv, d, d_model, rank, n_agents, CacheScheme{k, {}}, trace, x_of, opt);
        std::printf("| %s | %.2f | %.2f | %.2f | %.0f | %.2f | %.2f | %.2f |\n", r.scheme.c_str(), r.ttft_ms, r.total_ms - r.ttft_ms,
                    r.total_ms, double(r.total_seq_len) / (r.total_ms * 1e-3), double(r.bytes.key) / 1e6, double(r.bytes.value) / 1e6,
                    double(r.bytes.lr) / 1e6);
        std::fflush(stdout);
      }
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "trace_replay: %s\n", e.what());
    return 1;
  }
  return 0;
}
