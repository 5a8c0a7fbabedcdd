// Compiles the header-only drop-in against the reference's own types
// (taskchol::CsrMatrix / FillPattern / RangeList / FactorResult /
// BreakdownError) exactly as a reference user would call it. Run: the GPU
// result is compared with the reference's factor_serial bit for bit; on a
// machine without a GPU the call fails cleanly with a runtime_error.
#include <cstdio>
#include <cstring>

#include "taskchol/taskchol.hpp"
#include "taskchol/pipeline.hpp"
#include "tacho_b200.hpp"

int main() {
  using namespace taskchol;
  std::vector<index_t> ti, tj;
  std::vector<double> tv;
  const index_t g = 24;
  for (index_t r = 0; r < g; ++r)
    for (index_t c = 0; c < g; ++c) {
      const index_t i = r * g + c;
      ti.push_back(i); tj.push_back(i); tv.push_back(4.0);
      if (c + 1 < g) { ti.push_back(i); tj.push_back(i + 1); tv.push_back(-1.0);
                       ti.push_back(i + 1); tj.push_back(i); tv.push_back(-1.0); }
      if (r + 1 < g) { ti.push_back(i); tj.push_back(i + g); tv.push_back(-1.0);
                       ti.push_back(i + g); tj.push_back(i); tv.push_back(-1.0); }
    }
  const CsrMatrix a = csr_from_triplets(g * g, g * g, ti, tj, tv);
  AnalyzeOptions opt;
  opt.level = 1;
  const Analysis an = analyze(a, opt);
  const FactorResult serial = factor_serial(an.a_permuted, an.pattern);
  try {
    const FactorResult gpu = tacho_b200::factor_by_blocks_gpu<FactorResult, BreakdownError>(
        an.a_permuted, an.pattern, an.ranges);
    const bool same = gpu.factor.values.size() == serial.factor.values.size() &&
                      std::memcmp(gpu.factor.values.data(), serial.factor.values.data(),
                                  8 * serial.factor.values.size()) == 0;
    std::printf("gpu backend=%s tasks=%lld bitwise=%d\n", gpu.stats.backend.c_str(),
                gpu.stats.total_tasks(), same ? 1 : 0);
    return same ? 0 : 1;
  } catch (const std::runtime_error& e) {
    std::printf("no device: %s\n", e.what());
    return 3;
  }
}
