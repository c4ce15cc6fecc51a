// Instances of the DMMA stage kernel for KB = 3, 4 (K <= 64); see
// qtt_dmma_kernel.cuh.  Split across units so nvcc compiles them in parallel.
#include "qtt_dmma_kernel.cuh"

namespace qtt {
namespace dmma {
namespace {

template <int KB, int NB>
constexpr KernelFn entry() {
  if constexpr (dmma_instantiated(KB, NB)) return &level_dmma_kernel<KB, NB>;
  else return nullptr;
}

#define QTT_ROW(KB)                                                                                     \
  {entry<KB, 1>(), entry<KB, 2>(), entry<KB, 3>(), entry<KB, 4>(), entry<KB, 5>(), entry<KB, 6>(),     \
   entry<KB, 7>(), entry<KB, 8>(), entry<KB, 9>(), entry<KB, 10>(), entry<KB, 11>(), entry<KB, 12>(),   \
   entry<KB, 13>(), entry<KB, 14>(), entry<KB, 15>(), entry<KB, 16>()}

const KernelFn kTable[2][kMaxNB] = {QTT_ROW(3), QTT_ROW(4)};

}  // namespace

KernelFn lookup_kb34(int KB, int NB) {
  if (KB < 3 || KB > 4 || NB < 1 || NB > kMaxNB) return nullptr;
  return kTable[KB - 3][NB - 1];
}

}  // namespace dmma
}  // namespace qtt
