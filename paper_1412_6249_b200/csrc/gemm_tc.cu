// tcgen05 3xTF32 implicit-GEMM engine (placeholder: declines every shape).
#include "gemm_common.cuh"
#include "gemm_engines.cuh"

namespace bf {

template <class LA, class LB, class Epi>
int tc_gemm(const LA&, const LB&, int, int, int, const Epi&, float*, int64_t, cudaStream_t,
            const char*) {
  return -1;
}

#define BF_TC_INST(LA, LB, EPI) \
  template int tc_gemm<LA, LB, EPI>(const LA&, const LB&, int, int, int, const EPI&, float*, \
                                    int64_t, cudaStream_t, const char*);
BF_TC_INST(LdFwdX, LdRowK, EpiNCHW)
BF_TC_INST(LdDgradDY, LdDgradW, EpiNCHW)
BF_TC_INST(LdWgradX, LdWgradDY, EpiT)
BF_TC_INST(LdColK, LdRowK, EpiT)
BF_TC_INST(LdRowK, LdRowK, EpiT)
BF_TC_INST(LdColK, LdColK, EpiT)

}  // namespace bf

extern "C" int bf_has_tcgen05(void) { return 0; }
