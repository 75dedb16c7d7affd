// Ahead-of-time instantiations of the element kernel for dim 3 (one
// translation unit per dimension so they compile in parallel).
#include "assemble_kernel.cuh"

namespace pdg {

cudaError_t launch_assemble_dim3(int P, bool sym, const KArgs& a, const pdg_coeffs& C, cudaStream_t st) {
  switch (P * 2 + (sym ? 1 : 0)) {
    case 0: return launch_assemble<3, 0, false>(a, C, st);
    case 1: return launch_assemble<3, 0, true>(a, C, st);
    case 2: return launch_assemble<3, 1, false>(a, C, st);
    case 3: return launch_assemble<3, 1, true>(a, C, st);
    case 4: return launch_assemble<3, 2, false>(a, C, st);
    case 5: return launch_assemble<3, 2, true>(a, C, st);
    case 6: return launch_assemble<3, 3, false>(a, C, st);
    case 7: return launch_assemble<3, 3, true>(a, C, st);
    case 8: return launch_assemble<3, 4, false>(a, C, st);
    case 9: return launch_assemble<3, 4, true>(a, C, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace pdg
