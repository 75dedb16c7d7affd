// Instantiations of the element kernel for dim 3 (split per dimension so
// the two translation units compile in parallel).
#include "assemble_kernel.cuh"

namespace pdg {

cudaError_t launch_assemble_dim3(int P, bool sym, const pdg_mesh& m, const pdg_basis& B, const pdg_coeffs& C,
                                 const pdg_rules& R, const pdg_params& prm, const pdg_pattern& pat,
                                 const double* sigma, const int8_t* flow, double* values, int write_cols,
                                 double* rhs, uint32_t* flags, cudaStream_t st, int mode) {
  switch (P * 2 + (sym ? 1 : 0)) {
    case 0: return launch_assemble<3, 0, false>(m, B, C, R, prm, pat, sigma, flow, values, write_cols, rhs, flags, st, mode);
    case 1: return launch_assemble<3, 0, true>(m, B, C, R, prm, pat, sigma, flow, values, write_cols, rhs, flags, st, mode);
    case 2: return launch_assemble<3, 1, false>(m, B, C, R, prm, pat, sigma, flow, values, write_cols, rhs, flags, st, mode);
    case 3: return launch_assemble<3, 1, true>(m, B, C, R, prm, pat, sigma, flow, values, write_cols, rhs, flags, st, mode);
    case 4: return launch_assemble<3, 2, false>(m, B, C, R, prm, pat, sigma, flow, values, write_cols, rhs, flags, st, mode);
    case 5: return launch_assemble<3, 2, true>(m, B, C, R, prm, pat, sigma, flow, values, write_cols, rhs, flags, st, mode);
    case 6: return launch_assemble<3, 3, false>(m, B, C, R, prm, pat, sigma, flow, values, write_cols, rhs, flags, st, mode);
    case 7: return launch_assemble<3, 3, true>(m, B, C, R, prm, pat, sigma, flow, values, write_cols, rhs, flags, st, mode);
    case 8: return launch_assemble<3, 4, false>(m, B, C, R, prm, pat, sigma, flow, values, write_cols, rhs, flags, st, mode);
    case 9: return launch_assemble<3, 4, true>(m, B, C, R, prm, pat, sigma, flow, values, write_cols, rhs, flags, st, mode);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace pdg
