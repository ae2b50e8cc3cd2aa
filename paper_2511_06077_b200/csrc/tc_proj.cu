// tc_proj.cu -- history projection X~(i) = LN(SwiGLUFFN(i)(X)) for every layer (Eq.(2)).
// Provisional driver: per layer, two tcgen05 GEMMs (SwiGLU epilogue -> H bf16, then W_o with
// a LayerNorm epilogue) over row blocks.
#include <algorithm>

#include "tc.h"

namespace stca {

cudaError_t tc_project(const TcProj &p, cudaStream_t st) {
  const int64_t R = 1 << 18;
  for (int i = 0; i < p.M; ++i) {
    for (int64_t r0 = 0; r0 < p.rows; r0 += R) {
      const int64_t rows = std::min<int64_t>(R, p.rows - r0);
      const bf16 *x = (const bf16 *)p.X + r0 * p.d;
      bf16 *out = (bf16 *)p.out + (int64_t)i * p.out_layer_stride + r0 * p.d;
      cudaError_t e = tc_ffn(x, p.d, rows, p.W1[i], p.Wo[i], p.d, p.rd, p.g[i], p.b[i], p.eps, out, p.d, nullptr, 0, st);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

}  // namespace stca
