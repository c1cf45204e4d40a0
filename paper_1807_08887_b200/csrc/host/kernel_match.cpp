// Kernel selection by TDL body (§4.1: an operator IS its TDL description).
//
// The element-wise, LSTM-cell and window sub-operators are hand-written kernels, each computing one fixed
// TDL function.  A def is bound to a kernel when its canonical text (tdl.cpp canonical_def: parameter and
// variable names replaced by their positions, real literals by '#') equals the kernel's canonical TDL
// below; the literals become the kernel's constants (momentum, learning rate, loss scale, 1/(H*W)).  The
// def's NAME plays no part: a def named "relu" with another body gets no kernel (tofu_exec_create fails with
// TOFU_ERR_ARG), and a def of any name with the relu body runs the relu kernel.  GEMM and convolution defs
// are matched structurally elsewhere (gemm_form, conv_geom).
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "tdl.h"

namespace tofu {

namespace {

// kernel id -> canonical TDL (constants written as 0.5: any real literal canonicalises to '#')
const std::vector<std::pair<std::string, std::string>>& kernel_tdl() {
  static const std::vector<std::pair<std::string, std::string>> t = {
      {"relu", "def f(X(2)) -> lambda i, j: max(X[i, j], 0)"},
      {"relu4", "def f(X(4)) -> lambda b, y, x, c: max(X[b, y, x, c], 0)"},
      {"relu_grad", "def f(X(2), D(2)) -> lambda i, j: select(X[i, j] > 0, D[i, j], 0)"},
      {"relu_grad4", "def f(Y(4), D(4)) -> lambda b, y, x, c: select(Y[b, y, x, c] > 0, D[b, y, x, c], 0)"},
      {"mse_grad", "def f(Y(2), T(2)) -> lambda i, j: (Y[i, j] - T[i, j]) * 0.5"},
      {"sumsq", "def f(Y(2), T(2)) -> lambda : reduce(Sum; i, j; (Y[i, j] - T[i, j]) * (Y[i, j] - T[i, j]) * 0.5)"},
      {"mom", "def f(M(2), G(2)) -> lambda i, j: M[i, j] * 0.5 + G[i, j]"},
      {"mom3", "def f(M(3), G(3)) -> lambda i, g, j: M[i, g, j] * 0.5 + G[i, g, j]"},
      {"mom4", "def f(M(4), G(4)) -> lambda a, b, c, d: M[a, b, c, d] * 0.5 + G[a, b, c, d]"},
      {"sgd", "def f(W(2), M(2)) -> lambda i, j: W[i, j] - M[i, j] * 0.5"},
      {"sgd3", "def f(W(3), M(3)) -> lambda i, g, j: W[i, g, j] - M[i, g, j] * 0.5"},
      {"sgd4", "def f(W(4), M(4)) -> lambda a, b, c, d: W[a, b, c, d] - M[a, b, c, d] * 0.5"},
      {"add4", "def f(A(4), B(4)) -> lambda b, y, x, c: A[b, y, x, c] + B[b, y, x, c]"},
      {"addrelu", "def f(A(4), B(4)) -> lambda b, y, x, c: max(A[b, y, x, c] + B[b, y, x, c], 0)"},
      // LSTM cell: c_t = f * c_{t-1} + i * g, h_t = o * tanh(c_t), and their gradients
      {"cell_c",
       "def f(GX(3), GH(3), CP(2)) -> lambda b, h: sigmoid((GX[b, 1, h] + GH[b, 1, h])) * CP[b, h] + "
       "sigmoid((GX[b, 0, h] + GH[b, 0, h])) * tanh((GX[b, 2, h] + GH[b, 2, h]))"},
      {"cell_h", "def f(GX(3), GH(3), C(2)) -> lambda b, h: sigmoid((GX[b, 3, h] + GH[b, 3, h])) * tanh(C[b, h])"},
      {"cell_bwd_a",
       "def f(GX(3), GH(3), CP(2), C(2), DU(2), DR(2), DN(2)) -> lambda b, g, h: select(g == 0, (DN[b, h] + (DU[b, h] "
       "+ DR[b, h]) * sigmoid((GX[b, 3, h] + GH[b, 3, h])) * (1 - tanh(C[b, h]) * tanh(C[b, h]))) * tanh((GX[b, 2, h] "
       "+ GH[b, 2, h])) * sigmoid((GX[b, 0, h] + GH[b, 0, h])) * (1 - sigmoid((GX[b, 0, h] + GH[b, 0, h]))), "
       "select(g == 1, (DN[b, h] + (DU[b, h] + DR[b, h]) * sigmoid((GX[b, 3, h] + GH[b, 3, h])) * (1 - tanh(C[b, h]) "
       "* tanh(C[b, h]))) * CP[b, h] * sigmoid((GX[b, 1, h] + GH[b, 1, h])) * (1 - sigmoid((GX[b, 1, h] + GH[b, 1, "
       "h]))), select(g == 2, (DN[b, h] + (DU[b, h] + DR[b, h]) * sigmoid((GX[b, 3, h] + GH[b, 3, h])) * (1 - "
       "tanh(C[b, h]) * tanh(C[b, h]))) * sigmoid((GX[b, 0, h] + GH[b, 0, h])) * (1 - tanh((GX[b, 2, h] + GH[b, 2, "
       "h])) * tanh((GX[b, 2, h] + GH[b, 2, h]))), (DU[b, h] + DR[b, h]) * tanh(C[b, h]) * sigmoid((GX[b, 3, h] + "
       "GH[b, 3, h])) * (1 - sigmoid((GX[b, 3, h] + GH[b, 3, h]))))))"},
      {"cell_bwd_c",
       "def f(GX(3), GH(3), C(2), DU(2), DR(2), DN(2)) -> lambda b, h: (DN[b, h] + (DU[b, h] + DR[b, h]) * "
       "sigmoid((GX[b, 3, h] + GH[b, 3, h])) * (1 - tanh(C[b, h]) * tanh(C[b, h]))) * sigmoid((GX[b, 1, h] + "
       "GH[b, 1, h]))"},
      // window ops (reading R12): 3x3 / stride 2 / pad 1 max pool and its gradient, global average pool
      {"maxpool", "def f(X(4)) -> lambda b, y, x, c: reduce(Max; ky, kx; X[b, 2*y + ky - 1, 2*x + kx - 1, c])"},
      {"maxpool_grad",
       "def f(X(4), Y(4), D(4), K(3)) -> lambda b, y, x, c: reduce(Sum; ty, tx; select(X[b, y, x, c] == Y[b, (y - "
       "2*ty + 1) / 2, (x - 2*tx + 1) / 2, c], D[b, (y - 2*ty + 1) / 2, (x - 2*tx + 1) / 2, c] * K[(y + 1) % 2 + "
       "2*ty, (x + 1) % 2 + 2*tx, c], 0))"},
      {"gap", "def f(X(4)) -> lambda b, c: reduce(Sum; y, x; X[b, y, x, c] * 0.5)"},
      {"gap_grad", "def f(D(2)) -> lambda b, y, x, c: D[b, c] * 0.5"},
  };
  return t;
}

const std::map<std::string, std::string>& canonical_table() {
  static const std::map<std::string, std::string> m = [] {
    std::map<std::string, std::string> r;
    for (auto& kv : kernel_tdl()) {
      std::vector<double> c;
      r[canonical_def(parse_tdl(kv.second), c)] = kv.first;
    }
    return r;
  }();
  return m;
}

}  // namespace

void match_kernel(OpDef& d) {
  d.kernel.clear();
  d.kconst.clear();
  if (d.src.empty()) return;
  std::vector<double> c;
  const std::string key = canonical_def(d, c);
  auto it = canonical_table().find(key);
  if (it == canonical_table().end()) return;
  d.kernel = it->second;
  d.kconst = c;
}

}  // namespace tofu
