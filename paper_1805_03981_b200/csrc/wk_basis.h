// 1-D quadrature rules and nodal basis tables, computed natively in long double.
//
// Native restatement of the reference's host setup
// (/root/reference/pkg/src/wavekernel/quadrature.py:110-254 and
// kernels.py:153-157): Gauss and Gauss-Lobatto rules on [0,1], Lagrange
// value/derivative matrices, L2 projection between Gauss-collocated degrees.
// The CUDA kernels consume only the derived n x n tables built here, so the
// shared library is self-contained (no Python needed to set it up).
#pragma once
#include <vector>

namespace wk {

using Mat = std::vector<long double>;  // row-major

void gauss_rule(int n, std::vector<long double>& x, std::vector<long double>& w);
void gauss_lobatto_rule(int n, std::vector<long double>& x, std::vector<long double>& w);
// out[i*nn + j] = L_j(pts_i) (deriv=false) or L_j'(pts_i) (deriv=true)
Mat lagrange(const std::vector<long double>& nodes, const std::vector<long double>& pts,
             bool deriv);
Mat matmul(const Mat& a, const Mat& b, int m, int k, int n);
Mat transpose(const Mat& a, int m, int n);
Mat inverse(const Mat& a, int n);  // Gauss-Jordan, partial pivoting

// GL nodes of degree k (k=0 -> the single Gauss point, as quadrature.py:246-250)
std::vector<long double> gl_nodes(int k);
std::vector<long double> g_nodes(int k);
// Gauss(k_from) -> Gauss(k_to) resize: L2 projection down (quadrature.py:221-236)
// or interpolation up (operator.py:314-315); shape (k_to+1) x (k_from+1).
Mat resize_gauss(int k_from, int k_to);

}  // namespace wk
