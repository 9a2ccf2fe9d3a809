// The reaction terms g of the two test models, shared by the nonlinearity kernel (K*3) and the
// fused small-grid step (K*5).  Pointwise, coupling the species only at a point
// (eq:twocompdisc).
//   Schnakenberg: g1 = rho (a_u - u + u^2 v),  g2 = rho (a_v - u^2 v)
//   FitzHugh-Nagumo: g1 = rho (-u (u^2 - 1) - v),  g2 = rho a1 (u - a2 v)
#pragma once
#include "kx_internal.h"

namespace kx {

__device__ __forceinline__ void g_point(int model, const double* p, double u, double v,
                                        double& g1, double& g2) {
  if (model == MODEL_SCHNAKENBERG) {
    // p = {du, dv, rho, au, av}
    const double u2v = u * u * v;
    g1 = p[2] * (p[3] - u + u2v);
    g2 = p[2] * (p[4] - u2v);
  } else if (model == MODEL_FHN) {
    // p = {du, dv, rho, a1, a2}
    g1 = p[2] * (-u * (u * u - 1.0) - v);
    g2 = p[2] * p[3] * (u - p[4] * v);
  } else {
    g1 = 0.0;
    g2 = 0.0;
  }
}

}  // namespace kx
