/* Oracle helper (test infrastructure only): the param_dtype perturbation of Alg. 1.
 *
 * PAPER.md P:169/P:175 (Alg. 1 lines 3 and 9) perturb the parameters in their storage dtype.
 * Reading: the perturbed fp32 points are
 *     theta_plus  = fl32(theta + eta * v),  theta_minus = fl32(theta - eta * v)
 * each with ONE rounding (C99 fmaf is correctly rounded), out of place.  numpy has no fma,
 * so this one loop lives in C.  Compile without fast-math.
 */
#include <math.h>
#include <stdint.h>

void oracle_perturb_f32(const float* theta, const float* v, float eta,
                        float* plus, float* minus, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        plus[i] = fmaf(eta, v[i], theta[i]);
        minus[i] = fmaf(-eta, v[i], theta[i]);
    }
}
