// Device pieces of the discretisation shared by the stage kernels and the AMR flux-register
// kernel: face averages (CENTERED4 P:344-345, UPWIND readings #4-#5).
#pragma once
#include "vlasov.h"

namespace vk {

// <f> on the face between f0 and fp1 from the 4-cell stencil (fm1, f0, fp1, fp2); `upw` is the
// advection speed on the face (vbar_j on x-faces, a = -E_i on v-faces): if > 0 the left/lower
// third-order stencil receives the larger provisional weight.
template <int RECON>
__device__ __forceinline__ double face_avg(double fm1, double f0, double fp1, double fp2, double upw) {
    if (RECON == VLASOV_CENTERED4) {
        return (7.0 * (f0 + fp1) - (fm1 + fp2)) * (1.0 / 12.0);
    } else {
        const double L = (-fm1 + 5.0 * f0 + 2.0 * fp1) * (1.0 / 6.0);
        const double R = (2.0 * f0 + 5.0 * fp1 - fp2) * (1.0 / 6.0);
        const double d2l = fm1 - 2.0 * f0 + fp1, d1l = fp1 - fm1;
        const double d2r = f0 - 2.0 * fp1 + fp2, d1r = fp2 - f0;
        const double sl = 1.0e-6 + ((13.0 / 12.0) * d2l * d2l + 0.25 * d1l * d1l);
        const double sr = 1.0e-6 + ((13.0 / 12.0) * d2r * d2r + 0.25 * d1r * d1r);
        // hat w_L = alpha_L/(alpha_L+alpha_R), alpha = 0.5/s^2  ==  s_R^2/(s_L^2 + s_R^2)
        const double ql = sl * sl, qr = sr * sr;
        const double inv = 1.0 / (ql + qr);
        const double wl = qr * inv, wr = ql * inv;
        const double big = fmax(wl, wr), small = fmin(wl, wr);
        return (upw > 0.0) ? (big * L + small * R) : (small * L + big * R);
    }
}

// 12 <f> (the stage kernels carry face values and fluxes times 12 and fold 1/12 into the
// divergence factors: one multiply less per face for CENTERED4)
template <int RECON>
__device__ __forceinline__ double face12(double fm1, double f0, double fp1, double fp2, double upw) {
    if (RECON == VLASOV_CENTERED4) return 7.0 * (f0 + fp1) - (fm1 + fp2);
    return 12.0 * face_avg<RECON>(fm1, f0, fp1, fp2, upw);
}

}  // namespace vk
