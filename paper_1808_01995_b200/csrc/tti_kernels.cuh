// tti_kernels.cuh -- TTI (tilted transverse isotropy) pseudo-acoustic forward step, sm_100a.
//
// The reference has no anisotropic operator; this is the builder's
// formulation:
//   m p_tt + damp p_t = (1+2 eps) H0(p) + sqrt(1+2 delta) Hz(r)
//   m r_tt + damp r_t = sqrt(1+2 delta) H0(p) + Hz(r)
//   g(f)  = a D0 f + b D1 f + c D2 f,   (a,b,c) = (sin th cos ph, sin th sin ph, cos th)
//   Hz(f) = D0(a g) + D1(b g) + D2(c g) = -Dbar^T Dbar f,     H0 = L - Hz
// with D_i the centred order-k first derivative and L the acoustic order-k Laplacian, time
// stepping / damping / injection / sampling as in the acoustic operator.
//
// Round-1 status: a first correct path -- two straightforward kernels per step (rotated
// gradient g for p and r, then divergence + Laplacian + update) with the intermediate g
// going through HBM/L2.  Fusing the two passes on chip (north star item 2) is the next
// step; bench numbers for this operator are reported against its 48 B/node roofline as is.
#pragma once

#include <cuda_runtime.h>

#include "acoustic_kernel.cuh"

namespace sfb {

struct TtiParams {
    float c0;             // w2_0 * sum_d 1/h_d^2
    float lx[kMaxK], ly[kMaxK], lz[kMaxK];   // Laplacian weights / h^2 per axis
    float fx[kMaxK], fy[kMaxK], fz[kMaxK];   // first-derivative weights / h per axis
    float qscale;         // 1/(2 dt)
    int K;
    int n0, N1, N2, pitch;
    long long plane;
    const float *a, *b, *c;     // unit symmetry axis, wavefield layout (ghost planes)
    const float *e1, *e2;       // 1+2 eps, sqrt(1+2 delta), compact
    const float *rm;            // dt^2/m, compact
    const float *damp;          // dense damping (compact) or null
    const float *dz, *dy, *dx;  // separable damping profiles
    const float *pc, *rc;       // level t (ghost planes)
    float *po, *ro;             // level t-1 in, level t+1 out (in place)
    float *gp, *gr;             // rotated gradients of p and r (ghost planes, zero outside)
};

constexpr int kTtiBX = 64, kTtiBY = 4;

// pass 1: g(p), g(r) at every owned node
__global__ void __launch_bounds__(kTtiBX * kTtiBY)
tti_gradient_kernel(const __grid_constant__ TtiParams p) {
    const int x = blockIdx.x * kTtiBX + threadIdx.x;
    const int y = blockIdx.y * kTtiBY + threadIdx.y;
    const int z = blockIdx.z;
    if (x >= p.N2 || y >= p.N1) return;
    const long long q = (long long)(z + p.K) * p.plane + (long long)y * p.pitch + x;
    float dp[3] = {0.f, 0.f, 0.f}, dr[3] = {0.f, 0.f, 0.f};
    for (int j = 1; j <= p.K; ++j) {
        const long long oz = (long long)j * p.plane;
        dp[0] = fmaf(p.fz[j - 1], __ldg(p.pc + q + oz) - __ldg(p.pc + q - oz), dp[0]);
        dr[0] = fmaf(p.fz[j - 1], __ldg(p.rc + q + oz) - __ldg(p.rc + q - oz), dr[0]);
        const long long oy = (long long)j * p.pitch;
        const bool yu = y + j < p.N1, yd = y - j >= 0;
        const float pyu = yu ? __ldg(p.pc + q + oy) : 0.f, pyd = yd ? __ldg(p.pc + q - oy) : 0.f;
        const float ryu = yu ? __ldg(p.rc + q + oy) : 0.f, ryd = yd ? __ldg(p.rc + q - oy) : 0.f;
        dp[1] = fmaf(p.fy[j - 1], pyu - pyd, dp[1]);
        dr[1] = fmaf(p.fy[j - 1], ryu - ryd, dr[1]);
        const bool xu = x + j < p.N2, xd = x - j >= 0;
        const float pxu = xu ? __ldg(p.pc + q + j) : 0.f, pxd = xd ? __ldg(p.pc + q - j) : 0.f;
        const float rxu = xu ? __ldg(p.rc + q + j) : 0.f, rxd = xd ? __ldg(p.rc + q - j) : 0.f;
        dp[2] = fmaf(p.fx[j - 1], pxu - pxd, dp[2]);
        dr[2] = fmaf(p.fx[j - 1], rxu - rxd, dr[2]);
    }
    const float a = __ldg(p.a + q), b = __ldg(p.b + q), c = __ldg(p.c + q);
    p.gp[q] = fmaf(a, dp[0], fmaf(b, dp[1], c * dp[2]));
    p.gr[q] = fmaf(a, dr[0], fmaf(b, dr[1], c * dr[2]));
}

// pass 2: Hz(p), Hz(r), L(p) and the leapfrog update of both fields
__global__ void __launch_bounds__(kTtiBX * kTtiBY)
tti_update_kernel(const __grid_constant__ TtiParams p) {
    const int x = blockIdx.x * kTtiBX + threadIdx.x;
    const int y = blockIdx.y * kTtiBY + threadIdx.y;
    const int z = blockIdx.z;
    if (x >= p.N2 || y >= p.N1) return;
    const long long q = (long long)(z + p.K) * p.plane + (long long)y * p.pitch + x;
    const long long k = (long long)z * p.plane + (long long)y * p.pitch + x;
    const float pcq = __ldg(p.pc + q), rcq = __ldg(p.rc + q);
    float hzp = 0.f, hzr = 0.f, lap = p.c0 * pcq;
    for (int j = 1; j <= p.K; ++j) {
        {   // axis 0: ghost planes hold zeros (or the neighbour slab), no bounds needed
            const long long o = (long long)j * p.plane;
            const float nu = __ldg(p.a + q + o), nd = __ldg(p.a + q - o);
            hzp = fmaf(p.fz[j - 1], nu * __ldg(p.gp + q + o) - nd * __ldg(p.gp + q - o), hzp);
            hzr = fmaf(p.fz[j - 1], nu * __ldg(p.gr + q + o) - nd * __ldg(p.gr + q - o), hzr);
            lap = fmaf(p.lz[j - 1], __ldg(p.pc + q + o) + __ldg(p.pc + q - o), lap);
        }
        {
            const long long o = (long long)j * p.pitch;
            const bool u = y + j < p.N1, d = y - j >= 0;
            const float nu = u ? __ldg(p.b + q + o) : 0.f, nd = d ? __ldg(p.b + q - o) : 0.f;
            const float gpu_ = u ? __ldg(p.gp + q + o) : 0.f, gpd = d ? __ldg(p.gp + q - o) : 0.f;
            const float gru = u ? __ldg(p.gr + q + o) : 0.f, grd = d ? __ldg(p.gr + q - o) : 0.f;
            const float pu = u ? __ldg(p.pc + q + o) : 0.f, pd = d ? __ldg(p.pc + q - o) : 0.f;
            hzp = fmaf(p.fy[j - 1], nu * gpu_ - nd * gpd, hzp);
            hzr = fmaf(p.fy[j - 1], nu * gru - nd * grd, hzr);
            lap = fmaf(p.ly[j - 1], pu + pd, lap);
        }
        {
            const bool u = x + j < p.N2, d = x - j >= 0;
            const float nu = u ? __ldg(p.c + q + j) : 0.f, nd = d ? __ldg(p.c + q - j) : 0.f;
            const float gpu_ = u ? __ldg(p.gp + q + j) : 0.f, gpd = d ? __ldg(p.gp + q - j) : 0.f;
            const float gru = u ? __ldg(p.gr + q + j) : 0.f, grd = d ? __ldg(p.gr + q - j) : 0.f;
            const float pu = u ? __ldg(p.pc + q + j) : 0.f, pd = d ? __ldg(p.pc + q - j) : 0.f;
            hzp = fmaf(p.fx[j - 1], nu * gpu_ - nd * gpd, hzp);
            hzr = fmaf(p.fx[j - 1], nu * gru - nd * grd, hzr);
            lap = fmaf(p.lx[j - 1], pu + pd, lap);
        }
    }
    const float h0 = lap - hzp;
    const float e1 = __ldg(p.e1 + k), e2 = __ldg(p.e2 + k);
    const float rhs_p = fmaf(e1, h0, e2 * hzr);
    const float rhs_r = fmaf(e2, h0, hzr);
    const float rm = __ldg(p.rm + k);
    const float dmp = p.damp ? __ldg(p.damp + k) : (__ldg(p.dz + z) + __ldg(p.dy + y) + __ldg(p.dx + x));
    const float qq = dmp * rm * p.qscale;
    const float c1 = fast_rcp(1.f + qq), c2 = (1.f - qq) * c1;
    p.po[q] = fmaf(c1, fmaf(rm, rhs_p, 2.f * pcq), -c2 * p.po[q]);
    p.ro[q] = fmaf(c1, fmaf(rm, rhs_r, 2.f * rcq), -c2 * p.ro[q]);
}

// set-up: unit symmetry axis and Thomsen factors from the f64 inputs
__global__ void tti_setup_kernel(const double* __restrict__ eps, const double* __restrict__ delta,
                                 const double* __restrict__ theta, const double* __restrict__ phi,
                                 float* a, float* b, float* c, float* e1, float* e2,
                                 long long rows, int n2, int pitch, long long ghost_off) {
    const long long row = blockIdx.y * (long long)gridDim.z + blockIdx.z;
    if (row >= rows) return;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n2; x += gridDim.x * blockDim.x) {
        const long long s = row * n2 + x, d = row * pitch + x;
        double st, ct, sp, cp;
        sincos(theta[s], &st, &ct);
        sincos(phi[s], &sp, &cp);
        a[ghost_off + d] = (float)(st * cp);
        b[ghost_off + d] = (float)(st * sp);
        c[ghost_off + d] = (float)ct;
        e1[d] = (float)(1.0 + 2.0 * eps[s]);
        e2[d] = (float)sqrt(1.0 + 2.0 * delta[s]);
    }
}

}  // namespace sfb
