// point_kernels.cuh -- sparse source injection and receiver sampling, sm_100a.
//
// Scatter: SparseFunction::inject as used by the operators (proj/src/sparse.cpp:138-150,
// proj/src/seismic_ops.cpp:74-76,101-103,129-131):
//     field(base_p + bits c) += trace[t][p] * w[p][c] * dt^2 / m(base_p + bits c)
// The reference runs it serially, point-major / corner-minor (proj/src/lower.cpp:198).
// Here the (point, corner) pairs are regrouped once, on the host, by destination node
// (CSR, entries of a node kept in the reference's order), so one thread owns one node:
// no atomics, results independent of scheduling, same summation order per node.
//
// Gather: SparseFunction::interpolate (proj/src/sparse.cpp:130-136,
// proj/src/seismic_ops.cpp:77,104):  trace[t][p] = sum_c w[p][c] * field(base_p + bits c).
#pragma once

#include <cuda_runtime.h>

namespace sfb {

struct PointParams {
    // scatter
    int ncell;                    // nodes handled by this launch
    const int* cell_start;        // [ncell+1] entry ranges (already offset to the launch range)
    const long long* cell_u;      // node index inside a wavefield buffer (ghost planes included)
    const long long* cell_c;      // node index inside compact arrays (r, snap, usave, grad)
    const int* ent_point;         // entry -> point
    const float* ent_w;           // entry -> weight
    const float* inj_row;         // trace row t of the injected cloud
    float* target;                // level being injected
    const float* r;               // dt^2/m
    float* snap;                  // optional snapshot copy of target
    const float* usave;           // optional: imaging correction for the injected amount
    float* grad;
    float inv_dt2;
    // fused halo push: an injected node of a boundary plane group is mirrored into the
    // neighbour's ghost plane (peer memory), like the planes themselves
    float* peer_lo;               // neighbour below: its high ghost planes
    float* peer_hi;               // neighbour above: its low ghost planes
    long long plane;              // floats per plane
    int K, n0;
    // gather
    int nsmp;
    const long long* smp_idx;     // base node index inside a wavefield buffer, -1 = not owned
    const float* smp_w;           // [nsmp][ncorner]
    const float* field;           // level t
    float* smp_row;               // trace row t of the sampled cloud
    int ncorner;
    long long corner_off[8];
};

constexpr int kPointThreads = 128;

// blocks [0, nb_inj) scatter, the rest gather
static __global__ void __launch_bounds__(kPointThreads)
point_step_kernel(const __grid_constant__ PointParams p, int nb_inj) {
    // launched with programmatic stream serialization (see pdl_enter in acoustic_kernel.cuh)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if ((int)blockIdx.x < nb_inj) {
        const int i = blockIdx.x * kPointThreads + threadIdx.x;
        if (i >= p.ncell) return;
        const int e0 = p.cell_start[i], e1 = p.cell_start[i + 1];
        float s = 0.f;
        for (int e = e0; e < e1; ++e) s = fmaf(p.ent_w[e], p.inj_row[p.ent_point[e]], s);
        const long long cu = p.cell_u[i], cc = p.cell_c[i];
        const float add = s * p.r[cc];
        const float v = __ldcg(p.target + cu) + add;
        p.target[cu] = v;
        if (p.peer_lo || p.peer_hi) {
            const long long zb = cu / p.plane;   // buffer plane: owned plane z sits at z + K
            if (p.peer_lo && zb < 2 * p.K) p.peer_lo[cu - (long long)p.K * p.plane] = v;
            if (p.peer_hi && zb >= p.n0) p.peer_hi[cu - (long long)p.n0 * p.plane] = v;
        }
        if (p.snap) p.snap[cc] = __ldcg(p.snap + cc) + add;
        if (p.usave)
            p.grad[cc] = fmaf(-__ldcg(p.usave + cc) * p.inv_dt2, add, __ldcg(p.grad + cc));
    } else {
        const int i = (blockIdx.x - nb_inj) * kPointThreads + threadIdx.x;
        if (i >= p.nsmp) return;
        const long long b = p.smp_idx[i];
        float s = 0.f;
        if (b >= 0) {
            const float* w = p.smp_w + (long long)i * p.ncorner;
            // corners with zero weight (points on lattice lines) are not fetched
            for (int c = 0; c < p.ncorner; ++c) {
                const float wc = w[c];
                if (wc != 0.f) s = fmaf(wc, __ldcg(p.field + b + p.corner_off[c]), s);
            }
        }
        p.smp_row[i] = s;
    }
}

// ---- setup / conversion kernels ------------------------------------------------------

// r = dt^2 / m evaluated in f64, stored fp32 in the pitched device layout
static __global__ void convert_r_kernel(const double* __restrict__ m, float* __restrict__ r,
                                 long long rows, int n2, int pitch, double dt2) {
    const long long row = blockIdx.y * (long long)gridDim.z + blockIdx.z;
    if (row >= rows) return;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n2; x += gridDim.x * blockDim.x)
        r[row * pitch + x] = (float)(dt2 / m[row * n2 + x]);
}

static __global__ void convert_f64_f32_pitched(const double* __restrict__ src, float* __restrict__ dst,
                                        long long rows, int n2, int pitch) {
    const long long row = blockIdx.y * (long long)gridDim.z + blockIdx.z;
    if (row >= rows) return;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n2; x += gridDim.x * blockDim.x)
        dst[row * pitch + x] = (float)src[row * n2 + x];
}

static __global__ void convert_f32_pitched_f64(const float* __restrict__ src, double* __restrict__ dst,
                                        long long rows, int n2, int pitch) {
    const long long row = blockIdx.y * (long long)gridDim.z + blockIdx.z;
    if (row >= rows) return;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n2; x += gridDim.x * blockDim.x)
        dst[row * n2 + x] = (double)src[row * pitch + x];
}

// fp32 pitched rows -> fp32 compact rows
static __global__ void pack_f32_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                       long long rows, int n2, int pitch) {
    const long long row = blockIdx.y * (long long)gridDim.z + blockIdx.z;
    if (row >= rows) return;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n2; x += gridDim.x * blockDim.x)
        dst[row * n2 + x] = src[row * pitch + x];
}

static __global__ void convert_f64_f32_flat(const double* __restrict__ src, float* __restrict__ dst,
                                     long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        dst[i] = (float)src[i];
}

static __global__ void convert_f32_f64_flat(const float* __restrict__ src, double* __restrict__ dst,
                                     long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        dst[i] = (double)src[i];
}

// NaN/Inf guard of the reference engines (proj/src/execute.cpp:397-417,
// proj/src/emit.cpp:333-341): flag = 1 if any value is non-finite
static __global__ void finite_check_kernel(const float* __restrict__ a, long long n, int* flag) {
    int bad = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        bad |= !isfinite(a[i]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

}  // namespace sfb
