// acoustic_kernel.cuh -- space-order-k 3-D star-stencil step for the damped acoustic
// wave equation, sm_100a.
//
// Computes, for every owned node of one slab (the closed
// form the reference pins at proj/tests/test_compiler.cpp:80,84):
//     u[t+1] = ( L(u[t]) - m (u[t-1] - 2 u[t]) / dt^2 + damp u[t-1] / (2 dt) ) * inv0
// evaluated in the algebraically identical, better conditioned fp32 form
//     u[t+1] = c1 (2 u[t] + r L(u[t])) - c2 u[t-1],
//     r = dt^2/m,  q = damp r / (2 dt),  c1 = 1/(1+q),  c2 = (1-q) c1.
// The adjoint update (proj/src/seismic_ops.cpp:97-100) is the same expression with the
// roles of t-1 and t+1 swapped, so this kernel serves forward, adjoint and gradient.
//
// Data movement.  Every global read is a TMA box load (cp.async.bulk.tensor.3d) issued by
// one producer lane and landing in shared memory behind an mbarrier; out-of-grid elements
// are zero-filled by the TMA unit, which is the reference's zero halo
// (proj/include/sf/function.hpp:17).  u[t] is streamed along the slowest axis d0 in
// (d1,d2) tiles with a (K, KP) halo into a ring of NST planes; consumer threads keep the
// 2K+1 d0 neighbours of their four nodes in a register queue and read the in-plane
// neighbours of the centre plane from the ring.  u[t-1], r (and damp) tiles of the output
// plane go through a second, NAUX-deep ring, so they are prefetched NAUX planes ahead
// without holding registers.  u[t+1] overwrites u[t-1] in place with one 128-bit store.
// A node therefore costs its compulsory 20 bytes of HBM traffic (16 when damping is
// rebuilt from its three 1-D profiles).  Optional fused outputs: forward snapshot and the
// imaging condition grad -= u_saved * v.dt2 (proj/src/seismic_ops.cpp:132).
//
// Synchronisation.  full[s]: TMA completion of ring stage s (+ the aux stage issued with
// it).  done[i % NAUX]: all consumer warps finished the shared-memory reads of iteration
// i, which frees u plane i-K's stage and the aux stage of iteration i (NAUX = NST - K
// makes both the same event).  No block-wide barrier inside the plane loop.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace sfb {

constexpr int kMaxK = 8;

struct StencilCoef {
    float c0;           // w_0 * sum_d 1/h_d^2 over active axes
    float cx[kMaxK];    // w_j / h_2^2 (contiguous axis)
    float cy[kMaxK];    // w_j / h_1^2
    float cz[kMaxK];    // w_j / h_0^2 (streaming axis)
    float qscale;       // 1 / (2 dt)
    float inv_dt2;      // 1 / dt^2
};

struct StepParams {
    StencilCoef k;
    const float* dz;     // separable damping profiles: damp = dz[i0] + dy[i1] + dx[i2]
    const float* dy;
    const float* dx;
    float* uo;           // level being overwritten (ghost planes included)
    float* snap;         // optional copy of the new level (compact)
    const float* usave;  // optional saved forward level (compact) -> imaging
    float* grad;         // imaging accumulator (compact)
    int N1, N2;
    int pitch;           // floats per row (multiple of 4)
    long long plane;     // floats per plane
    int z_lo, z_hi;      // owned output planes [z_lo, z_hi) handled by this launch
    int chunk;           // output planes per block
    int z_jump;          // extra plane offset of blocks with blockIdx.z >= 1 (0 = contiguous):
                         // one launch covers the two boundary plane groups of a slab
    // fused halo push: distance (in floats, 0 = none) from a node of `uo` written by the
    // blocks with blockIdx.z == 0 / >= 1 to its mirror in the neighbouring slab's ghost planes
    // (peer memory).  Boundary launches only (a block's chunk is exactly one boundary plane
    // group).  A block-uniform offset instead of a second pointer: no per-thread register.
    long long peer_delta0;
    long long peer_delta1;
    // PUSH kernels: only the first `push_planes` output planes of a block are pushed (the
    // whole chunk in a boundary launch), and with desc_last the block with the highest
    // blockIdx.z sweeps its chunk DOWNWARDS, so that a launch over the whole slab produces --
    // and pushes -- both boundary plane groups first (single-launch slab step)
    int push_planes;
    int desc_last;
};

// the tensor maps of one launch: u[t] with halo box (u) and with plain box (f); u[t-1], r,
// damp with plain box
struct StepMaps {
    CUtensorMap u, f, o, r, d;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// Consumer release of a pipeline stage.  An mbarrier.arrive does NOT wait for earlier
// shared-memory loads of the warp that are still in flight (ptxas puts no scoreboard wait on
// it), and on B200 the producer's next TMA write was observed to overtake such a load: rows
// of a stage read one pipeline round too new, a run-to-run difference under load
// (tools/probe_determinism4.py).  So every release carries a register dependency on data the
// iteration loaded: `dep` must derive from every shared-memory load instruction of the
// iteration; it is masked with an opaque zero (blockDim.z - 1) into the barrier address.
__device__ __forceinline__ void mbar_release(uint64_t* bar, float dep) {
    const uint32_t zero = blockDim.z - 1u;
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                     smem_u32(bar) + (__float_as_uint(dep) & zero))
                 : "memory");
}
// Programmatic dependent launch: the kernels of the time loop are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so a kernel may start (barrier set-up,
// parameter loads) while its predecessor in the stream drains.  pdl_enter() lets the NEXT
// kernel start early and then waits until every earlier kernel has completed and its writes
// are visible: nothing a predecessor wrote may be touched before it.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar), ok;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(addr), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y,
                                            int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}
// 1/x: MUFU.RCP plus one Newton step (branch free; error below 1 ulp for x >= 1)
__device__ __forceinline__ float fast_rcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return fmaf(y, fmaf(-x, y, 1.f), y);
}

// L(u) for the four nodes of a thread: d0 neighbours from the register queue, d1/d2
// neighbours from the haloed centre box `cp` in shared memory (16-byte loads only).
// Packed fp32 pairs (Blackwell FADD2 / FMUL2 / FFMA2): one issue slot for two nodes.  The
// kernels are issue-bound at high order, not FMA-pipe-bound, so the d0 and d1 parts of the
// stencil -- whose operands are register-aligned pairs -- run packed.  Results are the same
// IEEE roundings as the scalar instructions.
__device__ __forceinline__ float2 f2_add(float2 a, float2 b) {
    unsigned long long ra, rb, rd;
    asm("mov.b64 %0, {%1, %2};" : "=l"(ra) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(rb) : "f"(b.x), "f"(b.y));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(rd) : "l"(ra), "l"(rb));
    float2 d;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(rd));
    return d;
}
__device__ __forceinline__ float2 f2_sub(float2 a, float2 b) {
    unsigned long long ra, rb, rd;
    asm("mov.b64 %0, {%1, %2};" : "=l"(ra) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(rb) : "f"(b.x), "f"(b.y));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(rd) : "l"(ra), "l"(rb));
    float2 d;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(rd));
    return d;
}
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b) {
    unsigned long long ra, rb, rd;
    asm("mov.b64 %0, {%1, %2};" : "=l"(ra) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(rb) : "f"(b.x), "f"(b.y));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(rd) : "l"(ra), "l"(rb));
    float2 d;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(rd));
    return d;
}
__device__ __forceinline__ float2 f2_fma(float2 a, float2 b, float2 c) {
    unsigned long long ra, rb, rc, rd;
    asm("mov.b64 %0, {%1, %2};" : "=l"(ra) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(rb) : "f"(b.x), "f"(b.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(rc) : "f"(c.x), "f"(c.y));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
    float2 d;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(rd));
    return d;
}
__device__ __forceinline__ float2 f2_splat(float v) { return make_float2(v, v); }

// The register queue is addressed through a compile-time rotation ROT: logical plane i of
// the queue lives in q[(i + ROT) % (2K+1)].  Kernels that shift the queue every iteration
// use ROT = 0; the unrolled-rotation kernels advance ROT instead of moving registers.
// A queue array with more than 2K+1 slots is a sliding window instead: logical plane i lives
// in q[i + ROT] (the unrolled-by-two kernels, which shift by two planes every second plane).
template <int K, int KP, int SW, int ROT = 0, int QN = 2 * K + 1>
__device__ __forceinline__ void stencil_acc(const StencilCoef& k, const float (&q)[QN][4],
                                            const float* cp, int tx, int ty, float (&acc)[4]) {
        constexpr int Q = 2 * K + 1;
#define SFB_Q(i) q[QN == Q ? ((i) + ROT) % Q : (i) + ROT]
        // centre and streaming-axis neighbours from the register queue, two nodes per op
        float2 a01 = f2_mul(f2_splat(k.c0), make_float2(SFB_Q(K)[0], SFB_Q(K)[1]));
        float2 a23 = f2_mul(f2_splat(k.c0), make_float2(SFB_Q(K)[2], SFB_Q(K)[3]));
#pragma unroll
        for (int j = 1; j <= K; ++j) {
            const float2 w = f2_splat(k.cz[j - 1]);
            a01 = f2_fma(w, f2_add(make_float2(SFB_Q(K - j)[0], SFB_Q(K - j)[1]),
                                   make_float2(SFB_Q(K + j)[0], SFB_Q(K + j)[1])), a01);
            a23 = f2_fma(w, f2_add(make_float2(SFB_Q(K - j)[2], SFB_Q(K - j)[3]),
                                   make_float2(SFB_Q(K + j)[2], SFB_Q(K + j)[3])), a23);
        }
        // d1 neighbours: the column strip above and below (aligned pairs again)
        {
            const float* colp = cp + ty * SW + KP + 4 * tx;
#pragma unroll
            for (int j = 1; j <= K; ++j) {
                const float4 lo = *reinterpret_cast<const float4*>(colp + (K - j) * SW);
                const float4 hi = *reinterpret_cast<const float4*>(colp + (K + j) * SW);
                const float2 w = f2_splat(k.cy[j - 1]);
                a01 = f2_fma(w, f2_add(make_float2(lo.x, lo.y), make_float2(hi.x, hi.y)), a01);
                a23 = f2_fma(w, f2_add(make_float2(lo.z, lo.w), make_float2(hi.z, hi.w)), a23);
            }
        }
        // contiguous-axis neighbours: one aligned row segment.  For even j the operand pairs
        // (xr[KP+c-j], xr[KP+c+1-j]), c = 0, 2, are register-aligned pairs of the loaded
        // float4s and run packed; for odd j they straddle two pairs and stay scalar.  Each
        // node still accumulates j = 1 .. K in order with the same roundings.
        float2 x01 = make_float2(0.f, 0.f), x23 = make_float2(0.f, 0.f);
        {
            float xr[2 * KP + 4];
            const float* rowp = cp + (ty + K) * SW + 4 * tx;
#pragma unroll
            for (int v = 0; v < (2 * KP + 4) / 4; ++v) {
                if (v == KP / 4) {  // own float4: already in the queue
#pragma unroll
                    for (int c = 0; c < 4; ++c) xr[4 * v + c] = SFB_Q(K)[c];
                } else {
                    const float4 t4 = *reinterpret_cast<const float4*>(rowp + 4 * v);
                    xr[4 * v + 0] = t4.x;
                    xr[4 * v + 1] = t4.y;
                    xr[4 * v + 2] = t4.z;
                    xr[4 * v + 3] = t4.w;
                }
            }
#pragma unroll
            for (int j = 1; j <= K; ++j) {
                if (j % 2 == 0) {
                    const float2 w = f2_splat(k.cx[j - 1]);
                    x01 = f2_fma(w, f2_add(make_float2(xr[KP - j], xr[KP + 1 - j]),
                                           make_float2(xr[KP + j], xr[KP + 1 + j])), x01);
                    x23 = f2_fma(w, f2_add(make_float2(xr[KP + 2 - j], xr[KP + 3 - j]),
                                           make_float2(xr[KP + 2 + j], xr[KP + 3 + j])), x23);
                } else {
                    x01.x = fmaf(k.cx[j - 1], xr[KP - j] + xr[KP + j], x01.x);
                    x01.y = fmaf(k.cx[j - 1], xr[KP + 1 - j] + xr[KP + 1 + j], x01.y);
                    x23.x = fmaf(k.cx[j - 1], xr[KP + 2 - j] + xr[KP + 2 + j], x23.x);
                    x23.y = fmaf(k.cx[j - 1], xr[KP + 3 - j] + xr[KP + 3 + j], x23.y);
                }
            }
        }
        a01 = f2_add(a01, x01);
        a23 = f2_add(a23, x23);
        acc[0] = a01.x;
        acc[1] = a01.y;
        acc[2] = a23.x;
        acc[3] = a23.y;
#undef SFB_Q
}

// One output plane for the four nodes of a thread: stencil from the register queue (d0)
// and the centre plane in shared memory `cp` (d1, d2), then -- after telling the producer
// that this iteration's shared-memory reads are over -- damping, leapfrog and the stores.
template <int K, int KP, int SW, bool SEP, int ROT = 0, bool PUSH = false, int QN = 2 * K + 1>
__device__ __forceinline__ void plane_update(const StepParams& p, const float (&q)[QN][4],
                                             const float* cp, int tx, int ty, float4 o4, float4 r4,
                                             float4 d4, const float (&dxy)[4], float dzv,
                                             bool warp_dxy, bool rin, bool lane0,
                                             uint64_t* done_bar, float* po, long long gc,
                                             bool push_now = false) {
        // physical slot of the centre plane
        constexpr int QC = QN == 2 * K + 1 ? (K + ROT) % (2 * K + 1) : K + ROT;
        float acc[4];
        stencil_acc<K, KP, SW, ROT, QN>(p.k, q, cp, tx, ty, acc);

        const float rv[4] = {r4.x, r4.y, r4.z, r4.w};
        const float ov[4] = {o4.x, o4.y, o4.z, o4.w};
        float dv[4] = {d4.x, d4.y, d4.z, d4.w};
        bool damped;
        if (SEP) {
            damped = warp_dxy || dzv != 0.f;
#pragma unroll
            for (int c = 0; c < 4; ++c) dv[c] = dxy[c] + dzv;
        } else {
            damped = __any_sync(0xffffffffu, (dv[0] + dv[1]) + (dv[2] + dv[3]) != 0.f);
        }
        float un[4];
        if (damped) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float qq = dv[c] * rv[c] * p.k.qscale;
                const float c1 = fast_rcp(1.f + qq);
                const float c2 = (1.f - qq) * c1;
                const float t = fmaf(rv[c], acc[c], 2.f * q[QC][c]);
                un[c] = fmaf(c1, t, -c2 * ov[c]);
            }
        } else {
            const float2 u01 = make_float2(q[QC][0], q[QC][1]), u23 = make_float2(q[QC][2], q[QC][3]);
            const float2 t01 = f2_fma(make_float2(rv[0], rv[1]), make_float2(acc[0], acc[1]),
                                      f2_add(u01, u01));
            const float2 t23 = f2_fma(make_float2(rv[2], rv[3]), make_float2(acc[2], acc[3]),
                                      f2_add(u23, u23));
            const float2 n01 = f2_add(t01, make_float2(-ov[0], -ov[1]));
            const float2 n23 = f2_add(t23, make_float2(-ov[2], -ov[3]));
            un[0] = n01.x;
            un[1] = n01.y;
            un[2] = n23.x;
            un[3] = n23.y;
        }
        // un[0] depends on every shared-memory load of this iteration (queue feed, centre
        // box row and columns, aux boxes): the stage may be refilled once it is known
        __syncwarp();
        if (lane0) mbar_release(done_bar, un[0]);
        if (rin) {
            __stcs(reinterpret_cast<float4*>(po), make_float4(un[0], un[1], un[2], un[3]));
            // PUSH kernels (boundary launches of linked slabs): the same plane goes straight
            // into the neighbour's ghost planes over NVLink.  A separate instantiation: even a
            // never-taken branch here costs the issue-bound kernels 2-3 %.
            if constexpr (PUSH) {
                // low plane group: block z = 0; high plane group: the last block
                const long long peer_delta =
                    blockIdx.z == 0 ? p.peer_delta0
                                    : (blockIdx.z == gridDim.z - 1 ? p.peer_delta1 : 0);
                if (peer_delta && push_now)
                    *reinterpret_cast<float4*>(po + peer_delta) =
                        make_float4(un[0], un[1], un[2], un[3]);
            }
            if (p.snap)
                __stcs(reinterpret_cast<float4*>(p.snap + gc),
                       make_float4(un[0], un[1], un[2], un[3]));
            if (p.usave) {
                const float4 g4 = __ldcs(reinterpret_cast<const float4*>(p.grad + gc));
                const float4 s4 = __ldcs(reinterpret_cast<const float4*>(p.usave + gc));
                float4 gn;
                gn.x = fmaf(-s4.x * p.k.inv_dt2, (un[0] - 2.f * q[QC][0]) + ov[0], g4.x);
                gn.y = fmaf(-s4.y * p.k.inv_dt2, (un[1] - 2.f * q[QC][1]) + ov[1], g4.y);
                gn.z = fmaf(-s4.z * p.k.inv_dt2, (un[2] - 2.f * q[QC][2]) + ov[2], g4.z);
                gn.w = fmaf(-s4.w * p.k.inv_dt2, (un[3] - 2.f * q[QC][3]) + ov[3], g4.w);
                __stcs(reinterpret_cast<float4*>(p.grad + gc), gn);
            }
        }
}

template <int K, int TXV, int TY, int NST, bool SEP>
struct StepShape {
    static constexpr int KP = (K + 3) & ~3;       // x halo rounded to a float4
    static constexpr int TX = TXV * 4;
    static constexpr int SW = TX + 2 * KP;        // ring row width (floats)
    static constexpr int SH = TY + 2 * K;         // ring rows
    static constexpr int BOX = SW * SH;           // floats moved per u box
    static constexpr int STAGE = ((BOX + 31) / 32) * 32;
    static constexpr int NAUX = NST - K;          // aux ring depth == planes of lookahead + 1
    static constexpr int NARR = SEP ? 2 : 3;      // aux arrays: u[t-1], r, (damp)
    static constexpr int ABOX = TX * TY;          // floats per aux box
    static constexpr int NCONS = TXV * TY;        // consumer threads, four nodes each
    static constexpr int NTHREADS = NCONS + 32;   // + producer warp
    static constexpr size_t SMEM =
        size_t(NST) * STAGE * 4 + size_t(NAUX) * NARR * ABOX * 4 + (NST + NAUX) * 8 + 128;
    static_assert(NCONS % 32 == 0, "tile shape");
    static_assert(NAUX >= 2, "need at least one plane of lookahead");
    static_assert((ABOX * 4) % 128 == 0, "aux boxes must keep 128-byte alignment");
};

template <int K, int TXV, int TY, int NST, bool SEP, bool PUSH = false>
__global__ void __launch_bounds__(StepShape<K, TXV, TY, NST, SEP>::NTHREADS)
acoustic_step_kernel(const __grid_constant__ StepMaps tm, const __grid_constant__ StepParams p) {
    using S = StepShape<K, TXV, TY, NST, SEP>;
    constexpr int KP = S::KP, SW = S::SW, STAGE = S::STAGE, Q = 2 * K + 1;
    constexpr int NAUX = S::NAUX, NARR = S::NARR, ABOX = S::ABOX, TX = S::TX;
    constexpr int NCW = S::NCONS / 32;

    extern __shared__ unsigned char smem_raw[];
    const uint32_t mis = smem_u32(smem_raw) & 127u;
    float* ring = reinterpret_cast<float*>(smem_raw + ((128u - mis) & 127u));
    float* aux = ring + NST * STAGE;
    uint64_t* full = reinterpret_cast<uint64_t*>(aux + NAUX * NARR * ABOX);
    uint64_t* done = full + NST;

    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int zb = p.z_lo + blockIdx.z * p.chunk + (blockIdx.z ? p.z_jump : 0);
    const int ze = min(zb + p.chunk, p.z_hi);
    const int nplanes = (ze - zb) + 2 * K;  // u buffer planes zb .. ze+2K-1 (ghost offset K)
    // sweep direction (PUSH kernels only): iteration n loads buffer plane zl0 + dir n and,
    // from n = 2K on, writes owned plane zo0 + dir (n - 2K).  The stencil is symmetric in
    // d0, so a downward sweep computes the same sums with the two queue halves swapped.
    const bool desc = PUSH && p.desc_last && gridDim.z > 1 && blockIdx.z == gridDim.z - 1;
    const int dir = desc ? -1 : 1;
    const int zl0 = desc ? ze - 1 + 2 * K : zb;
    const int zo0 = desc ? ze - 1 : zb;

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < NST; ++s) mbar_init(full + s, 1);
#pragma unroll
        for (int s = 0; s < NAUX; ++s) mbar_init(done + s, NCW);
        mbar_fence_init();
    }
    __syncthreads();
    pdl_enter();

    if (tid >= S::NCONS) {
        // ---- producer warp: one lane streams the planes of this block ----------------
        if (tid == S::NCONS) {
            int s = 0, a = 0, dph = 0;
            for (int n = 0; n < nplanes; ++n) {
                if (n >= NAUX) mbar_wait(done + a, dph);  // iteration n - NAUX is finished
                const bool out = n >= 2 * K;
                mbar_arrive_expect_tx(full + s, (S::BOX + (out ? NARR * ABOX : 0)) * 4);
                tma_load_3d(ring + s * STAGE, &tm.u, x0 - KP, y0 - K, zl0 + dir * n, full + s);
                if (out) {
                    // iteration n uses aux stage (n - 2K) % NAUX; 2K % NAUX is folded into a0
                    constexpr int A0 = (NAUX - (2 * K) % NAUX) % NAUX;
                    int as = a + A0;
                    if (as >= NAUX) as -= NAUX;
                    float* ad = aux + as * NARR * ABOX;
                    const int zo = zo0 + dir * (n - 2 * K);
                    tma_load_3d(ad, &tm.o, x0, y0, zo + K, full + s);
                    tma_load_3d(ad + ABOX, &tm.r, x0, y0, zo, full + s);
                    if (!SEP) tma_load_3d(ad + 2 * ABOX, &tm.d, x0, y0, zo, full + s);
                }
                if (++s == NST) s = 0;
                if (++a == NAUX) {
                    a = 0;
                    if (n >= NAUX) dph ^= 1;
                }
            }
        }
        return;
    }

    // ---- consumers -------------------------------------------------------------------
    const int tx = tid % TXV, ty = tid / TXV;
    const int x = x0 + 4 * tx, y = y0 + ty;
    const bool rin = x < p.N2 && y < p.N1;
    const bool lane0 = (tid & 31) == 0;

    float dxy[4] = {0.f, 0.f, 0.f, 0.f};
    bool warp_dxy = false;
    if (SEP) {
        if (rin) {
            const float4 dx4 = __ldg(reinterpret_cast<const float4*>(p.dx + x));
            const float dyv = __ldg(p.dy + y);
            dxy[0] = dx4.x + dyv;
            dxy[1] = dx4.y + dyv;
            dxy[2] = dx4.z + dyv;
            dxy[3] = dx4.w + dyv;
        }
        warp_dxy = __any_sync(0xffffffffu, (dxy[0] + dxy[1]) + (dxy[2] + dxy[3]) != 0.f);
    }

    float q[Q][4];
#pragma unroll
    for (int j = 0; j < Q; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c) q[j][c] = 0.f;

    const int own = (ty + K) * SW + KP + 4 * tx;  // own float4 inside a u stage
    const int aown = ty * TX + 4 * tx;            // own float4 inside an aux box
    int s = 0;
    uint32_t fph = 0;

    // prologue: the first 2K planes only fill the register queue
    for (int n = 0; n < 2 * K; ++n) {
        mbar_wait(full + s, fph);
        const float4 v = *reinterpret_cast<const float4*>(ring + s * STAGE + own);
#pragma unroll
        for (int j = 0; j < Q - 1; ++j)
#pragma unroll
            for (int c = 0; c < 4; ++c) q[j][c] = q[j + 1][c];
        q[Q - 1][0] = v.x;
        q[Q - 1][1] = v.y;
        q[Q - 1][2] = v.z;
        q[Q - 1][3] = v.w;
        __syncwarp();
        if (lane0) mbar_release(done + (n % NAUX), v.x);
        if (++s == NST) {
            s = 0;
            fph ^= 1;
        }
    }

    // running element offset of this thread's float4 in the output plane
    long long gc = (long long)zo0 * p.plane + (long long)y * p.pitch + x;  // compact arrays
    float* po = p.uo + gc + (long long)K * p.plane;
    const long long zstep = desc ? -p.plane : p.plane;
    int cs = K % NST;  // stage of the centre plane (plane K is the first centre)
    int as = 0;        // aux stage / done slot of this iteration: (n - 2K) % NAUX ...
    int ds = (2 * K) % NAUX;  // ... and n % NAUX
    float dzn = 0.f;
    if (SEP) dzn = __ldg(p.dz + zo0);

    for (int n = 2 * K; n < nplanes; ++n) {
        mbar_wait(full + s, fph);
        {
            const float4 v = *reinterpret_cast<const float4*>(ring + s * STAGE + own);
#pragma unroll
            for (int j = 0; j < Q - 1; ++j)
#pragma unroll
                for (int c = 0; c < 4; ++c) q[j][c] = q[j + 1][c];
            q[Q - 1][0] = v.x;
            q[Q - 1][1] = v.y;
            q[Q - 1][2] = v.z;
            q[Q - 1][3] = v.w;
        }
        const float* ap = aux + as * NARR * ABOX + aown;
        const float4 o4 = *reinterpret_cast<const float4*>(ap);
        const float4 r4 = *reinterpret_cast<const float4*>(ap + ABOX);
        float4 d4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (!SEP) d4 = *reinterpret_cast<const float4*>(ap + 2 * ABOX);
        const float dzv = dzn;
        if (SEP && n + 1 < nplanes) dzn = __ldg(p.dz + (zo0 + dir * (n + 1 - 2 * K)));

        plane_update<K, KP, SW, SEP, 0, PUSH>(p, q, ring + cs * STAGE, tx, ty, o4, r4, d4, dxy, dzv, warp_dxy,
                                     rin, lane0, done + ds, po, gc, PUSH && n - 2 * K < p.push_planes);
        po += zstep;
        gc += zstep;
        if (++s == NST) {
            s = 0;
            fph ^= 1;
        }
        if (++cs == NST) cs = 0;
        if (++as == NAUX) as = 0;
        if (++ds == NAUX) ds = 0;
    }
}

// ---------------------------------------------------------------------------------------
// "Dual-stream" variant.  The ring kernel above keeps every plane between the newest and
// the centre one in shared memory (NST = K + 3 haloed stages), which at high order leaves
// room for a single block per SM.  Here a plane of u[t] is fetched twice instead: once as
// a plain TX x TY box when it is the newest plane (it only feeds the register queue) and
// once, K iterations later, as the haloed box when it is the centre plane (the second
// fetch hits L2: K planes of a few MB).  Everything an iteration needs -- feed box, centre
// box, aux boxes -- sits in ONE stage of an NS-deep ring, so shared memory no longer grows
// with K and one full/done barrier pair per stage orders it all.
template <int K, int TXV, int TY, int NS, bool SEP>
struct DualShape {
    static constexpr int KP = (K + 3) & ~3;
    static constexpr int TX = TXV * 4;
    static constexpr int SW = TX + 2 * KP;
    static constexpr int SH = TY + 2 * K;
    static constexpr int CBOX = SW * SH;                 // centre box (floats)
    static constexpr int CPAD = ((CBOX + 31) / 32) * 32;
    static constexpr int ABOX = TX * TY;                 // feed / aux box
    static constexpr int NARR = SEP ? 2 : 3;
    static constexpr int STAGE = ABOX + CPAD + NARR * ABOX;
    static constexpr int NCONS = TXV * TY;
    static constexpr int NTHREADS = NCONS + 32;
    static constexpr size_t SMEM = size_t(NS) * STAGE * 4 + 2 * NS * 8 + 128;
    static_assert(NCONS % 32 == 0 && (ABOX * 4) % 128 == 0 && NS >= 2, "tile shape");
};

template <int Q, int R, class F>
__device__ __forceinline__ void rotate_run(F& f, int& n, int nplanes) {
    if constexpr (R < Q) {
        if (n >= nplanes) return;
        f(std::integral_constant<int, R>{});
        ++n;
        rotate_run<Q, R + 1>(f, n, nplanes);
    }
}

// SLIDE: the queue is a window of 2K+2 slots; the plane loop is unrolled by two (plane n uses
// slots [0, 2K], plane n+1 slots [1, 2K+1]) and the window moves by two slots afterwards:
// half the register moves per plane of the plain shifting queue, two copies of the loop body
// instead of the 2K+1 of ROTATE.
template <int K, int TXV, int TY, int NS, bool SEP, int MINB, bool ROTATE, bool PUSH = false,
          bool SLIDE = false>
__global__ void __launch_bounds__(DualShape<K, TXV, TY, NS, SEP>::NTHREADS, MINB)
acoustic_step_dual_kernel(const __grid_constant__ StepMaps tm,
                          const __grid_constant__ StepParams p) {
    using S = DualShape<K, TXV, TY, NS, SEP>;
    static_assert(!(ROTATE && SLIDE), "one queue scheme at a time");
    constexpr int KP = S::KP, SW = S::SW, STAGE = S::STAGE, Q = 2 * K + 1;
#ifndef SFB_SLIDE_U
#define SFB_SLIDE_U 2
#endif
    constexpr int SU = SFB_SLIDE_U;               // planes per slide of the window
    constexpr int QN = SLIDE ? Q + SU - 1 : Q;
    constexpr int NARR = S::NARR, ABOX = S::ABOX, CPAD = S::CPAD, TX = S::TX;
    constexpr int NCW = S::NCONS / 32;

    extern __shared__ unsigned char smem_raw[];
    const uint32_t mis = smem_u32(smem_raw) & 127u;
    float* ring = reinterpret_cast<float*>(smem_raw + ((128u - mis) & 127u));
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + NS * STAGE);
    uint64_t* done = full + NS;

    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int zb = p.z_lo + blockIdx.z * p.chunk + (blockIdx.z ? p.z_jump : 0);
    const int ze = min(zb + p.chunk, p.z_hi);
    const int nplanes = (ze - zb) + 2 * K;
    // sweep direction (PUSH kernels only), see acoustic_step_kernel
    const bool desc = PUSH && p.desc_last && gridDim.z > 1 && blockIdx.z == gridDim.z - 1;
    const int dir = desc ? -1 : 1;
    const int zl0 = desc ? ze - 1 + 2 * K : zb;
    const int zo0 = desc ? ze - 1 : zb;

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            mbar_init(full + s, 1);
            mbar_init(done + s, NCW);
        }
        mbar_fence_init();
    }
    __syncthreads();
    pdl_enter();

    if (tid >= S::NCONS) {
        if (tid == S::NCONS) {
            int s = 0;
            uint32_t dph = 0;
            for (int n = 0; n < nplanes; ++n) {
                if (n >= NS) mbar_wait(done + s, dph);  // iteration n - NS released the stage
                const bool out = n >= 2 * K;
                float* st = ring + s * STAGE;
                mbar_arrive_expect_tx(full + s, (ABOX + (out ? S::CBOX + NARR * ABOX : 0)) * 4);
                tma_load_3d(st, &tm.f, x0, y0, zl0 + dir * n, full + s);       // newest plane
                if (out) {
                    const int zo = zo0 + dir * (n - 2 * K);
                    tma_load_3d(st + ABOX, &tm.u, x0 - KP, y0 - K, zo + K, full + s);  // centre
                    float* ad = st + ABOX + CPAD;
                    tma_load_3d(ad, &tm.o, x0, y0, zo + K, full + s);
                    tma_load_3d(ad + ABOX, &tm.r, x0, y0, zo, full + s);
                    if (!SEP) tma_load_3d(ad + 2 * ABOX, &tm.d, x0, y0, zo, full + s);
                }
                if (++s == NS) {
                    s = 0;
                    if (n >= NS) dph ^= 1;
                }
            }
        }
        return;
    }

    const int tx = tid % TXV, ty = tid / TXV;
    const int x = x0 + 4 * tx, y = y0 + ty;
    const bool rin = x < p.N2 && y < p.N1;
    const bool lane0 = (tid & 31) == 0;

    float dxy[4] = {0.f, 0.f, 0.f, 0.f};
    bool warp_dxy = false;
    if (SEP) {
        if (rin) {
            const float4 dx4 = __ldg(reinterpret_cast<const float4*>(p.dx + x));
            const float dyv = __ldg(p.dy + y);
            dxy[0] = dx4.x + dyv;
            dxy[1] = dx4.y + dyv;
            dxy[2] = dx4.z + dyv;
            dxy[3] = dx4.w + dyv;
        }
        warp_dxy = __any_sync(0xffffffffu, (dxy[0] + dxy[1]) + (dxy[2] + dxy[3]) != 0.f);
    }

    float q[QN][4];
#pragma unroll
    for (int j = 0; j < QN; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c) q[j][c] = 0.f;

    const int aown = ty * TX + 4 * tx;
    long long gc = (long long)zo0 * p.plane + (long long)y * p.pitch + x;
    float* po = p.uo + gc + (long long)K * p.plane;
    const long long zstep = desc ? -p.plane : p.plane;
    float dzn = 0.f;
    if (SEP) dzn = __ldg(p.dz + zo0);
    int s = 0;
    uint32_t fph = 0;

    // one plane: take the newest plane into the queue, and from iteration 2K on update one
    // output plane.  R is the queue rotation (compile-time in the unrolled variant).
    auto iteration = [&](auto rot, int n) {
        constexpr int R = decltype(rot)::value;
        mbar_wait(full + s, fph);
        const float* st = ring + s * STAGE;
        // logical slot Q-1 (newest) under the rotation / window offset of this iteration
        constexpr int NEW = SLIDE ? Q - 1 + R : (Q - 1 + R) % Q;
        {
            const float4 v = *reinterpret_cast<const float4*>(st + aown);
            if constexpr (!ROTATE && !SLIDE) {
#pragma unroll
                for (int j = 0; j < Q - 1; ++j)
#pragma unroll
                    for (int c = 0; c < 4; ++c) q[j][c] = q[j + 1][c];
            }
            q[NEW][0] = v.x;
            q[NEW][1] = v.y;
            q[NEW][2] = v.z;
            q[NEW][3] = v.w;
        }
        if (n < 2 * K) {
            __syncwarp();
            if (lane0) mbar_release(done + s, q[NEW][0]);
        } else {
            const float* ap = st + ABOX + CPAD + aown;
            const float4 o4 = *reinterpret_cast<const float4*>(ap);
            const float4 r4 = *reinterpret_cast<const float4*>(ap + ABOX);
            float4 d4 = make_float4(0.f, 0.f, 0.f, 0.f);
            if (!SEP) d4 = *reinterpret_cast<const float4*>(ap + 2 * ABOX);
            const float dzv = dzn;
            if (SEP && n + 1 < nplanes) dzn = __ldg(p.dz + (zo0 + dir * (n + 1 - 2 * K)));
            plane_update<K, KP, SW, SEP, R, PUSH, QN>(p, q, st + ABOX, tx, ty, o4, r4, d4, dxy, dzv,
                                                warp_dxy, rin, lane0, done + s, po, gc,
                                                PUSH && n - 2 * K < p.push_planes);
            po += zstep;
            gc += zstep;
        }
        if (++s == NS) {
            s = 0;
            fph ^= 1;
        }
    };
    if constexpr (ROTATE) {
        // unrolled by 2K+1: iteration i of a round sees the queue rotated by i+1 (the slot
        // of the oldest plane is overwritten by the newest), so no register moves at all
        int n = 0;
        while (n < nplanes) {
            auto step = [&](auto r) { iteration(std::integral_constant<int, (decltype(r)::value + 1) % Q>{}, n); };
            rotate_run<Q, 0>(step, n, nplanes);
        }
    } else if constexpr (SLIDE) {
        for (int n = 0; n < nplanes; n += SU) {
            iteration(std::integral_constant<int, 0>{}, n);
            if (n + 1 < nplanes) iteration(std::integral_constant<int, 1>{}, n + 1);
            if constexpr (SU > 2) {
                if (n + 2 < nplanes) iteration(std::integral_constant<int, 2>{}, n + 2);
            }
            if constexpr (SU > 3) {
                if (n + 3 < nplanes) iteration(std::integral_constant<int, 3>{}, n + 3);
            }
#pragma unroll
            for (int j = 0; j < Q - 1; ++j)
#pragma unroll
                for (int c = 0; c < 4; ++c) q[j][c] = q[j + SU][c];
        }
    } else {
        for (int n = 0; n < nplanes; ++n) iteration(std::integral_constant<int, 0>{}, n);
    }
}

}  // namespace sfb
