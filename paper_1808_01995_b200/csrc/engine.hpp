// engine.hpp -- internal interface of the host logic behind the C-ABI (not installed): plan
// set-up and data movement (engine_setup.cu), the acoustic time loops (engine_step.cu), the
// TTI time loop (engine_tti.cu).  capi.cu holds the extern "C" layer only.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "fdweights.hpp"
#include "plan.hpp"

namespace sfb {

// ---- error plumbing: no exception crosses the ABI ------------------------------------------
extern thread_local std::string g_create_err;   // last error of calls that have no plan yet

template <typename F>
int guarded(sfb_plan* plan, F&& f) {
    try {
        if (plan) {
            cudaError_t e = cudaSetDevice(plan->device);
            if (e != cudaSuccess)
                throw Failure(SFB_ERR_CAPABILITY,
                              std::string("cudaSetDevice: ") + cudaGetErrorString(e));
        }
        f();
        return SFB_OK;
    } catch (const Failure& e) {
        (plan ? plan->err : g_create_err) = e.what();
        return e.code;
    } catch (const std::exception& e) {
        (plan ? plan->err : g_create_err) = e.what();
        return SFB_ERR_CUDA;
    }
}

inline void require(bool ok, int code, const char* msg) {
    if (!ok) throw Failure(code, msg);
}

inline long long round_up(long long v, long long m) { return (v + m - 1) / m * m; }

// ---- engine_setup.cu: tensor maps, tile choice, field / trace movement, point tables -------
struct IntView {
    const double* ptr;
    long long s[3];
};

void make_tensor_maps(Plan& P);
// dual: -1 any, 0 ring kernel, 1 dual-stream, 2 dual-stream with the rotated (unrolled) queue
void select_variant(Plan& P, int txv, int ty, int nst, int dual = -1);
void encode_map(CUtensorMap* tm, void* base, long long n2, long long n1, long long n0,
                long long pitch, long long plane, int box_w, int box_h);
IntView embed_view(const Plan& P, const double* ptr, const int64_t* stride);
void upload_f64_planes(Plan& P, const IntView& v, DevBuf& tmp, long long gz0, long long cnt);
void upload_f64(Plan& P, const IntView& v, DevBuf& tmp);
void download_f64(Plan& P, const DevBuf& tmp, double* ptr, const int64_t* stride);
dim3 row_grid(const Plan& P, long long rows);
void download_field(Plan& P, const float* dev, const sfb_field_mview* out);
void detect_separable_damping(Plan& P, const IntView& v, const DevBuf& damp_f64, long long ref_plane);
void build_cloud(Plan& P, Cloud& c);
constexpr size_t kStageBytes = 32u << 20;  // per half
// sampled rows leave the device in chunks of about this size while the loop runs: small enough
// that the copy and the host-side widening of a chunk hide behind the next steps and the tail
// after the last step is short (a 592^3 step is 0.54 ms, a row of 512 x 512 traces 1 MB;
// measured on configs[1] over 20 steps: 4 MB chunks leave 1.0 ms outside the loop, 1 MB 0.78)
constexpr size_t kRowChunkBytes = 1u << 20;

template <typename Fn>
void parallel_chunks(long long n, Fn&& fn) {
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const unsigned nthr = unsigned(std::max<long long>(1, std::min<long long>(hw, n / 65536)));
    if (nthr <= 1) {
        fn(0, n);
        return;
    }
    std::vector<std::thread> pool;
    const long long per = (n + nthr - 1) / nthr;
    for (unsigned i = 0; i < nthr; ++i) {
        const long long b = i * per, e = std::min(n, b + per);
        if (b < e) pool.emplace_back([=, &fn] { fn(b, e); });
    }
    for (auto& t : pool) t.join();
}

void widen(const float* src, double* dst, long long n);
void narrow(const double* src, float* dst, long long n);
void upload_f32(Plan& P, const double* host, float* dev, long long n);
void download_f32(Plan& P, const float* dev, double* host, long long n);
void upload_traces(Plan& P, Cloud& c, const double* host);
void download_traces(Plan& P, Cloud& c, double* host);

// ---- engine_step.cu: the acoustic time loops --------------------------------------------------
struct OpRoles {
    bool backward;
    int inj, smp;  // cloud indices, -1 = none
    bool imaging;
};

OpRoles roles(int op);
constexpr int kPartBoundaryPair = 100;   // internal: LOW and HIGH plane groups in one launch
// internal: the whole slab in ONE push launch -- chunk 0 sweeps up, the last chunk sweeps down,
// so both boundary plane groups are computed and pushed first (sfb_step_slab_fused)
constexpr int kPartSlabFused = 101;
int fused_chunk(const Plan& P);

// explicit fused outputs / buffer set of one step (checkpointed runs); without it the
// save_every rules of the plain runs apply
struct StepExtras {
    bool alt = false;            // step the recompute pair f[2] instead of u[2]
    float* snap = nullptr;       // copy of the new level
    const float* usave = nullptr;  // forward level to image against
};

void step_begin(Plan& P, int op, long long save_every);
void part_range(const Plan& P, int part, int& lo, int& hi);
cudaStream_t part_stream(Plan& P, int part);
void mark_stream(Plan& P, int part);
void step_compute(Plan& P, int op, long long t, int part, const StepExtras* ex = nullptr);
// part: SFB_PART_ALL = every node + gather; SFB_PART_LOW = nodes of both boundary plane
// groups (boundary stream); SFB_PART_INTERIOR = remaining nodes + gather
// peer_lo / peer_hi: with a target override, the neighbours' ghost planes of THAT field (the
// TTI pair injects into r as well); without one the plan's own peer pointers are used
void step_points(Plan& P, int op, long long t, int part, float* target_override = nullptr,
                 bool allow_gather = true, const StepExtras* ex = nullptr,
                 float* peer_lo = nullptr, float* peer_hi = nullptr);
// only >= 0: scan that wavefield buffer alone (the level computed last)
void finite_guard(Plan& P, const char* what, int only = -1);
// Streams the sampled trace rows to the caller's f64 table while the time loop runs: every
// `rows` completed rows are copied (fp32, copy stream, pinned half) and the previous chunk
// is widened on host threads in the shadow of the GPU.
struct RowStreamer {
    Plan& P;
    Cloud& c;
    double* host;
    long long rows;            // rows per chunk
    long long lo = -1, hi = -1;  // rows gathered since the last flush
    int b = 0;
    long long pend_row[2] = {0, 0}, pend_rows[2] = {0, 0};

    RowStreamer(Plan& p, Cloud& cl, double* h) : P(p), c(cl), host(h) {
        rows = std::max<long long>(1, (long long)(kRowChunkBytes / 4) / std::max<long long>(c.np, 1));
        P.stage.ensure(size_t(rows * c.np));
    }
    void drain(int i) {
        if (!pend_rows[i]) return;
        SFB_CUDA(cudaEventSynchronize(P.stage.moved[i]));
        widen(P.stage.p[i], host + pend_row[i] * c.np, pend_rows[i] * c.np);
        pend_rows[i] = 0;
    }
    void flush() {
        if (lo < 0) return;
        PinnedStage& st = P.stage;
        SFB_CUDA(cudaEventRecord(st.ready[b], P.s_main));
        SFB_CUDA(cudaStreamWaitEvent(st.copy, st.ready[b], 0));
        SFB_CUDA(cudaMemcpyAsync(st.p[b], c.tr_out.as<float>() + lo * c.np,
                                 size_t((hi - lo + 1) * c.np) * 4, cudaMemcpyDeviceToHost, st.copy));
        SFB_CUDA(cudaEventRecord(st.moved[b], st.copy));
        pend_row[b] = lo;
        pend_rows[b] = hi - lo + 1;
        lo = hi = -1;
        b ^= 1;
        drain(b);  // the half we are about to reuse: its copy was queued a chunk ago
    }
    void row_done(long long t) {
        lo = lo < 0 ? t : std::min(lo, t);
        hi = hi < 0 ? t : std::max(hi, t);
        if (hi - lo + 1 >= rows) flush();
    }
    void finish() {
        flush();
        drain(0);
        drain(1);
        // rows 0 and nt-1 are never sampled (structural zeros, seismic_ops.hpp:13-16)
        std::fill(host, host + c.np, 0.0);
        if (P.desc.nt > 1) std::fill(host + (P.desc.nt - 1) * c.np, host + P.desc.nt * c.np, 0.0);
    }
};

// The mirror image for the injected cloud: a table of many traces (the receiver data of an
// adjoint run or a gradient sweep) reaches the device chunk by chunk in sweep order, one chunk
// ahead of the step that injects it (narrowed on the host, copy stream, pinned halves of its
// own), instead of as a whole before the first step.
struct RowFeeder {
    Plan& P;
    Cloud& c;
    const double* host;
    bool backward;
    long long rows, next;      // rows per chunk; next row to send, in sweep order
    long long first, last;     // rows the run reads: [first, last] (default: 1 .. nt - 2)
    int b = 0;
    bool used[2] = {false, false};

    RowFeeder(Plan& p, Cloud& cl, const double* h, bool back, long long row_first = 1,
              long long row_last = -1)
        : P(p), c(cl), host(h), backward(back), first(row_first),
          last(row_last < 0 ? p.desc.nt - 2 : row_last) {
        rows = std::max<long long>(1, (long long)(kRowChunkBytes / 4) / std::max<long long>(c.np, 1));
        next = backward ? last : first;
        P.stage_in.ensure(size_t(rows * c.np));
    }
    ~RowFeeder() {
        if (more()) c.has_in = false;   // a run that failed half-way leaves a partial table
    }
    bool more() const { return backward ? next >= first : next <= last; }
    void send() {
        long long lo, hi;
        if (backward) {
            hi = next;
            lo = std::max<long long>(first, hi - rows + 1);
            next = lo - 1;
        } else {
            lo = next;
            hi = std::min<long long>(last, lo + rows - 1);
            next = hi + 1;
        }
        PinnedStage& st = P.stage_in;
        if (used[b]) SFB_CUDA(cudaEventSynchronize(st.moved[b]));
        narrow(host + lo * c.np, st.p[b], (hi - lo + 1) * c.np);
        SFB_CUDA(cudaMemcpyAsync(c.tr_in.as<float>() + lo * c.np, st.p[b],
                                 size_t((hi - lo + 1) * c.np) * 4, cudaMemcpyHostToDevice, st.copy));
        SFB_CUDA(cudaEventRecord(st.moved[b], st.copy));
        SFB_CUDA(cudaStreamWaitEvent(P.s_main, st.moved[b], 0));   // later launches see the rows
        used[b] = true;
        b ^= 1;
    }
    // the rows of step t, and the chunk after them, are on their way
    void before_step(long long t) {
        while (more() && (backward ? next >= t - rows : next <= t + rows)) send();
    }
    void finish() {
        while (more()) send();
        c.has_in = true;
    }
};

// stream_out: the sampled table goes to this host table while the loop runs; stream_in: the
// injected table comes from this host table while the loop runs (else it is resident already)
void run_op(Plan& P, int op, long long save_every, sfb_report* rep, double* stream_out = nullptr,
            const double* stream_in = nullptr);
void run_window(Plan& P, int op, long long t_from, long long t_to, bool with_points,
                sfb_report* report);
void forward_checkpointed(Plan& P, long long C, sfb_report* rep, double* stream_out);
void gradient_checkpointed(Plan& P, sfb_report* rep);

// ---- engine_tti.cu: the TTI time loop -----------------------------------------------------------
void tti_make_maps(Plan& P);
void tti_begin(Plan& P);
void tti_rot(Plan& P, long long t, int part);
void tti_update(Plan& P, long long t, int part, bool with_points = true);
void run_tti(Plan& P, sfb_report* rep, double* stream_out);

}  // namespace sfb
