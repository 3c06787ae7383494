/*
 * sfb200.h -- C-ABI of the B200-native wave-propagator engine (libsfb200.so).
 *
 * This is the drop-in boundary for ONE path of the reference ("sf", arXiv 1808.01995
 * re-creation): the time-stepping acoustic propagators behind
 *   forward_operator / adjoint_operator / gradient_operator / run_wave / run_gradient /
 *   fwi_gradient            (proj/include/sf/seismic_ops.hpp:28-73)
 * plus a TTI forward operator the reference does not have.
 *
 * What it replaces.  The reference chooses its engine in run_window
 * (proj/src/seismic_ops.cpp:44-54) and its only native seam is a C function loaded by
 * name,
 *   void sf_kernel(double** F, const double* S, const long** B, long t_from, long t_to)
 * (proj/src/emit.cpp:214-215,261,288): F = field base pointers, S = scalar symbols,
 * B = per-cloud base tables.  The entry points below carry the same information
 * explicitly (fields with strides, scalars by name, point tables) and run the whole
 * window [1, nt-1) on the GPU.  Plain pointers and sizes only; every function returns
 * an int status; no C++ exception crosses this boundary.  Host pointers are borrowed
 * for the duration of a call; device memory is owned by the plan.
 *
 * Conventions are the reference's: axes d0,d1,d2 = x,y,z row-major with the last axis
 * contiguous (proj/include/sf/function.hpp:15-17); metres, milliseconds, m/ms; corner
 * index c of a point uses axis 0 as least-significant bit (proj/include/sf/sparse.hpp:
 * 23-25); trace tables are [nt][npoints] (sparse.hpp:46-49); time level t of a buffered
 * field is reference slot t mod 3 (proj/src/execute.cpp:187-199).
 *
 * There is no CPU fallback: every compute entry point fails with SFB_ERR_CAPABILITY when
 * no sm_100 device is usable.
 */
#ifndef SFB200_H
#define SFB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFB_ABI_VERSION 1

#if defined(__GNUC__)
#define SFB_API __attribute__((visibility("default")))
#else
#define SFB_API
#endif

/* status codes; the C++ host layer maps them onto the sf::Error family
 * (proj/include/sf/error.hpp:9-59) */
enum {
    SFB_OK = 0,
    SFB_ERR_PARAMETER = 1,  /* sf::ParameterError  */
    SFB_ERR_STABILITY = 2,  /* sf::StabilityError: CFL violated or non-finite field */
    SFB_ERR_LOCATION = 3,   /* sf::LocationError   */
    SFB_ERR_CAPABILITY = 4, /* sf::CapabilityError: no usable device / kernel image */
    SFB_ERR_BINDING = 5,    /* sf::BindingError: model or point tables not set */
    SFB_ERR_CUDA = 6,       /* CUDA runtime failure (message in sfb_last_error) */
    SFB_ERR_ORDER = 7       /* sf::OrderError: unsupported space order */
};

typedef struct sfb_plan_s sfb_plan;

/* Grid + time axis of one operator.  Replaces Grid (proj/include/sf/grid.hpp:30-71) and
 * the dt/nt bindings of run_window (proj/src/seismic_ops.cpp:44-50). */
typedef struct {
    int32_t ndim;        /* 1..3 */
    int64_t shape[3];    /* computational (padded) node counts, reference axis order */
    double spacing[3];
    int32_t space_order; /* even, 2..16 */
    double dt;
    int64_t nt;          /* time samples; the window is [1, nt-1) */
    int32_t device;      /* CUDA ordinal */
    /* slab decomposition of the slowest axis of the 3-D embedding (new: the reference
     * is single-address-space).  The plan owns planes [slab_lo, slab_hi) of that axis
     * and keeps space_order/2 ghost planes per side; 0,0 means the whole axis. */
    int64_t slab_lo, slab_hi;
} sfb_plan_desc;

/* Strided view of a host f64 field (FunctionBase storage, proj/include/sf/function.hpp:
 * 35-73): ptr addresses interior node (0,..,0); stride[d] is in elements. */
typedef struct {
    const double* ptr;
    int64_t stride[3];
} sfb_field_view;

typedef struct {
    double* ptr;
    int64_t stride[3];
} sfb_field_mview;

/* mirrors ExecutionReport (proj/include/sf/execute.hpp:40-46); seconds = stepping loop
 * only, measured on the device. */
typedef struct {
    double seconds;
    long long flops;
    double gflops;
    long steps;
    double gpts_per_s;     /* shape[0]*shape[1]*shape[2]*steps / seconds / 1e9 */
    long kernel_launches;  /* launches issued inside the stepping loop */
} sfb_report;

enum { SFB_CLOUD_SRC = 0, SFB_CLOUD_REC = 1 };
enum { SFB_OP_FORWARD = 0, SFB_OP_ADJOINT = 1, SFB_OP_GRADIENT = 2, SFB_OP_TTI_FORWARD = 3 };

SFB_API int sfb_abi_version(void);
/* message of the last failure on this plan (or of the last failed create when NULL) */
SFB_API const char* sfb_last_error(const sfb_plan* plan);
SFB_API int sfb_device_count(int* count);

SFB_API int sfb_plan_create(const sfb_plan_desc* desc, sfb_plan** out);
SFB_API int sfb_plan_destroy(sfb_plan* plan);

/* exact centred second/first-derivative weights w_0..w_K the plan uses; replaces
 * fd_weights (proj/src/fdcoeff.cpp:60-95).  out must hold space_order/2 + 1 doubles. */
SFB_API int sfb_fd_weights(int deriv_order, int space_order, double* out);
/* CFL bound of SeismicModel::critical_dt (proj/src/model.cpp:103-111) */
SFB_API int sfb_critical_dt(int ndim, const double* spacing, double v_max, int space_order,
                    double* out);

/* m and damp of SeismicModel (proj/include/sf/model.hpp:33-34), any halo via strides.
 * v_max is the model's maximum velocity for the CFL gate of check_cfl
 * (proj/src/seismic_ops.cpp:15-22); pass 0 to skip the gate. */
SFB_API int sfb_set_model(sfb_plan* plan, const sfb_field_view* m, const sfb_field_view* damp,
                  double v_max);
/* the same for one slab of a decomposed run whose rank never holds the global fields: the
 * views cover the plan's own planes [slab_lo, slab_hi) only (plane 0 of the view = global
 * plane slab_lo).  Large weak-scaling runs (BASELINE.json configs[4]) build m and damp per
 * rank. */
SFB_API int sfb_set_model_slab(sfb_plan* plan, const sfb_field_view* m_slab,
                               const sfb_field_view* damp_slab, double v_max);
/* anisotropy fields of the TTI operator (no reference counterpart) */
SFB_API int sfb_set_model_tti(sfb_plan* plan, const sfb_field_view* epsilon,
                      const sfb_field_view* delta, const sfb_field_view* theta,
                      const sfb_field_view* phi);

/* point tables of SparseFunction::locate (proj/src/sparse.cpp:36-70):
 * base int64 [np][ndim], w f64 [np][2^ndim], indices global. */
SFB_API int sfb_set_points(sfb_plan* plan, int cloud, int64_t np, const int64_t* base,
                   const double* w);
/* locate on the plan's grid: coords [np][ndim] physical units, origin of the padded grid */
SFB_API int sfb_locate(const sfb_plan_desc* desc, const double* origin, int64_t np,
               const double* coords, int64_t* base, double* w);

/* forward_operator + run_wave (proj/src/seismic_ops.cpp:58-82,137-141).
 * src [nt][n_src] in; rec [nt][n_rec] out (rows 0, 1, nt-1 are zeros).
 * save_every > 0 keeps forward levels t % save_every == 0 in HBM for sfb_gradient
 * (save_every = 1 is the reference's save=true). */
SFB_API int sfb_forward(sfb_plan* plan, const double* src, double* rec, int64_t save_every,
                sfb_report* report);
/* the same forward run keeping only the state at every checkpoint_every-th level (>= 2);
 * sfb_gradient then recomputes the history one segment at a time and images against EVERY
 * level (the reference's exact imaging condition) without holding nt levels: the memory
 * strategy the reference leaves out of scope */
SFB_API int sfb_forward_checkpointed(sfb_plan* plan, const double* src, double* rec,
                                     int64_t checkpoint_every, sfb_report* report);
/* adjoint_operator + run_wave (seismic_ops.cpp:84-107): rec [nt][n_rec] in, srca
 * [nt][n_src] out. */
SFB_API int sfb_adjoint(sfb_plan* plan, const double* rec, double* srca, sfb_report* report);
/* gradient_operator + run_gradient (seismic_ops.cpp:109-135,143-147): resid [nt][n_rec]
 * in; grad over the padded grid out (written through the strided view).  Needs the
 * history of the last sfb_forward with save_every > 0. */
SFB_API int sfb_gradient(sfb_plan* plan, const double* resid, const sfb_field_mview* grad,
                 sfb_report* report);
/* TTI forward: src in, rec (sampled p) out. */
SFB_API int sfb_tti_forward(sfb_plan* plan, const double* src, double* rec, sfb_report* report);

/* wavefield of the last run at time level `level` (the two most recent levels, or any
 * saved level); field = 0 (u / v / p) or 1 (TTI r). */
SFB_API int sfb_get_wavefield(sfb_plan* plan, int field, int64_t level, const sfb_field_mview* out);

/* ---- device-resident variant (bench `value`; inputs already in HBM) ----------------
 * upload traces once, run any number of times, download when wanted. */
SFB_API int sfb_upload_traces(sfb_plan* plan, int cloud, const double* traces);
SFB_API int sfb_download_traces(sfb_plan* plan, int cloud, double* traces);
SFB_API int sfb_run_resident(sfb_plan* plan, int op, int64_t save_every, sfb_report* report);
/* steps t in [t_from, t_to) of an operator begun with sfb_step_begin, without touching the
 * state first (descending for the backward operators; SFB_OP_TTI_FORWARD runs its two
 * launches per step); timed on the device */
SFB_API int sfb_run_steps(sfb_plan* plan, int op, int64_t t_from, int64_t t_to,
                          sfb_report* report);
/* the same window with the dense update kernel alone (no scatter / gather launches):
 * report->seconds / report->steps is that kernel's average launch duration, which the
 * roofline figure of bench.py is computed from */
SFB_API int sfb_time_stencil(sfb_plan* plan, int op, int64_t t_from, int64_t t_to,
                             sfb_report* report);

/* ---- slab stepping (multi-GPU; the caller moves ghost planes between ranks) --------
 * One time step is: sfb_step_begin (zeroes state when t is the first step of the window),
 * sfb_step_compute(part) for the boundary planes then the interior, the caller's halo
 * exchange of the freshly written level, sfb_step_points (scatter + gather).
 * Pointers returned are device pointers into the plan's wavefield buffers. */
enum { SFB_PART_ALL = 0, SFB_PART_LOW = 1, SFB_PART_HIGH = 2, SFB_PART_INTERIOR = 3 };
SFB_API int sfb_step_begin(sfb_plan* plan, int op, int64_t save_every);
SFB_API int sfb_step_compute(sfb_plan* plan, int op, int64_t t, int part);
/* scatter (+ gather): part ALL = every node and the gather; LOW (or HIGH) = the nodes of
 * both boundary plane groups, on the boundary stream, so they are in place before the
 * planes are shipped; INTERIOR = the remaining nodes and the gather */
SFB_API int sfb_step_points(sfb_plan* plan, int op, int64_t t, int part);
/* the two halves of one slab step as single calls: boundary = compute LOW, compute HIGH,
 * points LOW (boundary stream); interior = compute INTERIOR, points INTERIOR (main stream) */
SFB_API int sfb_step_slab_boundary(sfb_plan* plan, int op, int64_t t);
SFB_API int sfb_step_slab_interior(sfb_plan* plan, int op, int64_t t);
SFB_API int sfb_step_end(sfb_plan* plan, int op);
/* binds one level of a forward history that lives in host memory (the reference's saved
 * TimeFunction, proj/src/seismic_ops.cpp:113-114) as saved level `level` for sfb_gradient;
 * levels that are never put stay zero */
SFB_API int sfb_put_history(sfb_plan* plan, int64_t save_every, int64_t level,
                            const sfb_field_view* u);
/* gradient accumulated by the last gradient sweep (owned planes only are written) */
SFB_API int sfb_get_gradient(sfb_plan* plan, const sfb_field_mview* grad);
/* ghost / boundary plane blocks of the level written at step t of `op`:
 * send_lo/send_hi = owned boundary planes to ship, recv_lo/recv_hi = ghost planes to
 * fill; each is `*count` contiguous floats. */
SFB_API int sfb_halo_blocks(sfb_plan* plan, int op, int64_t t, void** send_lo, void** send_hi,
                    void** recv_lo, void** recv_hi, int64_t* count);
/* ---- fused halo push (one process driving several slabs / GPUs).  After sfb_link_peers the
 * boundary half-step (sfb_step_slab_boundary) writes its K boundary planes -- and the nodes
 * injected into them -- directly into the neighbours' ghost planes as it computes them (peer
 * stores over NVLink): no copy, no send/recv.  Ordering is by events: before its next
 * step a plan calls sfb_peer_wait(plan, neighbour) for each neighbour, which makes both of
 * its streams wait for that neighbour's last boundary half-step (its pushes have landed) and
 * its boundary stream -- the one that stores into peer memory -- also for the neighbour's
 * last INTERIOR half-step, whose gather is the last reader of the ghost planes this plan
 * overwrites next (a receiver cell that straddles the cut reads one).  Acoustic
 * operators; lo / hi are the plans of the slabs below / above, or NULL at an outer face. */
SFB_API int sfb_link_peers(sfb_plan* plan, sfb_plan* lo, sfb_plan* hi);
/* The whole step of a linked slab as ONE update launch plus one point launch on the main
 * stream: the first d0 chunk sweeps upwards and the last one downwards, so both boundary
 * plane groups are the first planes computed and their peer stores travel while the rest of
 * the slab updates; no block spends queue-fill planes on a boundary group of its own (the
 * split protocol's boundary blocks stream 2K planes for K outputs).  The point launch
 * mirrors injected boundary nodes and gathers; the plan's two counters / events are then
 * signalled together.  Same results, bit for bit, as the split protocol and the single
 * domain.  Follow it with sfb_peer_wait / sfb_peer_wait_ipc as usual. */
SFB_API int sfb_step_slab_fused(sfb_plan* plan, int op, int64_t t);
SFB_API int sfb_peer_wait(sfb_plan* plan, sfb_plan* neighbour);
/* The same between processes (one per GPU): sfb_peer_export fills a blob of
 * SFB_PEER_BLOB_BYTES (CUDA IPC handles of the plan's wavefield buffers and of its step
 * counter) that the caller ships to the neighbouring ranks by any means;
 * sfb_link_peers_ipc maps the neighbours' blobs (NULL at an outer face).  Every boundary
 * half-step and every interior half-step then ends by writing one of the plan's two step
 * counters with a stream memory operation, and sfb_peer_wait_ipc makes the plan's streams
 * wait, on the device, until the neighbours' counters have reached its own (same two
 * conditions as sfb_peer_wait): no host-side handshake per step.  All linked
 * plans must make the same sequence of boundary half-steps, link before any of them steps,
 * and stay alive until every rank has synchronised its last step (their streams read this
 * plan's counter). */
#define SFB_PEER_BLOB_BYTES 1024
SFB_API int sfb_peer_export(sfb_plan* plan, void* blob);
SFB_API int sfb_link_peers_ipc(sfb_plan* plan, const void* lo_blob, const void* hi_blob);
SFB_API int sfb_peer_wait_ipc(sfb_plan* plan);

/* ---- TTI slab stepping.  One step of a slab is: sfb_tti_step_rot(part) (pass 1: g,
 * b g and L(p) on the owned planes; needs the ghost planes of p and r), the
 * caller's exchange of the K boundary planes of g (SFB_TTI_HALO_G_P / _G_R),
 * sfb_tti_step_update(part) (pass 2 + update + scatter/gather; call LOW before HIGH: HIGH
 * carries the point work of both boundary groups), the caller's exchange of the new p and r levels
 * (SFB_TTI_HALO_P / _R).  SURVEY.md 8e: "an extra exchange of the intermediate".
 * sfb_step_begin(SFB_OP_TTI_FORWARD) zeroes the state, sfb_step_end closes the run. */
enum { SFB_TTI_HALO_G_P = 0, SFB_TTI_HALO_G_R = 1, SFB_TTI_HALO_P = 2, SFB_TTI_HALO_R = 3 };
SFB_API int sfb_tti_step_rot(sfb_plan* plan, int64_t t, int part);
/* The TTI pair on LINKED slabs (sfb_link_peers / sfb_link_peers_ipc after sfb_set_model_tti):
 * each pass of a step is one launch over the whole slab whose edge chunks sweep towards the
 * interior and store their boundary planes -- g(p), g(r) in the first pass, the new p and r
 * in the second -- straight into the neighbours' ghost planes; the point launches mirror
 * injected boundary nodes of p and r.  One step of a plan is
 *     sfb_tti_step_rot_fused;  sfb_tti_peer_wait_g (per neighbour) / _g_ipc;
 *     sfb_tti_step_update_fused;  sfb_peer_wait (per neighbour) / sfb_peer_wait_ipc
 * with every plan making each call before any plan makes the next one when one process
 * drives several plans.  No copies, no send/recv; same bits as the single domain. */
SFB_API int sfb_tti_step_rot_fused(sfb_plan* plan, int64_t t);
SFB_API int sfb_tti_peer_wait_g(sfb_plan* plan, sfb_plan* neighbour);
SFB_API int sfb_tti_peer_wait_g_ipc(sfb_plan* plan);
SFB_API int sfb_tti_step_update_fused(sfb_plan* plan, int64_t t);
SFB_API int sfb_tti_step_update(sfb_plan* plan, int64_t t, int part);
SFB_API int sfb_tti_halo_blocks(sfb_plan* plan, int which, int64_t t, void** send_lo,
                                void** send_hi, void** recv_lo, void** recv_hi, int64_t* count);
/* A range of steps [t_from, t_to) of ONE rank's slab in a single call, with the trace tables
 * moving while the loop runs -- the slab counterpart of sfb_forward / sfb_adjoint /
 * sfb_tti_forward for a plan that is linked through CUDA IPC (or not linked at all: one
 * slab = the whole domain).  Per step: sfb_step_slab_fused + sfb_peer_wait_ipc (the TTI pair:
 * the four calls above).  `smp` (may be NULL): host f64 table [nt][np] of the sampled cloud;
 * its rows of the stepped range are filled as they are computed (fp32 over the bus, widened
 * on host threads in the shadow of the loop).  `inj` (may be NULL): host f64 table [nt][np]
 * of the injected cloud, fed to the device one chunk ahead of the step that needs it; NULL =
 * the table uploaded with sfb_upload_traces.  Backward operators run t_to - 1 down to t_from.
 * Bracket with sfb_step_begin (and a barrier between the ranks: nobody pushes into a field
 * its owner is still zeroing) and sfb_step_end.  Plans linked in-process (sfb_link_peers)
 * are stepped call by call instead: their ordering needs every plan to make each call
 * before any plan makes the next. */
SFB_API int sfb_slab_run(sfb_plan* plan, int op, int64_t t_from, int64_t t_to, const double* inj,
                         double* smp);
SFB_API int sfb_stream_sync(sfb_plan* plan);
/* test aid: keeps the plan's main (0) or boundary (1) stream busy for `microseconds`
 * (<= 1 s) at the point of the call, to shake out ordering races between linked slabs */
SFB_API int sfb_debug_stall(sfb_plan* plan, int boundary_stream, int64_t microseconds);
/* raw CUDA stream handles (cudaStream_t) the plan launches on: main, then boundary */
SFB_API int sfb_streams(sfb_plan* plan, void** main_stream, void** boundary_stream);
/* adopt caller-owned streams (e.g. the streams a collective library orders against) */
SFB_API int sfb_set_streams(sfb_plan* plan, void* main_stream, void* boundary_stream);
/* device-to-device copy of `count` floats on dst_plan's main stream (single-process
 * multi-slab runs and tests) */
SFB_API int sfb_copy_halo(sfb_plan* dst_plan, void* dst, const void* src, int64_t count);

/* ---- tile shape (the counterpart of the reference's loop-blocking autotune,
 * proj/include/sf/execute.hpp:56): threads along the contiguous axis (x4 nodes each),
 * tile rows, ring stages (0 = any; negative = the dual-stream kernel with that many
 * stages; -(100 + s) its rotated-queue, -(200 + s) its 2 x 2 patch, -(300 + s) its
 * sliding-window and -(400 + s) its tall variant with s stages), output planes per block
 * (0 = automatic).  Only compiled shapes are accepted. */
SFB_API int sfb_set_tile(sfb_plan* plan, int txv, int ty, int stages, int chunk);
SFB_API int sfb_get_tile(sfb_plan* plan, int* txv, int* ty, int* stages, int* chunk,
                         int* separable_damping);
/* times every compiled tile shape of the plan's order for `steps` launches (0 = default) on
 * the plan's own zeroed buffers and keeps the fastest: the counterpart of the reference's
 * autotune (proj/include/sf/execute.hpp:56).  Wavefield state is lost. */
SFB_API int sfb_autotune(sfb_plan* plan, int steps);
/* kernels launched by this plan since the last sfb_step_begin */
SFB_API int sfb_launch_count(sfb_plan* plan, int64_t* count);
/* on != 0: always stream the dense damp array, even when it is a sum of 1-D profiles
 * (build_damping, proj/src/model.cpp:35-56) that the kernel could rebuild on the fly.
 * Call before sfb_set_model. */
SFB_API int sfb_set_dense_damping(sfb_plan* plan, int on);

#ifdef __cplusplus
}
#endif
#endif /* SFB200_H */
