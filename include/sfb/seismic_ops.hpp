// seismic_ops.hpp -- the operator entry points of the wave-propagator path, GPU build.
//
// Same names, argument meaning and error behaviour as the reference's
// proj/include/sf/seismic_ops.hpp:13-97; each function cites the lines it replaces.  The
// engine behind them is libsfb200.so (include/sfb200.h): hand-written sm_100a kernels,
// no backend dispatch and no CPU fallback -- Backend / nthreads / tiles are accepted for
// source compatibility and ignored.
#pragma once

#include <memory>
#include <vector>

#include "sfb/geometry.hpp"
#include "sfb/model.hpp"

namespace sfb {

enum class Backend { Interpreter, Emitted, Auto };  // proj/include/sf/execute.hpp:22 (ignored)

// proj/include/sf/execute.hpp:40-46
struct ExecutionReport {
    double seconds = 0.0;  // stepping loop only, device time
    long long flops = 0;
    double gflops = 0.0;
    long steps = 0;
    std::vector<long> tiles;
    double gpts_per_s = 0.0;
    long kernel_launches = 0;
};

class Engine;  // owns one sfb_plan

// proj/include/sf/seismic_ops.hpp:17-23.  `inj` traces are caller input, `smp` traces are
// produced by the run; rows 0, 1 and nt-1 of the sampled traces are structural zeros.
struct WaveOp {
    std::shared_ptr<Engine> engine;
    std::shared_ptr<TimeFunction> wavefield;
    std::shared_ptr<SparseFunction> inj, smp;
    double dt = 0;
    long nt = 0;
    int space_order = 0;
    bool adjoint = false;
    // save=true keeps the forward history in HBM (every save_every-th level; 1 = the
    // reference's full history).  host_history additionally mirrors every saved level
    // into `wavefield` as the reference does (proj/src/seismic_ops.cpp:66-68).
    long save_every = 0;
    bool host_history = true;
    // with save: keep only the state at every checkpoint_every-th level (>= 2) and let the
    // gradient sweep recompute the levels in between (imaging at every level, the
    // reference's condition, without nt levels of memory).  No host mirror in this mode.
    long checkpoint_every = 0;
    // TTI operator only: the auxiliary field r of the coupled pair (wavefield holds p)
    bool tti = false;
    std::shared_ptr<TimeFunction> wavefield_r;
};

// proj/include/sf/seismic_ops.hpp:28-30, proj/src/seismic_ops.cpp:58-82
WaveOp forward_operator(const SeismicModel& model, const AcquisitionGeometry& geom,
                        int space_order, bool save = false, std::vector<long> tiles = {});
// proj/include/sf/seismic_ops.hpp:35-36, proj/src/seismic_ops.cpp:84-107
WaveOp adjoint_operator(const SeismicModel& model, const AcquisitionGeometry& geom,
                        int space_order);

// ---- TTI (no reference counterpart) ----------------
// Thomsen parameters and the tilt / azimuth of the symmetry axis on the model's padded
// grid.  The pseudo-acoustic system needs epsilon >= delta > -1/2 everywhere.
struct TtiModel {
    std::shared_ptr<Function> epsilon, delta, theta, phi;
    // fields over the physical shape, edge-extended into the absorbing layer like the
    // velocity (proj/src/model.cpp:92-100)
    TtiModel(const SeismicModel& model, const std::vector<double>& epsilon,
             const std::vector<double>& delta, const std::vector<double>& theta,
             const std::vector<double>& phi);
    double epsilon_max() const;
};

// largest stable dt of the TTI operator: the acoustic rule (proj/src/model.cpp:103-111)
// with v_max sqrt(1 + 2 eps_max), times 0.9 for the twice-applied first derivatives
double tti_critical_dt(const SeismicModel& model, const TtiModel& tti, int space_order);

// coupled (p, r) forward operator; sources are injected into both fields, receivers
// sample p.  StabilityError when dt exceeds tti_critical_dt or epsilon < delta somewhere.
WaveOp tti_forward_operator(const SeismicModel& model, const TtiModel& tti,
                            const AcquisitionGeometry& geom, int space_order);

// proj/include/sf/seismic_ops.hpp:40-47
struct GradientOp {
    std::shared_ptr<Engine> engine;
    std::shared_ptr<TimeFunction> v;
    std::shared_ptr<Function> grad;
    std::shared_ptr<SparseFunction> resid;
    double dt = 0;
    long nt = 0;
    int space_order = 0;
};

// proj/include/sf/seismic_ops.hpp:49-51, proj/src/seismic_ops.cpp:109-135.  saved_u must
// be the saved (non-buffered, nt-slot) wavefield of a forward operator that has run.
GradientOp gradient_operator(const SeismicModel& model, const AcquisitionGeometry& geom,
                             int space_order, std::shared_ptr<TimeFunction> saved_u);

// proj/include/sf/seismic_ops.hpp:55-58, proj/src/seismic_ops.cpp:137-147
ExecutionReport run_wave(WaveOp& w, Backend backend = Backend::Auto, int nthreads = 1);
ExecutionReport run_gradient(GradientOp& g, Backend backend = Backend::Auto,
                             int nthreads = 1);

// extension: run a forward or adjoint operator on a slab decomposition of the
// grid along axis 0 driven by this one process -- one slab per entry of `devices` (CUDA
// ordinals; an ordinal may repeat).  The slabs are linked with sfb_link_peers: each boundary
// half-step stores its planes straight into the neighbours' ghost planes (peer stores over
// NVLink) while the interior updates, and events order the slabs; there is no copy and no
// collective.  Fills w.smp's traces and the two live levels of w.wavefield exactly as
// run_wave does (the result is bit-identical to the single-device run).
ExecutionReport run_wave_slabs(WaveOp& w, const SeismicModel& model,
                               const AcquisitionGeometry& geom, const std::vector<int>& devices);
// the TTI pair on slabs: two neighbour exchanges per step (g between the passes, the new p
// and r levels after the update), both fused into the passes as peer stores between the
// linked plans (sfb_tti_step_rot_fused / sfb_tti_step_update_fused)
ExecutionReport run_wave_slabs(WaveOp& w, const SeismicModel& model, const TtiModel& tti,
                               const AcquisitionGeometry& geom, const std::vector<int>& devices);

// proj/include/sf/seismic_ops.hpp:61, proj/src/seismic_ops.cpp:149-160
double objective(const SparseFunction& pred, const std::vector<double>& observed);

// proj/include/sf/seismic_ops.hpp:63-73
struct GradientResult {
    double objective = 0;
    std::vector<double> gradient;  // per physical-domain cell, row-major
    std::vector<double> residual;
};

// proj/src/seismic_ops.cpp:197-216.  save_every is an extension (1 = reference): image
// against every save_every-th forward level only, which divides the HBM the history needs;
// checkpoint_every >= 2 instead keeps the exact imaging condition and recomputes the history
// segment by segment from sparse checkpoints (one extra forward pass).
GradientResult fwi_gradient(const SeismicModel& model, AcquisitionGeometry& geom,
                            const std::vector<double>& observed, int space_order,
                            Backend backend = Backend::Auto, long save_every = 1,
                            long checkpoint_every = 0);

// proj/include/sf/seismic_ops.hpp:75-97, proj/src/seismic_ops.cpp:218-286
struct FwiConfig {
    int space_order = 8;
    long n_iter = 15;
    double step_scale = 0.05;
    double m_min = 0, m_max = 0;
    Backend backend = Backend::Auto;
    int nthreads = 1;  // shots in flight at once (one engine each)
    // extension: CUDA ordinals the shots are dealt to round-robin (empty = the calling
    // thread's device).  Shot gradients are still reduced in shot order on the host, so the
    // result does not depend on the device list.
    std::vector<int> devices;
    // extension: memory strategy of every shot gradient (see fwi_gradient)
    long save_every = 1, checkpoint_every = 0;
};

struct FwiResult {
    std::vector<double> objectives;
    std::vector<double> model_rms;
    std::vector<double> final_m;
};

FwiResult fwi(SeismicModel& model, std::vector<AcquisitionGeometry>& shots,
              const std::vector<std::vector<double>>& observed, const FwiConfig& cfg,
              const std::vector<double>* true_m = nullptr);

// CUDA device the operators created by this thread run on (default 0)
void set_device(int ordinal);
int device();

}  // namespace sfb
