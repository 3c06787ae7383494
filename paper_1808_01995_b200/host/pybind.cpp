// pybind.cpp -- Python view of the C++ host layer (include/sfb/*.hpp) for tests and
// benchmarks.  No arithmetic here: every call forwards to the C++ classes.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include "sfb/gridio.hpp"
#include "sfb/seismic_ops.hpp"
#include "sfb/verify.hpp"

namespace py = pybind11;
using namespace sfb;

namespace {

using darray = py::array_t<double, py::array::c_style | py::array::forcecast>;

std::vector<double> flat(const darray& a) {
    return std::vector<double>(a.data(), a.data() + a.size());
}

// numpy view (no copy) of a field's interior; keeps the owner alive
py::array_t<double> interior_view(const std::shared_ptr<FieldBase>& f) {
    const std::size_t nd = f->extents().size();
    std::vector<py::ssize_t> shape(nd), strides(nd);
    std::vector<long> zero(nd, 0);
    for (std::size_t d = 0; d < nd; ++d) {
        shape[d] = f->extents()[d];
        strides[d] = f->stride(int(d)) * py::ssize_t(sizeof(double));
    }
    double* origin = f->values() + f->flat_index(zero);
    return py::array_t<double>(shape, strides, origin, py::cast(f));
}

py::array_t<double> traces_view(const std::shared_ptr<SparseFunction>& s) {
    return py::array_t<double>({py::ssize_t(s->nt()), py::ssize_t(s->npoints())},
                               {py::ssize_t(s->npoints() * sizeof(double)), py::ssize_t(sizeof(double))},
                               s->traces().data(), py::cast(s));
}

}  // namespace

PYBIND11_MODULE(_sfb_host, m) {
    m.doc() = "C++ host layer of the B200 wave propagators (mirror of sf/seismic_ops.hpp)";

    // translators run in reverse registration order: base first, members after
    auto& e_base = py::register_exception<Error>(m, "Error");
    py::register_exception<OrderError>(m, "OrderError", e_base.ptr());
    py::register_exception<LocationError>(m, "LocationError", e_base.ptr());
    py::register_exception<BindingError>(m, "BindingError", e_base.ptr());
    py::register_exception<ParameterError>(m, "ParameterError", e_base.ptr());
    py::register_exception<StabilityError>(m, "StabilityError", e_base.ptr());
    py::register_exception<CapabilityError>(m, "CapabilityError", e_base.ptr());

    py::enum_<DampProfile>(m, "DampProfile")
        .value("Linear", DampProfile::Linear)
        .value("Quadratic", DampProfile::Quadratic);
    py::enum_<Backend>(m, "Backend")
        .value("Interpreter", Backend::Interpreter)
        .value("Emitted", Backend::Emitted)
        .value("Auto", Backend::Auto);

    py::class_<Grid, std::shared_ptr<Grid>>(m, "Grid")
        .def(py::init<std::vector<long>, std::vector<double>, std::vector<double>>())
        .def_property_readonly("shape", &Grid::shape)
        .def_property_readonly("spacing", &Grid::spacing)
        .def_property_readonly("origin", &Grid::origin)
        .def("extent", &Grid::extent);

    py::class_<FieldBase, std::shared_ptr<FieldBase>>(m, "FieldBase")
        .def_property_readonly("name", &FieldBase::name)
        .def_property_readonly("space_order", &FieldBase::space_order)
        .def_property_readonly("extents", &FieldBase::extents)
        .def_property_readonly("halos", &FieldBase::halos)
        .def_property_readonly("time_buffered", &FieldBase::time_buffered)
        .def_property_readonly("time_slots", &FieldBase::time_slots)
        .def_property_readonly("storage_size", &FieldBase::storage_size)
        .def("padded_extent", &FieldBase::padded_extent)
        .def("stride", &FieldBase::stride)
        .def("at", [](const FieldBase& f, std::vector<long> c) { return f.at(c); })
        .def("set", [](FieldBase& f, std::vector<long> c, double v) { f.at(c) = v; })
        .def("array", [](std::shared_ptr<FieldBase> f) { return interior_view(f); });
    py::class_<Function, FieldBase, std::shared_ptr<Function>>(m, "Function")
        .def_static("create", &Function::create);
    py::class_<TimeFunction, FieldBase, std::shared_ptr<TimeFunction>>(m, "TimeFunction")
        .def_static("create",
                    [](std::string n, std::shared_ptr<Grid> g, int so, int to, py::object save) {
                        std::optional<long> s;
                        if (!save.is_none()) s = save.cast<long>();
                        return TimeFunction::create(std::move(n), std::move(g), so, to, s);
                    },
                    py::arg("name"), py::arg("grid"), py::arg("space_order"),
                    py::arg("time_order"), py::arg("save") = py::none());

    py::class_<SparseFunction, std::shared_ptr<SparseFunction>>(m, "SparseFunction")
        .def_static("create",
                    [](std::string n, std::shared_ptr<Grid> g, const darray& c, long nt) {
                        return SparseFunction::create(std::move(n), std::move(g), flat(c), nt);
                    })
        .def_property_readonly("npoints", &SparseFunction::npoints)
        .def_property_readonly("nt", &SparseFunction::nt)
        .def("locate", &SparseFunction::locate)
        .def_property_readonly("base_table", &SparseFunction::base_table)
        .def_property_readonly("weight_table", &SparseFunction::weight_table)
        .def_property_readonly("traces", [](std::shared_ptr<SparseFunction> s) { return traces_view(s); });

    m.def("build_damping", &build_damping, py::arg("grid"), py::arg("nbl"), py::arg("v_max"),
          py::arg("profile") = DampProfile::Quadratic, py::arg("space_order") = 2);

    py::class_<SeismicModel>(m, "SeismicModel")
        .def(py::init([](std::vector<long> shape, std::vector<double> spacing,
                         std::vector<double> origin, const darray& vel, long nbl, int order,
                         DampProfile prof) {
                 return new SeismicModel(std::move(shape), std::move(spacing), std::move(origin),
                                         flat(vel), nbl, order, prof);
             }),
             py::arg("shape"), py::arg("spacing"), py::arg("origin"), py::arg("velocity"),
             py::arg("nbl"), py::arg("space_order") = 8,
             py::arg("profile") = DampProfile::Quadratic)
        .def_property_readonly("grid", &SeismicModel::grid)
        .def_property_readonly("m", [](const SeismicModel& s) { return std::static_pointer_cast<FieldBase>(s.m()); })
        .def_property_readonly("damp", [](const SeismicModel& s) { return std::static_pointer_cast<FieldBase>(s.damp()); })
        .def_property_readonly("nbl", &SeismicModel::nbl)
        .def_property_readonly("space_order", &SeismicModel::space_order)
        .def_property_readonly("physical_shape", &SeismicModel::physical_shape)
        .def_property_readonly("v_min", &SeismicModel::v_min)
        .def_property_readonly("v_max", &SeismicModel::v_max)
        .def("critical_dt",
             [](const SeismicModel& s, py::object order, double gamma) {
                 return order.is_none() ? gamma * s.critical_dt()
                                        : s.critical_dt(order.cast<int>(), gamma);
             },
             py::arg("space_order") = py::none(), py::arg("gamma") = 1.0)
        .def("set_velocity", [](SeismicModel& s, const darray& v) { s.set_velocity(flat(v)); })
        .def("physical_m", [](const SeismicModel& s) { return py::array(py::cast(s.physical_m())); })
        .def("set_physical_m", [](SeismicModel& s, const darray& v) { s.set_physical_m(flat(v)); });

    m.def("ricker", [](double f0, double t0, double dt, long nt) { return py::array(py::cast(ricker(f0, t0, dt, nt))); });
    m.def("ricker_value", &ricker_value);
    m.def("dgauss4_value", &dgauss4_value);

    py::class_<AcquisitionGeometry>(m, "AcquisitionGeometry")
        .def(py::init([](const SeismicModel& model, const darray& src, const darray& rec, double t0,
                         double tn, double dt, double f0) {
                 return new AcquisitionGeometry(model, flat(src), flat(rec), t0, tn, dt, f0);
             }),
             py::keep_alive<1, 2>())
        .def_property_readonly("src", &AcquisitionGeometry::src)
        .def_property_readonly("rec", &AcquisitionGeometry::rec)
        .def_property_readonly("t0", &AcquisitionGeometry::t0)
        .def_property_readonly("tn", &AcquisitionGeometry::tn)
        .def_property_readonly("dt", &AcquisitionGeometry::dt)
        .def_property_readonly("f0", &AcquisitionGeometry::f0)
        .def_property_readonly("nt", &AcquisitionGeometry::nt)
        .def_property_readonly("n_src", &AcquisitionGeometry::n_src)
        .def_property_readonly("n_rec", &AcquisitionGeometry::n_rec);

    py::class_<ExecutionReport>(m, "ExecutionReport")
        .def_readonly("seconds", &ExecutionReport::seconds)
        .def_readonly("flops", &ExecutionReport::flops)
        .def_readonly("gflops", &ExecutionReport::gflops)
        .def_readonly("steps", &ExecutionReport::steps)
        .def_readonly("gpts_per_s", &ExecutionReport::gpts_per_s)
        .def_readonly("kernel_launches", &ExecutionReport::kernel_launches);

    py::class_<WaveOp>(m, "WaveOp")
        .def_property_readonly("wavefield", [](const WaveOp& w) { return w.wavefield; })
        .def_property_readonly("wavefield_r", [](const WaveOp& w) { return w.wavefield_r; })
        .def_property_readonly("inj", [](const WaveOp& w) { return w.inj; })
        .def_property_readonly("smp", [](const WaveOp& w) { return w.smp; })
        .def_readonly("dt", &WaveOp::dt)
        .def_readonly("nt", &WaveOp::nt)
        .def_readwrite("save_every", &WaveOp::save_every)
        .def_readwrite("host_history", &WaveOp::host_history)
        .def_readwrite("checkpoint_every", &WaveOp::checkpoint_every);
    py::class_<TtiModel>(m, "TtiModel")
        .def(py::init([](const SeismicModel& model, const darray& e, const darray& d, const darray& t,
                         const darray& p) { return new TtiModel(model, flat(e), flat(d), flat(t), flat(p)); }))
        .def_property_readonly("epsilon", [](const TtiModel& t) { return std::static_pointer_cast<FieldBase>(t.epsilon); })
        .def_property_readonly("delta", [](const TtiModel& t) { return std::static_pointer_cast<FieldBase>(t.delta); })
        .def_property_readonly("theta", [](const TtiModel& t) { return std::static_pointer_cast<FieldBase>(t.theta); })
        .def_property_readonly("phi", [](const TtiModel& t) { return std::static_pointer_cast<FieldBase>(t.phi); })
        .def("epsilon_max", &TtiModel::epsilon_max);
    m.def("tti_critical_dt", &tti_critical_dt);
    m.def("tti_forward_operator", &tti_forward_operator);

    py::class_<GradientOp>(m, "GradientOp")
        .def_property_readonly("v", [](const GradientOp& g) { return g.v; })
        .def_property_readonly("grad", [](const GradientOp& g) { return std::static_pointer_cast<FieldBase>(g.grad); })
        .def_property_readonly("resid", [](const GradientOp& g) { return g.resid; })
        .def_readonly("dt", &GradientOp::dt)
        .def_readonly("nt", &GradientOp::nt);

    m.def("forward_operator", &forward_operator, py::arg("model"), py::arg("geom"),
          py::arg("space_order"), py::arg("save") = false, py::arg("tiles") = std::vector<long>{});
    m.def("adjoint_operator", &adjoint_operator);
    m.def("gradient_operator", &gradient_operator);
    m.def("run_wave_slabs",
          py::overload_cast<WaveOp&, const SeismicModel&, const AcquisitionGeometry&,
                            const std::vector<int>&>(&run_wave_slabs),
          py::arg("op"), py::arg("model"), py::arg("geom"), py::arg("devices"),
          py::call_guard<py::gil_scoped_release>());
    m.def("run_wave_slabs_tti",
          py::overload_cast<WaveOp&, const SeismicModel&, const TtiModel&,
                            const AcquisitionGeometry&, const std::vector<int>&>(&run_wave_slabs),
          py::arg("op"), py::arg("model"), py::arg("tti"), py::arg("geom"), py::arg("devices"),
          py::call_guard<py::gil_scoped_release>());
    m.def("run_wave", &run_wave, py::arg("op"), py::arg("backend") = Backend::Auto,
          py::arg("nthreads") = 1, py::call_guard<py::gil_scoped_release>());
    m.def("run_gradient", &run_gradient, py::arg("op"), py::arg("backend") = Backend::Auto,
          py::arg("nthreads") = 1, py::call_guard<py::gil_scoped_release>());
    m.def("objective", [](const SparseFunction& s, const darray& obs) { return objective(s, flat(obs)); });

    py::class_<GradientResult>(m, "GradientResult")
        .def_readonly("objective", &GradientResult::objective)
        .def_property_readonly("gradient", [](const GradientResult& r) { return py::array(py::cast(r.gradient)); })
        .def_property_readonly("residual", [](const GradientResult& r) { return py::array(py::cast(r.residual)); });
    m.def("fwi_gradient",
          [](const SeismicModel& model, AcquisitionGeometry& geom, const darray& obs, int order,
             long save_every, long checkpoint_every) {
              return fwi_gradient(model, geom, flat(obs), order, Backend::Auto, save_every,
                                  checkpoint_every);
          },
          py::arg("model"), py::arg("geom"), py::arg("observed"), py::arg("space_order"),
          py::arg("save_every") = 1, py::arg("checkpoint_every") = 0);

    py::class_<FwiConfig>(m, "FwiConfig")
        .def(py::init<>())
        .def_readwrite("space_order", &FwiConfig::space_order)
        .def_readwrite("n_iter", &FwiConfig::n_iter)
        .def_readwrite("step_scale", &FwiConfig::step_scale)
        .def_readwrite("m_min", &FwiConfig::m_min)
        .def_readwrite("m_max", &FwiConfig::m_max)
        .def_readwrite("nthreads", &FwiConfig::nthreads)
        .def_readwrite("devices", &FwiConfig::devices)
        .def_readwrite("save_every", &FwiConfig::save_every)
        .def_readwrite("checkpoint_every", &FwiConfig::checkpoint_every);
    py::class_<FwiResult>(m, "FwiResult")
        .def_readonly("objectives", &FwiResult::objectives)
        .def_readonly("model_rms", &FwiResult::model_rms)
        .def_property_readonly("final_m", [](const FwiResult& r) { return py::array(py::cast(r.final_m)); });
    m.def("fwi",
          [](SeismicModel& model, py::list shots, std::vector<darray> observed, const FwiConfig& cfg,
             py::object true_m) {
              // shots are AcquisitionGeometry objects owned by Python; fwi works on copies of
              // the handles (the clouds are shared), like a std::vector the caller owns
              std::vector<AcquisitionGeometry> sv;
              for (auto h : shots) sv.push_back(h.cast<AcquisitionGeometry&>());
              std::vector<std::vector<double>> ov;
              for (auto& o : observed) ov.push_back(flat(o));
              std::vector<double> tm;
              if (!true_m.is_none()) tm = flat(true_m.cast<darray>());
              return fwi(model, sv, ov, cfg, true_m.is_none() ? nullptr : &tm);
          },
          py::arg("model"), py::arg("shots"), py::arg("observed"), py::arg("cfg"),
          py::arg("true_m") = py::none());

    m.def("set_device", &set_device);

    // verification recipes (proj/include/sf/verify.hpp, proj/include/sf/slopefit.hpp)
    py::class_<SlopeFit>(m, "SlopeFit")
        .def_readonly("slope", &SlopeFit::slope)
        .def_readonly("intercept", &SlopeFit::intercept)
        .def_readonly("residual", &SlopeFit::residual);
    m.def("fit_loglog", &fit_loglog);
    py::class_<AdjointConfig>(m, "AdjointConfig")
        .def(py::init<>())
        .def_readwrite("ndim", &AdjointConfig::ndim)
        .def_readwrite("n", &AdjointConfig::n)
        .def_readwrite("space_order", &AdjointConfig::space_order)
        .def_readwrite("h", &AdjointConfig::h)
        .def_readwrite("nbl", &AdjointConfig::nbl)
        .def_readwrite("tn", &AdjointConfig::tn)
        .def_readwrite("f0", &AdjointConfig::f0);
    py::class_<AdjointReport>(m, "AdjointReport")
        .def_readonly("forward_dot", &AdjointReport::forward_dot)
        .def_readonly("adjoint_dot", &AdjointReport::adjoint_dot)
        .def_readonly("rel_err", &AdjointReport::rel_err);
    m.def("adjoint_test", &adjoint_test, py::call_guard<py::gil_scoped_release>());
    py::class_<GradientConfig>(m, "GradientConfig")
        .def(py::init<>())
        .def_readwrite("nx", &GradientConfig::nx)
        .def_readwrite("nz", &GradientConfig::nz)
        .def_readwrite("h", &GradientConfig::h)
        .def_readwrite("space_order", &GradientConfig::space_order)
        .def_readwrite("nbl", &GradientConfig::nbl)
        .def_readwrite("tn", &GradientConfig::tn)
        .def_readwrite("f0", &GradientConfig::f0)
        .def_readwrite("steps", &GradientConfig::steps);
    py::class_<GradientReport>(m, "GradientReport")
        .def_readonly("phi0", &GradientReport::phi0)
        .def_readonly("dphi", &GradientReport::dphi)
        .def_readonly("steps", &GradientReport::steps)
        .def_readonly("eps0", &GradientReport::eps0)
        .def_readonly("eps1", &GradientReport::eps1)
        .def_readonly("eps1_fitted", &GradientReport::eps1_fitted)
        .def_readonly("fit0", &GradientReport::fit0)
        .def_readonly("fit1", &GradientReport::fit1)
        .def_readonly("fit1_valid", &GradientReport::fit1_valid);
    m.def("gradient_test", &gradient_test, py::call_guard<py::gil_scoped_release>());
    py::class_<BenchConfig>(m, "BenchConfig")
        .def(py::init<>())
        .def_readwrite("orders", &BenchConfig::orders)
        .def_readwrite("n", &BenchConfig::n)
        .def_readwrite("steps", &BenchConfig::steps)
        .def_readwrite("wall_order", &BenchConfig::wall_order)
        .def_readwrite("repeats", &BenchConfig::repeats);
    py::class_<BenchReport>(m, "BenchReport")
        .def_readonly("orders", &BenchReport::orders)
        .def_readonly("oi", &BenchReport::oi)
        .def_readonly("flops", &BenchReport::flops)
        .def_readonly("wall_small", &BenchReport::wall_small)
        .def_readonly("wall_big", &BenchReport::wall_big)
        .def_readonly("wall_ratio", &BenchReport::wall_ratio);
    m.def("bench", &bench, py::call_guard<py::gil_scoped_release>());

    // wire formats (proj/include/sf/gridio.hpp, proj/include/sf/sparse.hpp:97-104)
    m.def("write_grid", [](const std::string& path, std::vector<long> shape, const darray& data) {
        write_grid(path, shape, flat(data));
    });
    m.def("read_grid", [](const std::string& path) {
        GridData g = read_grid(path);
        py::array_t<double> a(std::vector<py::ssize_t>(g.shape.begin(), g.shape.end()));
        std::copy(g.data.begin(), g.data.end(), a.mutable_data());
        return a;
    });
    m.def("write_traces_table", [](const std::string& path, const darray& tr, double t0, double dt) {
        write_traces_csv(path, long(tr.shape(0)), long(tr.shape(1)), flat(tr), t0, dt);
    });
    m.def("write_traces_csv", [](const std::string& path, const SparseFunction& s,
                                 std::vector<double> times) { write_traces_csv(path, s, times); });
    m.def("read_traces_csv", [](const std::string& path, SparseFunction& s) {
        std::vector<double> times;
        read_traces_csv(path, s, &times);
        return times;
    });
    m.def("write_coords_csv", &write_coords_csv);
    m.def("read_coords_csv", &read_coords_csv);
}
