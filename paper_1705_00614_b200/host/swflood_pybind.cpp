// swflood_pybind.cpp — pybind11 bindings of the C++ drop-in API
// (include/swflood_b200.hpp), the `bindings/` module the reference's build
// expects (CMakeLists.txt:18-28) but never shipped.  Names, fields and
// defaults follow the reference headers (grid.hpp, sources.hpp, stepper.hpp);
// the flow arrays are exposed as numpy views onto the C++ vectors, so a
// step reads and writes them in place without copies.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include "swflood_b200.hpp"

namespace py = pybind11;
using namespace swflood;

namespace {

// numpy view of a std::vector<double> member, kept alive by its owner
template <class T>
py::array_t<double> view(T& owner, std::vector<double>& v, py::handle base) {
  (void)owner;
  return py::array_t<double>({(py::ssize_t)v.size()}, {(py::ssize_t)sizeof(double)}, v.data(),
                             base);
}

void assign(std::vector<double>& v, py::array_t<double, py::array::c_style | py::array::forcecast> a) {
  auto r = a.unchecked<1>();
  v.resize((size_t)r.shape(0));
  for (py::ssize_t k = 0; k < r.shape(0); ++k) v[(size_t)k] = r(k);
}

}  // namespace

PYBIND11_MODULE(swflood_native, m) {
  m.doc() = "B200 CSPH-TVD step (arXiv 1705.00614) behind the swflood C++ API";

  py::register_exception<ConfigError>(m, "ConfigError", PyExc_ValueError);
  py::register_exception<NumericalError>(m, "NumericalError", PyExc_ArithmeticError);
  // std::out_of_range -> IndexError (pybind11's default translation)

  py::class_<Vec2>(m, "Vec2")
      .def(py::init<>())
      .def(py::init([](double x, double y) { return Vec2{x, y}; }))
      .def_readwrite("x", &Vec2::x)
      .def_readwrite("y", &Vec2::y);

  // ---- grid.hpp ------------------------------------------------------------
  py::class_<Terrain>(m, "Terrain")
      .def(py::init<>())
      .def(py::init([](int nx, int ny, double h, double x0, double y0,
                       py::array_t<double, py::array::c_style | py::array::forcecast> b) {
             Terrain t;
             t.nx = nx;
             t.ny = ny;
             t.h = h;
             t.x0 = x0;
             t.y0 = y0;
             assign(t.b, b);
             return t;
           }),
           py::arg("nx"), py::arg("ny"), py::arg("h"), py::arg("x0"), py::arg("y0"), py::arg("b"))
      .def_readwrite("nx", &Terrain::nx)
      .def_readwrite("ny", &Terrain::ny)
      .def_readwrite("h", &Terrain::h)
      .def_readwrite("x0", &Terrain::x0)
      .def_readwrite("y0", &Terrain::y0)
      .def_property(
          "b", [](py::object self) { Terrain& t = self.cast<Terrain&>(); return view(t, t.b, self); },
          [](Terrain& t, py::array_t<double, py::array::c_style | py::array::forcecast> a) { assign(t.b, a); })
      .def("cells", &Terrain::cells)
      .def("idx", &Terrain::idx)
      .def("contains", &Terrain::contains)
      .def("cell_area", &Terrain::cell_area)
      .def("xc", &Terrain::xc)
      .def("yc", &Terrain::yc);

  py::class_<FlowState>(m, "FlowState")
      .def(py::init<>())
      .def_static("dry", &FlowState::dry, py::arg("terrain"))
      .def_readwrite("nx", &FlowState::nx)
      .def_readwrite("ny", &FlowState::ny)
      .def_readwrite("t", &FlowState::t)
      .def_property(
          "H", [](py::object self) { FlowState& s = self.cast<FlowState&>(); return view(s, s.H, self); },
          [](FlowState& s, py::array_t<double, py::array::c_style | py::array::forcecast> a) { assign(s.H, a); })
      .def_property(
          "HUx", [](py::object self) { FlowState& s = self.cast<FlowState&>(); return view(s, s.HUx, self); },
          [](FlowState& s, py::array_t<double, py::array::c_style | py::array::forcecast> a) { assign(s.HUx, a); })
      .def_property(
          "HUy", [](py::object self) { FlowState& s = self.cast<FlowState&>(); return view(s, s.HUy, self); },
          [](FlowState& s, py::array_t<double, py::array::c_style | py::array::forcecast> a) { assign(s.HUy, a); })
      .def("cells", &FlowState::cells)
      .def("idx", &FlowState::idx)
      .def("enforce_dry_rule", &FlowState::enforce_dry_rule);

  py::class_<PhysicalParams>(m, "PhysicalParams")
      .def(py::init<>())
      .def_readwrite("g", &PhysicalParams::g)
      .def_readwrite("n_manning", &PhysicalParams::n_manning)
      .def_property(
          "n_field",
          [](py::object self) { PhysicalParams& p = self.cast<PhysicalParams&>(); return view(p, p.n_field, self); },
          [](PhysicalParams& p, py::array_t<double, py::array::c_style | py::array::forcecast> a) { assign(p.n_field, a); })
      .def_readwrite("nu", &PhysicalParams::nu)
      .def_readwrite("omega_z", &PhysicalParams::omega_z)
      .def_readwrite("c_a", &PhysicalParams::c_a)
      .def_readwrite("rho_air", &PhysicalParams::rho_air)
      .def_readwrite("rho_water", &PhysicalParams::rho_water)
      .def_readwrite("eps_dry", &PhysicalParams::eps_dry)
      .def("manning", &PhysicalParams::manning);

  py::class_<WindSample>(m, "WindSample")
      .def(py::init<>())
      .def(py::init([](double t, double wx, double wy) { return WindSample{t, wx, wy}; }))
      .def_readwrite("t", &WindSample::t)
      .def_readwrite("wx", &WindSample::wx)
      .def_readwrite("wy", &WindSample::wy);
  py::class_<WindForcing>(m, "WindForcing")
      .def(py::init<>())
      .def(py::init([](std::vector<WindSample> s) { WindForcing w; w.series = std::move(s); return w; }))
      .def_readwrite("series", &WindForcing::series)
      .def("any", &WindForcing::any);

  // ---- sources.hpp ---------------------------------------------------------
  py::class_<CellRect>(m, "CellRect")
      .def(py::init<>())
      .def(py::init([](int i0, int j0, int i1, int j1) { return CellRect{i0, j0, i1, j1}; }))
      .def_readwrite("i0", &CellRect::i0)
      .def_readwrite("j0", &CellRect::j0)
      .def_readwrite("i1", &CellRect::i1)
      .def_readwrite("j1", &CellRect::j1)
      .def("count", &CellRect::count);
  py::class_<HydrographSample>(m, "HydrographSample")
      .def(py::init<>())
      .def(py::init([](double t, double q) { return HydrographSample{t, q}; }))
      .def_readwrite("t", &HydrographSample::t)
      .def_readwrite("q", &HydrographSample::q);
  py::class_<SourceSpec> src(m, "SourceSpec");
  py::enum_<SourceSpec::Kind>(src, "Kind")
      .value("Discharge", SourceSpec::Kind::Discharge)
      .value("Rain", SourceSpec::Kind::Rain);
  src.def(py::init<>())
      .def_readwrite("kind", &SourceSpec::kind)
      .def_readwrite("name", &SourceSpec::name)
      .def_readwrite("cells", &SourceSpec::cells)
      .def_readwrite("hydrograph", &SourceSpec::hydrograph)
      .def_readwrite("rate", &SourceSpec::rate)
      .def_readwrite("source_velocity", &SourceSpec::source_velocity)
      .def("discharge_at", &SourceSpec::discharge_at)
      .def("validate", &SourceSpec::validate);

  // ---- stepper.hpp ---------------------------------------------------------
  py::class_<TimestepControl>(m, "TimestepControl")
      .def(py::init<>())
      .def(py::init([](double courant, double dt_max, double dt_min) {
             TimestepControl k;
             k.courant = courant;
             k.dt_max = dt_max;
             k.dt_min = dt_min;
             return k;
           }),
           py::arg("courant") = 0.5, py::arg("dt_max") = 10.0, py::arg("dt_min") = 1e-9)
      .def_readwrite("courant", &TimestepControl::courant)
      .def_readwrite("dt_max", &TimestepControl::dt_max)
      .def_readwrite("dt_min", &TimestepControl::dt_min)
      .def("validate", &TimestepControl::validate);
  py::enum_<EdgeKind>(m, "EdgeKind").value("Reflective", EdgeKind::Reflective).value("Open", EdgeKind::Open);
  py::class_<BoundaryConfig>(m, "BoundaryConfig")
      .def(py::init<>())
      .def_readwrite("west", &BoundaryConfig::west)
      .def_readwrite("east", &BoundaryConfig::east)
      .def_readwrite("south", &BoundaryConfig::south)
      .def_readwrite("north", &BoundaryConfig::north)
      .def_static("all", &BoundaryConfig::all);
  py::class_<StepperOptions>(m, "StepperOptions")
      .def(py::init<>())
      .def_readwrite("block_size", &StepperOptions::block_size)
      .def_readwrite("skip_dry_blocks", &StepperOptions::skip_dry_blocks)
      .def_readwrite("workers", &StepperOptions::workers)
      .def_readwrite("boundaries", &StepperOptions::boundaries)
      .def_readwrite("devices", &StepperOptions::devices);
  py::class_<StageTimings>(m, "StageTimings")
      .def_readonly("mask", &StageTimings::mask)
      .def_readonly("forces", &StageTimings::forces)
      .def_readonly("dt", &StageTimings::dt)
      .def_readonly("predictor", &StageTimings::predictor)
      .def_readonly("mid_forces", &StageTimings::mid_forces)
      .def_readonly("corrector", &StageTimings::corrector)
      .def_readonly("flux", &StageTimings::flux)
      .def_readonly("finalize", &StageTimings::finalize)
      .def("total", &StageTimings::total);
  py::class_<StepInfo>(m, "StepInfo")
      .def_readonly("tau", &StepInfo::tau)
      .def_readonly("active_fraction", &StepInfo::active_fraction)
      .def_readonly("lagrangian_blocks", &StepInfo::lagrangian_blocks)
      .def_readonly("flux_blocks", &StepInfo::flux_blocks)
      .def_readonly("total_blocks", &StepInfo::total_blocks)
      .def_readonly("timings", &StepInfo::timings)
      .def_readonly("clamp_deficit_volume", &StepInfo::clamp_deficit_volume)
      .def_readonly("source_volume", &StepInfo::source_volume)
      .def_readonly("boundary_outflow_volume", &StepInfo::boundary_outflow_volume);

  // the terrain is held by pointer and must outlive the stepper
  // (stepper.cpp:129): keep_alive ties its lifetime to the stepper's
  py::class_<CsphTvdStepper>(m, "CsphTvdStepper")
      .def(py::init<const Terrain&, PhysicalParams, TimestepControl, StepperOptions>(),
           py::arg("terrain"), py::arg("params"), py::arg("control"),
           py::arg("options") = StepperOptions{}, py::keep_alive<1, 2>())
      .def("set_wind", &CsphTvdStepper::set_wind)
      .def("set_sources", &CsphTvdStepper::set_sources)
      .def("step", &CsphTvdStepper::step, py::arg("state"), py::arg("dt_cap") = 0.0,
           py::call_guard<py::gil_scoped_release>())
      .def("begin_step", &CsphTvdStepper::begin_step)
      .def("compute_forces", &CsphTvdStepper::compute_forces)
      .def("compute_dt", &CsphTvdStepper::compute_dt, py::arg("state"), py::arg("dt_cap") = 0.0)
      .def("predictor", &CsphTvdStepper::predictor)
      .def("mid_forces", &CsphTvdStepper::mid_forces)
      .def("corrector", &CsphTvdStepper::corrector)
      .def("flux", &CsphTvdStepper::flux)
      .def("final_update", &CsphTvdStepper::final_update)
      .def("terrain", &CsphTvdStepper::terrain, py::return_value_policy::reference_internal)
      .def("params", &CsphTvdStepper::params, py::return_value_policy::reference_internal)
      .def("control", &CsphTvdStepper::control, py::return_value_policy::reference_internal)
      .def("options", &CsphTvdStepper::options, py::return_value_policy::reference_internal)
      .def("last_clamp_deficit", &CsphTvdStepper::last_clamp_deficit)
      .def("last_source_volume", &CsphTvdStepper::last_source_volume)
      .def("last_boundary_outflow", &CsphTvdStepper::last_boundary_outflow);
}
