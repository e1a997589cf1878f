// swflood_io.cpp — scenario I/O (include/swflood/io.hpp).
#include "swflood/io.hpp"

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <random>
#include <sstream>

namespace swflood::io {

namespace {

std::string lower(std::string s) {
  for (char& c : s) c = (char)std::tolower((unsigned char)c);
  return s;
}

std::string trim(const std::string& s) {
  size_t a = s.find_first_not_of(" \t\r\n"), b = s.find_last_not_of(" \t\r\n");
  return a == std::string::npos ? "" : s.substr(a, b - a + 1);
}

[[noreturn]] void fail(const std::string& path, int line, const std::string& what) {
  throw ConfigError(path + ":" + std::to_string(line) + ": " + what);
}

double to_num(const std::string& path, int line, const std::string& tok) {
  char* end = nullptr;
  double v = std::strtod(tok.c_str(), &end);
  if (tok.empty() || end != tok.c_str() + tok.size()) fail(path, line, "not a number: '" + tok + "'");
  return v;
}

struct Raster {
  int nx = 0, ny = 0;
  double x0 = 0, y0 = 0, h = 0, nodata = -9999.0;
  bool has_nodata = false;
  std::vector<double> v;  // row-major, j northward
  std::vector<unsigned char> is_nodata;
};

Raster read_esri(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ConfigError("cannot open raster '" + path + "'");
  Raster R;
  std::map<std::string, double> hdr;
  std::string line;
  int ln = 0;
  std::streampos data_pos = 0;
  bool center_x = false, center_y = false;
  // header: keyword value lines until the first numeric line
  while (true) {
    data_pos = in.tellg();
    if (!std::getline(in, line)) fail(path, ln + 1, "missing data rows");
    ++ln;
    std::string t = trim(line);
    if (t.empty()) continue;
    if (std::isdigit((unsigned char)t[0]) || t[0] == '-' || t[0] == '+' || t[0] == '.') {
      --ln;
      in.seekg(data_pos);
      break;
    }
    std::istringstream ss(t);
    std::string key, val, extra;
    ss >> key >> val;
    if (val.empty() || (ss >> extra)) fail(path, ln, "malformed header line '" + t + "'");
    key = lower(key);
    if (key == "xllcenter") center_x = true, key = "xllcorner";
    if (key == "yllcenter") center_y = true, key = "yllcorner";
    static const char* known[] = {"ncols", "nrows", "xllcorner", "yllcorner", "cellsize",
                                  "nodata_value"};
    if (std::find_if(std::begin(known), std::end(known), [&](const char* k) { return key == k; }) ==
        std::end(known))
      fail(path, ln, "unknown header keyword '" + key + "'");
    hdr[key] = to_num(path, ln, val);
  }
  for (const char* k : {"ncols", "nrows", "xllcorner", "yllcorner", "cellsize"})
    if (!hdr.count(k)) fail(path, ln, std::string("malformed header: missing ") + k);
  R.nx = (int)hdr["ncols"];
  R.ny = (int)hdr["nrows"];
  R.h = hdr["cellsize"];
  if (R.nx < 1 || R.ny < 1 || R.nx != hdr["ncols"] || R.ny != hdr["nrows"])
    fail(path, ln, "malformed header: ncols/nrows must be positive integers");
  if (!(R.h > 0.0)) fail(path, ln, "malformed header: cellsize must be positive");
  R.x0 = hdr["xllcorner"] - (center_x ? 0.5 * R.h : 0.0);
  R.y0 = hdr["yllcorner"] - (center_y ? 0.5 * R.h : 0.0);
  if (hdr.count("nodata_value")) {
    R.has_nodata = true;
    R.nodata = hdr["nodata_value"];
  }
  R.v.assign((size_t)R.nx * R.ny, 0.0);
  R.is_nodata.assign(R.v.size(), 0);
  for (int r = 0; r < R.ny; ++r) {
    if (!std::getline(in, line)) fail(path, ln + 1, "expected " + std::to_string(R.ny) + " data rows, got " + std::to_string(r));
    ++ln;
    if (trim(line).empty()) {
      --r;
      continue;
    }
    std::istringstream ss(line);
    std::string tok;
    int c = 0;
    int j = R.ny - 1 - r;  // rows run north to south
    while (ss >> tok) {
      if (c >= R.nx) fail(path, ln, "data row " + std::to_string(r + 1) + " has more than ncols=" + std::to_string(R.nx) + " values");
      double x = to_num(path, ln, tok);
      size_t k = (size_t)c + (size_t)j * R.nx;
      R.v[k] = x;
      R.is_nodata[k] = R.has_nodata && x == R.nodata;
      ++c;
    }
    if (c != R.nx)
      fail(path, ln, "data row " + std::to_string(r + 1) + " has " + std::to_string(c) + " values, ncols=" + std::to_string(R.nx));
  }
  while (std::getline(in, line)) {
    ++ln;
    if (!trim(line).empty()) fail(path, ln, "extra data after nrows=" + std::to_string(R.ny) + " rows");
  }
  return R;
}

// ---- seeded synthetic terrains (sum of 10 random cosines, 5 m) ----
struct Cos {
  double kx, ky, ph;
};
std::vector<Cos> cosines(unsigned seed, double L) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  std::vector<Cos> c;
  for (int m = 0; m < 10; ++m) {
    double lam = L * (1.0 / 16.0 + U(rng) * (1.0 / 3.0 - 1.0 / 16.0));
    double ang = U(rng) * M_PI;
    double k = 2.0 * M_PI / lam;
    c.push_back({k * std::cos(ang), k * std::sin(ang), U(rng) * 2.0 * M_PI});
  }
  return c;
}

}  // namespace

Terrain load_terrain(const std::string& path) {
  Raster R = read_esri(path);
  Terrain T;
  T.nx = R.nx;
  T.ny = R.ny;
  T.h = R.h;
  T.x0 = R.x0;
  T.y0 = R.y0;
  T.b = std::move(R.v);
  for (size_t k = 0; k < T.b.size(); ++k)
    if (R.is_nodata[k]) T.b[k] = kNoDataBed;
  T.validate();
  return T;
}

std::vector<double> load_raster(const std::string& path, int* nx, int* ny, double* h, double* x0,
                                double* y0, double nodata_as) {
  Raster R = read_esri(path);
  for (size_t k = 0; k < R.v.size(); ++k)
    if (R.is_nodata[k]) R.v[k] = nodata_as;
  if (nx) *nx = R.nx;
  if (ny) *ny = R.ny;
  if (h) *h = R.h;
  if (x0) *x0 = R.x0;
  if (y0) *y0 = R.y0;
  return R.v;
}

void write_raster(const std::string& path, int nx, int ny, double x0, double y0, double h,
                  std::span<const double> v, double nodata, int precision) {
  if (v.size() != (size_t)nx * ny) throw ConfigError("write_raster: size mismatch for '" + path + "'");
  std::FILE* f = std::fopen(path.c_str(), "w");
  if (!f) throw std::runtime_error("cannot write '" + path + "': " + std::strerror(errno));
  std::fprintf(f, "ncols %d\nnrows %d\nxllcorner %.17g\nyllcorner %.17g\ncellsize %.17g\nNODATA_value %.17g\n",
               nx, ny, x0, y0, h, nodata);
  char fmt[16];
  std::snprintf(fmt, sizeof fmt, "%%.%de", precision);
  for (int r = 0; r < ny; ++r) {
    int j = ny - 1 - r;
    for (int i = 0; i < nx; ++i) {
      if (i) std::fputc(' ', f);
      double x = v[(size_t)i + (size_t)j * nx];
      std::fprintf(f, fmt, std::isfinite(x) ? x : nodata);
    }
    std::fputc('\n', f);
  }
  if (std::fclose(f) != 0) throw std::runtime_error("cannot write '" + path + "'");
}

// ---- scenario config ----------------------------------------------------------
ScenarioConfig load_scenario(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ConfigError("cannot open scenario '" + path + "'");
  std::string dir = path.find('/') == std::string::npos ? "." : path.substr(0, path.rfind('/'));
  auto resolve = [&](const std::string& p) { return p.empty() || p[0] == '/' ? p : dir + "/" + p; };
  ScenarioConfig C;
  std::string section, line;
  int ln = 0;
  SourceSpec* src = nullptr;
  auto edge = [&](const std::string& v) {
    std::string s = lower(v);
    if (s == "reflective") return EdgeKind::Reflective;
    if (s == "open") return EdgeKind::Open;
    fail(path, ln, "edge must be 'reflective' or 'open', got '" + v + "'");
  };
  auto boolean = [&](const std::string& v) {
    std::string s = lower(v);
    if (s == "true" || s == "1" || s == "on" || s == "yes") return true;
    if (s == "false" || s == "0" || s == "off" || s == "no") return false;
    fail(path, ln, "expected a boolean, got '" + v + "'");
  };
  while (std::getline(in, line)) {
    ++ln;
    std::string t = trim(line.substr(0, line.find('#')));
    if (t.empty()) continue;
    if (t.front() == '[') {
      if (t.back() != ']') fail(path, ln, "unterminated section header");
      std::string name = trim(t.substr(1, t.size() - 2));
      std::string kw = lower(name.substr(0, name.find(' ')));
      section = kw;
      src = nullptr;
      if (kw == "source") {
        C.sources.emplace_back();
        src = &C.sources.back();
        src->name = name.find(' ') == std::string::npos ? "source" : trim(name.substr(name.find(' ')));
      } else if (kw != "params" && kw != "control" && kw != "boundaries" && kw != "options" &&
                 kw != "initial" && kw != "wind" && kw != "run") {
        fail(path, ln, "unknown section [" + name + "]");
      }
      continue;
    }
    size_t eq = t.find('=');
    if (eq == std::string::npos) fail(path, ln, "expected key = value");
    std::string key = lower(trim(t.substr(0, eq))), val = trim(t.substr(eq + 1));
    std::string field = (section.empty() ? "" : section + ".") + key;
    auto num = [&]() { return to_num(path, ln, val); };
    if (section.empty() || section == "run") {
      if (key == "terrain") C.terrain_path = resolve(val);
      else if (key == "synthetic") C.synthetic = val;
      else if (key == "duration") C.duration = num();
      else if (key == "cadence") C.cadence = num();
      else if (key == "seed") C.seed = (unsigned)num();
      else fail(path, ln, "unknown key '" + field + "'");
    } else if (section == "params") {
      if (key == "g") C.params.g = num();
      else if (key == "n_manning") C.params.n_manning = num();
      else if (key == "nu") C.params.nu = num();
      else if (key == "omega_z") C.params.omega_z = num();
      else if (key == "latitude") C.params.omega_z = latitude_to_omega_z(num());
      else if (key == "c_a") C.params.c_a = num();
      else if (key == "rho_air") C.params.rho_air = num();
      else if (key == "rho_water") C.params.rho_water = num();
      else if (key == "eps_dry") C.params.eps_dry = num();
      else fail(path, ln, "unknown key '" + field + "'");
    } else if (section == "control") {
      if (key == "courant") C.control.courant = num();
      else if (key == "dt_max") C.control.dt_max = num();
      else if (key == "dt_min") C.control.dt_min = num();
      else fail(path, ln, "unknown key '" + field + "'");
    } else if (section == "boundaries") {
      if (key == "west") C.options.boundaries.west = edge(val);
      else if (key == "east") C.options.boundaries.east = edge(val);
      else if (key == "south") C.options.boundaries.south = edge(val);
      else if (key == "north") C.options.boundaries.north = edge(val);
      else if (key == "all") C.options.boundaries = BoundaryConfig::all(edge(val));
      else fail(path, ln, "unknown key '" + field + "'");
    } else if (section == "options") {
      if (key == "block_size") C.options.block_size = (int)num();
      else if (key == "skip_dry_blocks" || key == "skip") C.options.skip_dry_blocks = boolean(val);
      else if (key == "workers") C.options.workers = (int)num();
      else fail(path, ln, "unknown key '" + field + "'");
    } else if (section == "initial") {
      if (key == "mode") C.initial = lower(val);
      else if (key == "level") C.initial_level = num();
      else if (key == "raster") C.initial_raster = resolve(val);
      else fail(path, ln, "unknown key '" + field + "'");
    } else if (section == "wind") {
      if (key == "series") {  // t:wx:wy, ...
        std::stringstream ss(val);
        std::string item;
        while (std::getline(ss, item, ',')) {
          std::stringstream p(trim(item));
          std::string a, b, c;
          std::getline(p, a, ':');
          std::getline(p, b, ':');
          std::getline(p, c, ':');
          C.wind.series.push_back({to_num(path, ln, trim(a)), to_num(path, ln, trim(b)),
                                   to_num(path, ln, trim(c))});
        }
      } else if (key == "constant") {  // wx wy
        std::istringstream ss(val);
        std::string a, b;
        ss >> a >> b;
        C.wind = WindForcing::constant(to_num(path, ln, a), to_num(path, ln, b));
      } else {
        fail(path, ln, "unknown key '" + field + "'");
      }
    } else if (section == "source") {
      if (key == "kind") {
        std::string k = lower(val);
        if (k == "discharge") src->kind = SourceSpec::Kind::Discharge;
        else if (k == "rain") src->kind = SourceSpec::Kind::Rain;
        else fail(path, ln, "source kind must be discharge or rain");
      } else if (key == "cells") {  // i0 j0 i1 j1
        std::istringstream ss(val);
        std::string a[4];
        for (auto& x : a)
          if (!(ss >> x)) fail(path, ln, "cells needs 4 integers: i0 j0 i1 j1");
        src->cells = {(int)to_num(path, ln, a[0]), (int)to_num(path, ln, a[1]),
                      (int)to_num(path, ln, a[2]), (int)to_num(path, ln, a[3])};
      } else if (key == "hydrograph") {  // t:q, t:q
        std::stringstream ss(val);
        std::string item;
        while (std::getline(ss, item, ',')) {
          size_t c = item.find(':');
          if (c == std::string::npos) fail(path, ln, "hydrograph samples are t:q");
          src->hydrograph.push_back({to_num(path, ln, trim(item.substr(0, c))),
                                     to_num(path, ln, trim(item.substr(c + 1)))});
        }
        for (size_t k = 1; k < src->hydrograph.size(); ++k)
          if (!(src->hydrograph[k].t > src->hydrograph[k - 1].t))
            fail(path, ln, "source." + key + ": hydrograph times must be strictly increasing");
      } else if (key == "discharge") {
        src->hydrograph = {{0.0, num()}};
      } else if (key == "rate") {
        src->rate = num();
      } else if (key == "velocity") {
        std::istringstream ss(val);
        std::string a, b;
        ss >> a >> b;
        src->source_velocity = {to_num(path, ln, a), to_num(path, ln, b)};
      } else {
        fail(path, ln, "unknown key 'source." + key + "'");
      }
    }
  }
  if (C.terrain_path.empty() && C.synthetic.empty())
    throw ConfigError(path + ": scenario needs 'terrain = <file.asc>' or 'synthetic = ...'");
  if (!(C.duration > 0.0)) throw ConfigError(path + ": duration must be > 0");
  if (C.cadence == 0.0) C.cadence = C.duration;
  if (!(C.cadence > 0.0)) throw ConfigError(path + ": cadence must be > 0");
  C.params.validate();
  C.control.validate();
  C.wind.validate();
  return C;
}

Terrain scenario_terrain(const ScenarioConfig& C) {
  if (!C.terrain_path.empty()) return load_terrain(C.terrain_path);
  std::istringstream ss(C.synthetic);
  std::string kind;
  int n = 0;
  double h = 1.0;
  ss >> kind >> n >> h;
  if (n < 4) throw ConfigError("synthetic terrain: need 'KIND N H'");
  Terrain T;
  T.nx = T.ny = n;
  T.h = h;
  T.b.assign((size_t)n * n, 0.0);
  double L = n * h;
  if (kind == "lake" || kind == "floodplain") {
    auto cs = cosines(C.seed, L);
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        double x = T.xc(i), y = T.yc(j), z = 0.0;
        for (auto& c : cs) z += 0.5 * std::cos(c.kx * x + c.ky * y + c.ph);
        if (kind == "floodplain") {
          double yc = 0.5 * L + (L / 6.0) * std::sin(2.0 * M_PI * x / (L / 3.0));
          double w = 10.0 * h, p = std::max(0.0, 1.0 - ((y - yc) / w) * ((y - yc) / w));
          z += 5e-5 * (L - x) - 25.0 * p;
        }
        T.b[T.idx(i, j)] = z;
      }
  } else if (kind == "dam" || kind == "flat") {
    // flat bed
  } else {
    throw ConfigError("synthetic terrain: unknown kind '" + kind + "' (lake, floodplain, dam, flat)");
  }
  T.validate();
  return T;
}

FlowState scenario_initial_state(const ScenarioConfig& C, const Terrain& T) {
  FlowState s = FlowState::dry(T);
  std::string kind = C.synthetic.substr(0, C.synthetic.find(' '));
  if (C.initial == "dry") {
    if (kind == "dam")  // dam break: 1 m left of the centre line
      for (int j = 0; j < T.ny; ++j)
        for (int i = 0; i < T.nx / 2; ++i) s.H[T.idx(i, j)] = 1.0;
  } else if (C.initial == "level") {
    for (size_t k = 0; k < s.H.size(); ++k) s.H[k] = std::max(0.0, C.initial_level - T.b[k]);
  } else if (C.initial == "raster") {
    int nx = 0, ny = 0;
    s.H = load_raster(C.initial_raster, &nx, &ny, nullptr, nullptr, nullptr, 0.0);
    if (nx != T.nx || ny != T.ny) throw ConfigError("initial raster does not match the terrain");
  } else {
    throw ConfigError("initial.mode must be dry, level or raster");
  }
  s.enforce_dry_rule(C.params.eps_dry);
  for (size_t k = 0; k < s.H.size(); ++k)
    if (s.H[k] <= C.params.eps_dry) s.H[k] = 0.0;
  return s;
}

// ---- snapshots and summary ------------------------------------------------------
void write_snapshot(const FlowState& s, const Terrain& T, const PhysicalParams& P,
                    const std::string& dir, const std::string& stem) {
  size_t n = T.cells();
  std::vector<double> ux(n, 0.0), uy(n, 0.0), eta(n);
  for (size_t k = 0; k < n; ++k) {
    if (s.H[k] > P.eps_dry) {
      ux[k] = s.HUx[k] / s.H[k];
      uy[k] = s.HUy[k] / s.H[k];
    }
    eta[k] = s.H[k] + T.b[k];
  }
  std::string base = dir + "/" + stem;
  write_raster(base + "_H.asc", T.nx, T.ny, T.x0, T.y0, T.h, s.H);
  write_raster(base + "_Ux.asc", T.nx, T.ny, T.x0, T.y0, T.h, ux);
  write_raster(base + "_Uy.asc", T.nx, T.ny, T.x0, T.y0, T.h, uy);
  write_raster(base + "_eta.asc", T.nx, T.ny, T.x0, T.y0, T.h, eta);
}

SummaryRow summarize(const FlowState& s, const Terrain& T, const PhysicalParams& P) {
  SummaryRow r;
  r.t = s.t;
  r.volume = total_volume(s, T);
  size_t wet = 0;
  for (size_t k = 0; k < s.H.size(); ++k) {
    if (s.H[k] > P.eps_dry) {
      ++wet;
      double u = s.HUx[k] / s.H[k], v = s.HUy[k] / s.H[k];
      r.max_speed = std::max(r.max_speed, std::sqrt(u * u + v * v));
    }
  }
  r.wet_fraction = s.H.empty() ? 0.0 : double(wet) / double(s.H.size());
  return r;
}

SummaryWriter::SummaryWriter(const std::string& path) {
  f_ = std::fopen(path.c_str(), "w");
  if (!f_) throw std::runtime_error("cannot write '" + path + "'");
  std::fprintf(f_, "t,total_volume,wet_fraction,max_speed,tau,steps,source_volume,"
                   "boundary_outflow,clamp_deficit\n");
}

SummaryWriter::~SummaryWriter() {
  if (f_) std::fclose(f_);
}

void SummaryWriter::row(const SummaryRow& r) {
  std::fprintf(f_, "%.17g,%.17g,%.17g,%.17g,%.17g,%ld,%.17g,%.17g,%.17g\n", r.t, r.volume,
               r.wet_fraction, r.max_speed, r.tau, r.steps, r.source_volume, r.outflow_volume,
               r.clamp_deficit);
  std::fflush(f_);
  ++rows_;
}

}  // namespace swflood::io
