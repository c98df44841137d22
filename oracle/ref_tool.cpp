// Golden-vector generator and CPU-baseline timer driving the REFERENCE
// implementation through its own public API (/root/reference/proj/include/emie).
// TEST INFRASTRUCTURE ONLY: linked against oracle/_ref/libemie_ref.so, never
// against the B200 product library.
//
//   emie_ref_tool golden <case.bin> <outdir>
//       assemble_operator (greens.cpp:332) -> save_operator EMG1 (greens.cpp:405)
//       transform_operator (toeplitz.cpp:92) -> spec.bin (six comps, mode-major)
//       apply(SpectralOperator) (toeplitz.cpp:163) per test vector -> applyB_i.bin
//       dense_reference_apply (toeplitz.cpp:285) when the grid is small -> denseB_i.bin
//       build_system + apply(SystemOperator) (cie.cpp:24, 56) -> applyA_i.bin
//       solve_cie (cie.cpp:240) per rhs -> solve_r.bin + meta.json
//   emie_ref_tool bench-apply <case.bin> <reps> <nrhs>
//       times apply(SystemOperator) on a synthetic spectral operator of the
//       case's shape (operator values do not change the cost), all OMP threads
//   emie_ref_tool snapshot-check <file> [<resave>]
//       loads an EMG1 snapshot with the reference's load_operator, prints its
//       dimensions and a checksum of every stored entry, and optionally writes
//       it back with the reference's save_operator
//   emie_ref_tool bench-greens <case.bin> <stride>
//       times assemble_block over every stride-th offset with the same
//       per-thread designers / shared memo / dynamic schedule as
//       assemble_operator (greens.cpp:332-371); prints seconds and count
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include <omp.h>

#include "emie/cie.hpp"
#include "emie/greens.hpp"
#include "emie/toeplitz.hpp"

using namespace emie;

namespace {

struct Case {
  LayeredModel model;
  std::vector<double> breaks;
  int nx = 0, ny = 0;
  double hx = 0, hy = 0, x0 = 0, y0 = 0, omega = 0;
  std::vector<cdouble> sigma_a;  // empty: background everywhere
  std::vector<std::vector<cdouble>> vecs, rhs;
  double tol = 1e-8;
  int restart = 40, max_iters = 500;
};

template <class T>
T rd(std::ifstream& is) {
  T v;
  is.read(reinterpret_cast<char*>(&v), sizeof v);
  if (!is) throw std::runtime_error("case file truncated");
  return v;
}

std::vector<double> rdv(std::ifstream& is, std::size_t n) {
  std::vector<double> v(n);
  is.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n * 8));
  if (!is) throw std::runtime_error("case file truncated");
  return v;
}

std::vector<cdouble> rdc(std::ifstream& is, std::size_t n) {
  std::vector<cdouble> v(n);
  is.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n * 16));
  if (!is) throw std::runtime_error("case file truncated");
  return v;
}

Case read_case(const char* path) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw std::runtime_error(std::string("cannot open ") + path);
  char magic[8];
  is.read(magic, 8);
  if (std::memcmp(magic, "EMCASE1", 8) != 0) throw std::runtime_error("bad case magic");
  Case c;
  const int L = rd<int32_t>(is);
  c.model.tops = rdv(is, L);
  c.model.sigma = rdc(is, L + 1);
  const int nb = rd<int32_t>(is);
  c.breaks = rdv(is, nb);
  c.nx = rd<int32_t>(is);
  c.ny = rd<int32_t>(is);
  c.hx = rd<double>(is);
  c.hy = rd<double>(is);
  c.x0 = rd<double>(is);
  c.y0 = rd<double>(is);
  c.omega = rd<double>(is);
  const std::size_t nz = nb - 1;
  const std::size_t cells = static_cast<std::size_t>(c.nx) * c.ny * nz;
  if (rd<int32_t>(is)) c.sigma_a = rdc(is, cells);
  const int nvec = rd<int32_t>(is);
  for (int i = 0; i < nvec; ++i) c.vecs.push_back(rdc(is, 3 * cells));
  const int nrhs = rd<int32_t>(is);
  for (int i = 0; i < nrhs; ++i) c.rhs.push_back(rdc(is, 3 * cells));
  c.tol = rd<double>(is);
  c.restart = rd<int32_t>(is);
  c.max_iters = rd<int32_t>(is);
  return c;
}

AnomalyGrid make_case_grid(const Case& c) {
  AnomalyGrid g = make_grid(c.model, c.breaks, c.nx, c.ny, c.hx, c.hy, c.x0, c.y0);
  if (!c.sigma_a.empty()) {
    g.sigma_a = c.sigma_a;
    g.validate(c.model);
  }
  return g;
}

GridVector as_field(const Case& c, const std::vector<cdouble>& a) {
  GridVector v(c.nx, c.ny, static_cast<int>(c.breaks.size()) - 1);
  v.a = a;
  return v;
}

void write_raw(const std::string& path, const std::vector<cdouble>& v) {
  std::ofstream os(path, std::ios::binary | std::ios::trunc);
  os.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * 16));
  if (!os) throw std::runtime_error("write failed: " + path);
}

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int golden(const char* case_path, const std::string& out) {
  Case c = read_case(case_path);
  AnomalyGrid g = make_case_grid(c);
  const double t0 = now();
  CompressedGreensOperator op = assemble_operator(g, c.model, c.omega);
  const double t1 = now();
  save_operator(out + "/op.emg1", op);
  SpectralOperator s = transform_operator(op);
  const double t2 = now();
  {
    std::vector<cdouble> all;
    for (const auto& v : s.comp) all.insert(all.end(), v.begin(), v.end());
    write_raw(out + "/spec.bin", all);
  }
  const std::size_t cells = static_cast<std::size_t>(g.nx) * g.ny * g.nz();
  for (std::size_t i = 0; i < c.vecs.size(); ++i) {
    GridVector v = as_field(c, c.vecs[i]);
    write_raw(out + "/applyB_" + std::to_string(i) + ".bin", apply(s, v).a);
    if (cells <= 4096)
      write_raw(out + "/denseB_" + std::to_string(i) + ".bin", dense_reference_apply(op, v).a);
  }
  SystemOperator sys = build_system(g, s);
  write_raw(out + "/sys_s.bin", sys.s);
  write_raw(out + "/sys_r2.bin", sys.r2);
  {
    std::vector<cdouble> r1(sys.r1.begin(), sys.r1.end());
    write_raw(out + "/sys_r1.bin", r1);
  }
  for (std::size_t i = 0; i < c.vecs.size(); ++i)
    write_raw(out + "/applyA_" + std::to_string(i) + ".bin",
              apply(sys, as_field(c, c.vecs[i])).a);
  std::ofstream meta(out + "/meta.json");
  meta.precision(17);
  meta << "{\"greens_s\": " << (t1 - t0) << ", \"transform_s\": " << (t2 - t1)
       << ", \"ex\": " << s.ex << ", \"ey\": " << s.ey << ", \"qx\": " << s.qx
       << ", \"qy\": " << s.qy << ", \"threads\": " << omp_get_max_threads()
       << ", \"solves\": [";
  for (std::size_t r = 0; r < c.rhs.size(); ++r) {
    SolverConfig cfg;
    cfg.tol = c.tol;
    cfg.restart = c.restart;
    cfg.max_iters = c.max_iters;
    SolveReport rep;
    const double a = now();
    GridVector x = solve_cie(g, c.model, s, as_field(c, c.rhs[r]), cfg, &rep);
    const double b = now();
    write_raw(out + "/solve_" + std::to_string(r) + ".bin", x.a);
    meta << (r ? ", " : "") << "{\"status\": " << static_cast<int>(rep.status)
         << ", \"iterations\": " << rep.iterations << ", \"residual\": " << rep.residual
         << ", \"seconds\": " << (b - a) << ", \"history\": [";
    for (std::size_t k = 0; k < rep.history.size(); ++k)
      meta << (k ? ", " : "") << rep.history[k];
    meta << "]}";
  }
  meta << "]}\n";
  return 0;
}

int bench_apply(const char* case_path, int reps, int nrhs) {
  Case c = read_case(case_path);
  AnomalyGrid g = make_case_grid(c);
  const int nz = g.nz();
  // synthetic spectra of the right shape (transform_operator's layout,
  // toeplitz.cpp:100-108); values do not change the apply's cost
  SpectralOperator s;
  s.nx = g.nx;
  s.ny = g.ny;
  s.nz = nz;
  s.omega = c.omega;
  s.ex = smooth_embedding_size(2 * g.nx - 1);
  s.ey = smooth_embedding_size(2 * g.ny - 1);
  s.qx = s.ex / 2 + 1;
  s.qy = s.ey / 2 + 1;
  const std::size_t ntri = static_cast<std::size_t>(nz) * (nz + 1) / 2;
  const std::size_t nfull = static_cast<std::size_t>(nz) * nz;
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (int k = 0; k < 6; ++k) {
    s.comp[k].resize(s.mode_count() * (k < 4 ? ntri : nfull));
    for (auto& z : s.comp[k]) z = cdouble(u(rng), u(rng)) * 1e-3;
  }
  SystemOperator sys = build_system(g, s);
  std::vector<GridVector> in;
  for (int r = 0; r < nrhs; ++r) {
    GridVector v(g.nx, g.ny, nz);
    for (auto& z : v.a) z = cdouble(u(rng), u(rng));
    in.push_back(std::move(v));
  }
  GridVector sink = apply(sys, in[0]);  // warm-up (plan creation)
  std::vector<double> times;
  for (int i = 0; i < reps; ++i) {
    const double a = now();
    for (int r = 0; r < nrhs; ++r) sink = apply(sys, in[r]);
    times.push_back(now() - a);
  }
  std::printf("{\"threads\": %d, \"nrhs\": %d, \"times\": [", omp_get_max_threads(), nrhs);
  for (std::size_t i = 0; i < times.size(); ++i) std::printf("%s%.6f", i ? ", " : "", times[i]);
  std::printf("], \"check\": %.6e}\n", std::abs(sink.a[0]));
  return 0;
}

int bench_greens(const char* case_path, int stride) {
  Case c = read_case(case_path);
  AnomalyGrid g = make_case_grid(c);
  const int n_off = g.nx * g.ny;
  std::vector<int> offs;
  for (int o = 0; o < n_off; o += stride) offs.push_back(o);
  const int nthreads = omp_get_max_threads();
  std::vector<std::unique_ptr<FilterDesigner>> designers;
  for (int t = 0; t < nthreads; ++t) designers.push_back(std::make_unique<FilterDesigner>());
  MomentMemo memo(c.model, g.part, c.omega);
  std::vector<GreensBlock> blocks(offs.size());
  const double a = now();
#pragma omp parallel for schedule(dynamic)
  for (int i = 0; i < static_cast<int>(offs.size()); ++i)
    blocks[i] = assemble_block(g, c.omega, offs[i] / g.nx, offs[i] % g.nx,
                               *designers[omp_get_thread_num()], memo);
  const double b = now();
  double chk = 0;
  for (const auto& bl : blocks) chk += std::abs(bl.xx[0]);
  std::printf("{\"threads\": %d, \"offsets\": %zu, \"total_offsets\": %d, \"seconds\": %.6f, "
              "\"check\": %.6e}\n",
              nthreads, offs.size(), n_off, b - a, chk);
  return 0;
}

// load an EMG1 snapshot with the reference's load_operator (greens.cpp:425-446)
// and print the same checksum as tests/cpp/dropin_snapshot.cpp
int snapshot_check(const char* path, const char* resave) {
  const auto op = load_operator(path);
  if (!op) {
    std::printf("{\"loaded\": false}\n");
    return 3;
  }
  double s = 0.0, w = 1.0;
  for (const auto& b : op->blocks)
    for (const auto* c : {&b.xx, &b.yy, &b.zz, &b.xy, &b.xz, &b.yz})
      for (const auto& v : *c) {
        s += w * (v.real() + 0.5 * v.imag());
        w = w * 1.000001 + 1e-3;
      }
  std::printf("{\"loaded\": true, \"nx\": %d, \"ny\": %d, \"nz\": %d, \"omega\": %.17g, \"checksum\": %.17g}\n",
              op->nx, op->ny, op->nz, op->omega, s);
  if (resave) save_operator(resave, *op);  // the reference's own writer, for a byte comparison
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc >= 4 && std::string(argv[1]) == "golden") return golden(argv[2], argv[3]);
    if (argc >= 5 && std::string(argv[1]) == "bench-apply")
      return bench_apply(argv[2], std::atoi(argv[3]), std::atoi(argv[4]));
    if (argc >= 4 && std::string(argv[1]) == "bench-greens")
      return bench_greens(argv[2], std::atoi(argv[3]));
    if (argc >= 3 && std::string(argv[1]) == "snapshot-check")
      return snapshot_check(argv[2], argc >= 4 ? argv[3] : nullptr);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "emie_ref_tool: %s\n", e.what());
    return 2;
  }
  std::fprintf(stderr, "usage: emie_ref_tool golden|bench-apply|bench-greens ...\n");
  return 1;
}
