// extern "C" wrappers over the REFERENCE library (oracle/_ref/libemie_ref.so)
// so Python test infrastructure can call the reference's own functions with
// ctypes (fixture generation and oracle pinning). TEST INFRASTRUCTURE ONLY.
// Complex arrays are interleaved doubles (layout of std::complex<double>).
#include <complex>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "emie/cie.hpp"
#include "emie/greens.hpp"
#include "emie/hankel.hpp"
#include "emie/layered.hpp"
#include "emie/toeplitz.hpp"

using namespace emie;

namespace {
thread_local std::string g_err;

LayeredModel model_of(int L, const double* tops, const double* sigma) {
  LayeredModel m;
  m.tops.assign(tops, tops + L);
  for (int i = 0; i <= L; ++i) m.sigma.emplace_back(sigma[2 * i], sigma[2 * i + 1]);
  return m;
}

struct Ctx {
  LayeredModel model;
  AnomalyGrid grid;
  double omega = 0;
  CompressedGreensOperator op;
  SpectralOperator spec;
  SystemOperator sys;
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

void put(const std::vector<cdouble>& v, double* out) {
  std::memcpy(out, v.data(), v.size() * sizeof(cdouble));
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_design_weights(int oi, int oj, double hx, double hy, int alpha, int beta,
                       double* w, double* lam) {
  return guarded([&] {
    FilterWeights fw = design_weights(pair_geometry(oi, oj, hx, hy), alpha, beta);
    std::memcpy(w, fw.w.data(), fw.w.size() * 8);
    std::memcpy(lam, fw.lam.data(), fw.lam.size() * 8);
  });
}

double ref_kernel_output(int oi, int oj, double hx, double hy, int alpha, int beta, double s) {
  return kernel_output(pair_geometry(oi, oj, hx, hy), alpha, beta, s);
}

// st: [sig, eta, p, q, one_p, one_q, e2l, em1_2l, diag_a] each L+1 complex
int ref_spectral_state(int L, const double* tops, const double* sigma, double omega,
                       double lambda, int cond, double* st) {
  return guarded([&] {
    LayeredModel m = model_of(L, tops, sigma);
    SpectralLayerState s =
        build_spectral_state(m, omega, lambda, cond ? Gamma::cond : Gamma::unit);
    const std::vector<cdouble>* parts[9] = {&s.sig,   &s.eta,   &s.p,
                                            &s.q,     &s.one_p, &s.one_q,
                                            &s.e2l,   &s.em1_2l, &s.diag_a};
    for (int k = 0; k < 9; ++k) put(*parts[k], st + 2 * k * (L + 1));
  });
}

// tables: unit then cond, each 6 pair-orders x nz^2 complex
int ref_moment_tables(int L, const double* tops, const double* sigma, int nb,
                      const double* breaks, double omega, double lambda, double* tabs) {
  return guarded([&] {
    LayeredModel m = model_of(L, tops, sigma);
    VerticalPartition part = VerticalPartition::create(m, std::vector<double>(breaks, breaks + nb));
    SpectralLayerState su = build_spectral_state(m, omega, lambda, Gamma::unit);
    SpectralLayerState sc = build_spectral_state(m, omega, lambda, Gamma::cond);
    auto t = vertical_moment_tables(su, sc, part);
    const std::size_t nz2 = static_cast<std::size_t>(part.count()) * part.count();
    for (int k = 0; k < 6; ++k) put(t.first.w[k], tabs + 2 * k * nz2);
    for (int k = 0; k < 6; ++k) put(t.second.w[k], tabs + 2 * (6 + k) * nz2);
  });
}

void* ref_ctx_create(int L, const double* tops, const double* sigma, int nb,
                     const double* breaks, int nx, int ny, double hx, double hy,
                     double omega, const double* sigma_a) {
  Ctx* c = nullptr;
  int rc = guarded([&] {
    auto ctx = std::make_unique<Ctx>();
    ctx->model = model_of(L, tops, sigma);
    ctx->grid = make_grid(ctx->model, std::vector<double>(breaks, breaks + nb), nx, ny, hx,
                          hy, 0.0, 0.0);
    if (sigma_a) {
      std::memcpy(ctx->grid.sigma_a.data(), sigma_a, ctx->grid.sigma_a.size() * 16);
      ctx->grid.validate(ctx->model);
    }
    ctx->omega = omega;
    c = ctx.release();
  });
  return rc ? nullptr : c;
}

void ref_ctx_free(void* p) { delete static_cast<Ctx*>(p); }

// block at a signed offset in GreensBlock layout: xx yy zz xy (tri) xz yz (full)
int ref_assemble_block(void* p, int oi, int oj, double* out) {
  Ctx* c = static_cast<Ctx*>(p);
  return guarded([&] {
    GreensBlock b = assemble_block(c->grid, c->model, c->omega, oi, oj);
    double* o = out;
    for (const auto* v : {&b.xx, &b.yy, &b.zz, &b.xy, &b.xz, &b.yz}) {
      put(*v, o);
      o += 2 * v->size();
    }
  });
}

// assemble_block's lambda accumulation (greens.cpp:150-221, same loop order
// and the reference's own MomentMemo tables and v_functions) with
// caller-supplied filter weights w[6][nw] (greens.cpp:137 order) and
// abscissae lam[nw]: separates the filter design from the accumulation when
// a device build is compared with the reference (parity diagnostics only)
int ref_assemble_block_weights(void* p, int oi, int oj, const double* w, const double* lam, int nw,
                               double* out, double r_override) {
  Ctx* c = static_cast<Ctx*>(p);
  return guarded([&] {
    const AnomalyGrid& grid = c->grid;
    const int nz = grid.nz();
    const PairGeometry g = pair_geometry(oi, oj, grid.hx, grid.hy);
    const double R = r_override > 0.0 ? r_override : g.r;  // another reference distance (filter studies)
    const std::size_t ntri = static_cast<std::size_t>(nz) * (nz + 1) / 2, nfull = std::size_t(nz) * nz;
    std::vector<cdouble> a00(ntri), a20(ntri), a02(ntri), a11(ntri), az(ntri), axz(nfull), ayz(nfull);
    MomentMemo memo(c->model, grid.part, c->omega);
    for (int t = 0; t < nw; ++t) {
      const double lambda = lam[t] / R;
      const auto tabs = memo.get(lambda);
      const double w00 = w[t], w20 = w[nw + t], w02 = w[2 * nw + t];
      const double w11 = w[3 * nw + t], w10 = w[4 * nw + t], w01 = w[5 * nw + t];
      for (int k = 0; k < nz; ++k)
        for (int kp = 0; kp < nz; ++kp) {
          const VFunctions v = v_functions(tabs->first, tabs->second, k, kp, grid.sigma_b[k], c->omega);
          const cdouble f4 = lambda * v.v4;
          const std::size_t fi = static_cast<std::size_t>(k) * nz + kp;
          axz[fi] += w10 * f4;
          ayz[fi] += w01 * f4;
          if (k <= kp) {
            const std::size_t s = GreensBlock::tri(k, kp, nz);
            const cdouble f2 = (v.v1 + v.v3) / lambda;
            a00[s] += w00 * (lambda * v.v1);
            a20[s] += w20 * f2;
            a02[s] += w02 * f2;
            a11[s] += w11 * f2;
            az[s] += w00 * (lambda * (v.v2 + v.v5));
          }
        }
    }
    const double c3 = R * R * R / (4.0 * pi), c2 = R * R / (4.0 * pi), c1 = R / (4.0 * pi);
    cdouble* o = reinterpret_cast<cdouble*>(out);
    for (std::size_t s = 0; s < ntri; ++s) o[s] = c3 * a00[s] + c1 * a20[s];
    for (std::size_t s = 0; s < ntri; ++s) o[ntri + s] = c3 * a00[s] + c1 * a02[s];
    for (std::size_t s = 0; s < ntri; ++s) o[2 * ntri + s] = c3 * az[s];
    for (std::size_t s = 0; s < ntri; ++s) o[3 * ntri + s] = c1 * a11[s];
    for (std::size_t i = 0; i < nfull; ++i) o[4 * ntri + i] = c2 * axz[i];
    for (std::size_t i = 0; i < nfull; ++i) o[4 * ntri + nfull + i] = c2 * ayz[i];
  });
}

// v_functions (layered.cpp:397-408) of every (n, m) interval pair at one
// lambda: out[5][nz][nz] = v1..v5 (pins the device's V-function evaluation)
int ref_vfunctions(void* p, double lambda, double* out) {
  Ctx* c = static_cast<Ctx*>(p);
  return guarded([&] {
    const int nz = c->grid.nz();
    MomentMemo memo(c->model, c->grid.part, c->omega);
    const auto tabs = memo.get(lambda);
    cdouble* o = reinterpret_cast<cdouble*>(out);
    const std::size_t nz2 = std::size_t(nz) * nz;
    for (int n = 0; n < nz; ++n)
      for (int m = 0; m < nz; ++m) {
        const VFunctions v = v_functions(tabs->first, tabs->second, n, m, c->grid.sigma_b[n], c->omega);
        const std::size_t i = std::size_t(n) * nz + m;
        o[i] = v.v1;
        o[nz2 + i] = v.v2;
        o[2 * nz2 + i] = v.v3;
        o[3 * nz2 + i] = v.v4;
        o[4 * nz2 + i] = v.v5;
      }
  });
}

// nine components q[3a+b], each nz x nz
int ref_assemble_block_full(void* p, int oi, int oj, double* out) {
  Ctx* c = static_cast<Ctx*>(p);
  return guarded([&] {
    FilterDesigner d;
    MomentMemo memo(c->model, c->grid.part, c->omega);
    FullBlock f = assemble_block_full(c->grid, c->omega, oi, oj, d, memo);
    const std::size_t nz2 = static_cast<std::size_t>(f.nz) * f.nz;
    for (int q = 0; q < 9; ++q) put(f.q[q], out + 2 * q * nz2);
  });
}

// assemble_operator + transform_operator + build_system; op out offset-major
int ref_build(void* p, double* op_out, double* spec_out) {
  Ctx* c = static_cast<Ctx*>(p);
  return guarded([&] {
    c->op = assemble_operator(c->grid, c->model, c->omega);
    c->spec = transform_operator(c->op);
    c->sys = build_system(c->grid, c->spec);
    if (op_out) {
      double* o = op_out;
      for (const GreensBlock& b : c->op.blocks)
        for (const auto* v : {&b.xx, &b.yy, &b.zz, &b.xy, &b.xz, &b.yz}) {
          put(*v, o);
          o += 2 * v->size();
        }
    }
    if (spec_out) {
      double* o = spec_out;
      for (const auto& v : c->spec.comp) {
        put(v, o);
        o += 2 * v.size();
      }
    }
  });
}

// replace the operator by a given offset-major compressed operator
int ref_set_operator(void* p, const double* op_in) {
  Ctx* c = static_cast<Ctx*>(p);
  return guarded([&] {
    const int nz = c->grid.nz();
    const std::size_t ntri = static_cast<std::size_t>(nz) * (nz + 1) / 2;
    const std::size_t nfull = static_cast<std::size_t>(nz) * nz;
    std::vector<GreensBlock> blocks(static_cast<std::size_t>(c->grid.nx) * c->grid.ny);
    const cdouble* z = reinterpret_cast<const cdouble*>(op_in);
    for (auto& b : blocks) {
      b.nz = nz;
      for (auto* v : {&b.xx, &b.yy, &b.zz, &b.xy, &b.xz, &b.yz}) {
        const std::size_t n = (v == &b.xz || v == &b.yz) ? nfull : ntri;
        v->assign(z, z + n);
        z += n;
      }
    }
    c->op = compress(c->grid.nx, c->grid.ny, std::move(blocks), c->omega);
    c->spec = transform_operator(c->op);
    c->sys = build_system(c->grid, c->spec);
  });
}

int ref_spec_dims(void* p, int* dims) {
  Ctx* c = static_cast<Ctx*>(p);
  dims[0] = c->spec.ex;
  dims[1] = c->spec.ey;
  dims[2] = c->spec.qx;
  dims[3] = c->spec.qy;
  return 0;
}

// which: 0 = apply(SpectralOperator), 1 = apply(SystemOperator), 2 = dense
int ref_apply(void* p, int which, const double* in, double* out) {
  Ctx* c = static_cast<Ctx*>(p);
  return guarded([&] {
    GridVector v(c->grid.nx, c->grid.ny, c->grid.nz());
    std::memcpy(v.a.data(), in, v.a.size() * 16);
    GridVector r = which == 0 ? apply(c->spec, v)
                   : which == 1 ? apply(c->sys, v)
                                : dense_reference_apply(c->op, v);
    put(r.a, out);
  });
}

int ref_system_diagonals(void* p, double* s, double* r1, double* r2) {
  Ctx* c = static_cast<Ctx*>(p);
  put(c->sys.s, s);
  std::memcpy(r1, c->sys.r1.data(), c->sys.r1.size() * 8);
  put(c->sys.r2, r2);
  return 0;
}

// solve_cie; report = [status, iterations, residual]; history up to hcap
int ref_solve(void* p, const double* rhs, double tol, int restart, int max_iters,
              double* x, double* report, double* history, int hcap, int* hlen) {
  Ctx* c = static_cast<Ctx*>(p);
  return guarded([&] {
    GridVector b(c->grid.nx, c->grid.ny, c->grid.nz());
    std::memcpy(b.a.data(), rhs, b.a.size() * 16);
    SolverConfig cfg;
    cfg.tol = tol;
    cfg.restart = restart;
    cfg.max_iters = max_iters;
    SolveReport rep;
    GridVector r = solve_cie(c->grid, c->model, c->spec, b, cfg, &rep);
    put(r.a, x);
    report[0] = static_cast<int>(rep.status);
    report[1] = rep.iterations;
    report[2] = rep.residual;
    *hlen = static_cast<int>(rep.history.size());
    for (int i = 0; i < hcap && i < *hlen; ++i) history[i] = rep.history[i];
  });
}

}  // extern "C"
