// Drop-in host API — the SIREN SOS field (reference:
// proj/include/pact/nfield.hpp:37-233).
#ifndef PACT_B200_NFIELD_HPP
#define PACT_B200_NFIELD_HPP

#include <vector>

#include "pact/core.hpp"
#include "pact/io.hpp"

namespace pact {

struct SirenParams {
  int in_dim = 2;
  int hidden = 64;
  int n_hidden_layers = 2;
  double omega0 = 30.0;
  double out_scale = 100.0;
  double v0 = 1500.0;
  std::vector<double> theta;  // per layer: W row-major [rows][cols], then b

  int n_layers() const { return n_hidden_layers + 1; }
  /// (rows, cols) of layer l's weight matrix; the bias has `rows` entries.
  std::pair<int, int> layer_shape(int l) const {
    return {l == n_hidden_layers ? 1 : hidden, l == 0 ? in_dim : hidden};
  }
  size_t layer_offset(int l) const {
    size_t off = 0;
    for (int k = 0; k < l; ++k) {
      const auto [r, c] = layer_shape(k);
      off += static_cast<size_t>(r) * (c + 1);
    }
    return off;
  }
  const double* weights(int l) const { return theta.data() + layer_offset(l); }
  const double* bias(int l) const {
    const auto [r, c] = layer_shape(l);
    return theta.data() + layer_offset(l) + static_cast<size_t>(r) * c;
  }
  pact_siren c() const { return {in_dim, hidden, n_hidden_layers, omega0, out_scale, v0}; }
  size_t param_count() const {
    pact_siren s = c();
    return static_cast<size_t>(pact_siren_param_count(&s));
  }
};

inline size_t siren_param_count(int in_dim, int hidden, int n_hidden_layers) {
  pact_siren s{in_dim, hidden, n_hidden_layers, 30.0, 100.0, 1500.0};
  return static_cast<size_t>(pact_siren_param_count(&s));
}

/// init_siren (nfield.hpp:83-107): bit-identical parameters.
inline SirenParams init_siren(uint64_t seed, int hidden = 64, int n_hidden_layers = 2,
                              double omega0 = 30.0, double out_scale = 100.0, double v0 = 1500.0) {
  SirenParams p;
  p.hidden = hidden;
  p.n_hidden_layers = n_hidden_layers;
  p.omega0 = omega0;
  p.out_scale = out_scale;
  p.v0 = v0;
  pact_siren s = p.c();
  if (hidden >= 1 && n_hidden_layers >= 1) p.theta.resize(p.param_count());
  cuda::check(pact_init_siren(seed, &s, p.theta.data()));
  return p;
}

struct SosField {
  RasterGrid raster;
  CircularMask mask;
  std::vector<int> masked_indices;
  std::vector<Vec2> coords;
};

/// render_sos (nfield.hpp:145-162) — the SIREN runs on the GPU (fp32).
inline SosField render_sos(const SirenParams& params, const GridSpec& grid,
                           const CircularMask& mask) {
  grid.validate();
  if (!(mask.radius > 0.0)) throw ValidationError("render_sos: mask radius must be > 0");
  pact_grid g = grid.c();
  pact_mask m = mask.c();
  pact_siren s = params.c();
  SosField f;
  f.mask = mask;
  int n = pact_masked_count(&g, &m);
  std::vector<int32_t> idx(n > 0 ? n : 1);
  std::vector<float> co(2 * (n > 0 ? n : 1));
  cuda::check(pact_masked_pixels(&g, &m, idx.data(), co.data()));
  for (int i = 0; i < n; ++i) {
    f.masked_indices.push_back(idx[i]);
    Vec2 p = grid.world(idx[i] % grid.width, idx[i] / grid.width);
    f.coords.push_back({(p.x - mask.center.x) / mask.radius, (p.y - mask.center.y) / mask.radius});
  }
  cuda::Buffer<float> th(params.theta.size());
  cuda::upload_f32(th, params.theta);
  const size_t npx = static_cast<size_t>(grid.width) * grid.height;
  cuda::Buffer<float> dev(npx);
  cuda::check(pact_render_sos(cuda::context(), &s, th.ptr, &g, &m, nullptr, dev.ptr));
  f.raster = RasterGrid::zeros(grid);
  f.raster.values = cuda::download_f64(dev, params.v0);  // v = v0 + (v - v0)
  return f;
}

/// backprop_sos (nfield.hpp:166-233): gradient of sum_p grad_v[p] v(p).
inline std::vector<double> backprop_sos(const SirenParams& p, const SosField& field,
                                        const std::vector<double>& grad_v) {
  if (grad_v.size() != field.coords.size())
    throw ValidationError("backprop_sos: grad_v size does not match masked pixel count");
  GridSpec grid = field.raster.spec();
  pact_grid g = grid.c();
  pact_mask m = field.mask.c();
  pact_siren s = p.c();
  cuda::Buffer<float> th(p.theta.size());
  cuda::upload_f32(th, p.theta);
  cuda::Buffer<float> gv(grad_v.size());
  cuda::upload_f32(gv, grad_v);
  cuda::Buffer<double> out(p.theta.size());
  cuda::check(pact_siren_backward(cuda::context(), &s, th.ptr, &g, &m, gv.ptr, out.ptr));
  std::vector<double> grad(p.theta.size());
  out.download(grad.data());
  return grad;
}

// ---- SIRN checkpoints (nfield.hpp:235-289) ---------------------------------
// "SIRN", u32 n_layers, per layer u32 rows and u32 cols, f64 omega0,
// f64 out_scale, f64 v0, then the parameters as f32 in layer order (weights
// row-major, then bias).

inline void write_sirn(const std::string& path, const SirenParams& p) {
  io::detail::Encoder e;
  e.raw("SIRN", 4);
  e.put<uint32_t>(static_cast<uint32_t>(p.n_layers()));
  for (int l = 0; l < p.n_layers(); ++l) {
    const auto [r, c] = p.layer_shape(l);
    e.put<uint32_t>(static_cast<uint32_t>(r));
    e.put<uint32_t>(static_cast<uint32_t>(c));
  }
  e.put<double>(p.omega0);
  e.put<double>(p.out_scale);
  e.put<double>(p.v0);
  e.put_f32_array(p.theta);
  e.save(path);
}

inline SirenParams load_sirn(const std::string& path) {
  io::detail::Decoder d(path);
  d.magic("SIRN");
  const uint32_t n_layers = d.get<uint32_t>("n_layers");
  if (n_layers < 2 || n_layers > 64) throw ValidationError("SIRN: implausible layer count");
  std::vector<std::pair<uint32_t, uint32_t>> shape(n_layers);
  for (auto& sh : shape) {
    sh.first = d.get<uint32_t>("rows");
    sh.second = d.get<uint32_t>("cols");
  }
  SirenParams p;
  p.in_dim = static_cast<int>(shape.front().second);
  p.hidden = static_cast<int>(shape.front().first);
  p.n_hidden_layers = static_cast<int>(n_layers) - 1;
  const uint32_t h = static_cast<uint32_t>(p.hidden);
  for (uint32_t l = 1; l + 1 < n_layers; ++l)
    if (shape[l].first != h || shape[l].second != h)
      throw ValidationError("SIRN: inconsistent hidden layer shapes in " + path);
  if (shape.back().first != 1 || shape.back().second != h)
    throw ValidationError("SIRN: bad output layer shape in " + path);
  p.omega0 = d.get<double>("omega0");
  p.out_scale = d.get<double>("out_scale");
  p.v0 = d.get<double>("v0");
  if (!(p.omega0 > 0.0) || !std::isfinite(p.out_scale) || !(p.v0 > 0.0))
    throw ValidationError("SIRN: bad scalar fields in " + path);
  p.theta = d.f32_array(p.layer_offset(p.n_layers()), "theta",
                        "SIRN: non-finite parameter in " + path);
  return p;
}

}  // namespace pact

#endif
