// moeinfer_host.cpp -- the drop-in C++ API (include/moeinfer/*.hpp) over the
// C-ABI of libmoe_cuda.so (include/moe_cuda.h).
//
// Value semantics as in the reference (std::vector-backed containers in and
// out): every call validates on the host with the reference's messages
// (std::invalid_argument / std::out_of_range), uploads its operands, runs the
// sm_100a kernels, downloads the result.  No computation happens on the
// host except bookkeeping the reference also does on the host side of its
// API (make_grouped_problems, analytic TrafficCounter formulas).
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "moe_cuda.h"
#include "moeinfer/dequant.hpp"
#include "moeinfer/device.hpp"
#include "moeinfer/grouped_gemm.hpp"
#include "moeinfer/model.hpp"
#include "moeinfer/quantize.hpp"
#include "moeinfer/routing.hpp"

namespace moe {
namespace {

void check(int st) {
  if (st == MOE_OK) return;
  const std::string msg = moe_cuda_last_error();
  if (st == MOE_EINVAL) throw std::invalid_argument(msg);
  if (st == MOE_ERANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

// device buffer (default stream; D2H copies synchronise)
struct Dev {
  void* p = nullptr;
  size_t bytes = 0;
  explicit Dev(size_t n) : bytes(n) { check(moe_cuda_malloc(&p, n ? n : 16)); }
  Dev(const void* host, size_t n) : Dev(n) { up(host, n); }
  ~Dev() { moe_cuda_free(p); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  void up(const void* host, size_t n) { check(moe_cuda_memcpy(p, host, n, 0, nullptr)); }
  void down(void* host, size_t n) const { check(moe_cuda_memcpy(host, p, n, 1, nullptr)); }
  void zero() { check(moe_cuda_memset(p, 0, bytes, nullptr)); }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

const uint16_t* bits_of(const std::vector<Half>& v) {
  return reinterpret_cast<const uint16_t*>(v.data());
}
uint16_t* bits_of(std::vector<Half>& v) { return reinterpret_cast<uint16_t*>(v.data()); }

int gemm_mode() { return static_cast<int>(cuda::numerics()); }

void validate_problems(const HalfMat& x, std::span<const GroupedProblem> problems,
                       size_t n_experts, size_t m) {
  // proj/src/grouped_gemm.cpp:97-105
  require(x.cols == m, "grouped_gemm: activation width != weight rows");
  for (const auto& p : problems) {
    require(p.expert < n_experts, "grouped_gemm: expert out of range");
    require(p.row_begin <= p.row_end && p.row_end <= x.rows,
            "grouped_gemm: problem rows out of range");
  }
}

// run one grouped GEMM on the device over reference-layout weights
HalfMat run_grouped(const HalfMat& x, std::span<const GroupedProblem> problems, int bits,
                    const void* weights, size_t wbytes, const std::vector<Half>* scales,
                    size_t E, size_t m, size_t n, const HalfMat& bias, Activation act) {
  HalfMat out(x.rows, n);
  if (problems.empty() || x.rows == 0) return out;
  Dev dx(x.data.data(), x.size() * 2);
  Dev draw(weights, wbytes);
  Dev dtiled(static_cast<size_t>(moe_tiled_bytes(E, m, n, bits)));
  check(moe_tile_weights(draw.p, E, m, n, bits, dtiled.p, nullptr));
  std::vector<uint32_t> pr;
  for (const auto& p : problems) pr.insert(pr.end(), {p.expert, p.row_begin, p.row_end});
  Dev dp(pr.data(), pr.size() * 4);
  Dev dbias(bias.data.data(), bias.size() * 2);
  std::unique_ptr<Dev> dsc;
  if (scales) dsc = std::make_unique<Dev>(scales->data(), scales->size() * 2);
  Dev dout(out.size() * 2);
  dout.zero();  // rows outside every problem stay +0 (grouped_gemm.cpp:148)
  check(moe_grouped_gemm(dx.as<uint16_t>(), x.rows, m, dp.as<uint32_t>(),
                         static_cast<int64_t>(problems.size()), dtiled.p,
                         dsc ? dsc->as<uint16_t>() : nullptr, bits, E, n, dbias.as<uint16_t>(),
                         act == Activation::relu ? 1 : 0, gemm_mode(), dout.as<uint16_t>(),
                         nullptr));
  dout.down(out.data.data(), out.size() * 2);
  return out;
}

}  // namespace

// ------------------------------------------------------------------- dequant
Half debias_const_u8() {
  uint16_t a = 0, b = 0;
  moe_cuda_debias(&a, &b);
  return Half(a);
}
Half debias_const_u4() {
  uint16_t a = 0, b = 0;
  moe_cuda_debias(&a, &b);
  return Half(b);
}

// ------------------------------------------------------------------ quantize
// proj/src/quantize.cpp:14-32 restated for the host side of the API
Half quant_scale_from_maxabs(float maxabs, int qmax) {
  if (maxabs == 0.0f) return kHalfOne;
  const Half s = f32_to_half(maxabs / static_cast<float>(qmax));
  return s.bits == 0 ? kHalfMinSubnormal : s;
}

uint8_t quant_encode(Half w, Half scale, QuantBits bits) {
  const int qmax = quant_qmax(bits);
  long long q = std::llround(half_to_f64(w) / half_to_f64(scale));
  q = q < -qmax ? -qmax : (q > qmax ? qmax : q);
  return static_cast<uint8_t>(q + quant_offset(bits));
}

QuantizedExpertWeights quantize(const HalfTensor3& w, QuantBits bits, int /*threads*/) {
  require(w.e > 0 && w.m > 0 && w.n > 0, "quantize: empty weight tensor");
  if (bits == QuantBits::b4)
    require(w.n % 8 == 0, "quantize: 4-bit packing needs the column count divisible by 8");
  QuantizedExpertWeights q;
  q.bits = bits;
  q.e = w.e;
  q.m = w.m;
  q.n = w.n;
  q.packed.resize(bits == QuantBits::b4 ? w.size() / 2 : w.size());
  q.scales.resize(w.e * w.n);
  Dev dw(w.data.data(), w.size() * 2), dp(q.packed.size()), ds(q.scales.size() * 2);
  check(moe_quantize(dw.as<uint16_t>(), w.e, w.m, w.n, static_cast<int>(bits), dp.as<uint8_t>(),
                     ds.as<uint16_t>(), nullptr));
  dp.down(q.packed.data(), q.packed.size());
  ds.down(q.scales.data(), q.scales.size() * 2);
  return q;
}

std::vector<uint8_t> pack_int4_interleaved(std::span<const uint8_t> values) {
  require(values.size() % 8 == 0, "pack_int4_interleaved: length must be a multiple of 8");
  std::vector<uint8_t> out(values.size() / 2);
  if (values.empty()) return out;
  Dev dv(values.data(), values.size()), dp(out.size());
  check(moe_pack_int4(dv.as<uint8_t>(), values.size(), dp.as<uint8_t>(), nullptr));
  dp.down(out.data(), out.size());
  return out;
}

std::vector<uint8_t> unpack_int4_interleaved(std::span<const uint8_t> packed, size_t count) {
  require(count % 8 == 0, "unpack_int4_interleaved: count must be a multiple of 8");
  require(packed.size() * 2 == count, "unpack_int4_interleaved: packed size does not match count");
  std::vector<uint8_t> out(count);
  if (count == 0) return out;
  Dev dp(packed.data(), packed.size()), dv(count);
  check(moe_unpack_int4(dp.as<uint8_t>(), count, dv.as<uint8_t>(), nullptr));
  dv.down(out.data(), count);
  return out;
}

std::vector<uint8_t> unpack_expert(const QuantizedExpertWeights& qw, size_t ei) {
  require(ei < qw.e, "unpack_expert: expert index out of range");
  const auto slab = qw.expert_packed(ei);
  if (qw.bits == QuantBits::b8) return {slab.begin(), slab.end()};
  return unpack_int4_interleaved(slab, qw.m * qw.n);
}

// ------------------------------------------------------------------- dequant
static HalfTensor3 dequant(const QuantizedExpertWeights& qw, int fast) {
  // proj/src/dequant.cpp:32-41
  require(qw.e > 0 && qw.m > 0 && qw.n > 0, "dequantize: empty tensor");
  require(qw.scales.size() == qw.e * qw.n, "dequantize: scale count mismatch");
  const size_t want = qw.bits == QuantBits::b8 ? qw.e * qw.m * qw.n : qw.e * qw.m * qw.n / 2;
  require(qw.packed.size() == want, "dequantize: packed size mismatch");
  if (qw.bits == QuantBits::b4)
    require(qw.n % 8 == 0, "dequantize: 4-bit column count not a multiple of 8");
  HalfTensor3 out(qw.e, qw.m, qw.n);
  Dev dp(qw.packed.data(), qw.packed.size()), ds(qw.scales.data(), qw.scales.size() * 2);
  Dev dout(out.size() * 2);
  check(moe_dequantize(dp.as<uint8_t>(), ds.as<uint16_t>(), qw.e, qw.m, qw.n,
                       static_cast<int>(qw.bits), fast, dout.as<uint16_t>(), nullptr));
  dout.down(out.data.data(), out.size() * 2);
  return out;
}
HalfTensor3 dequantize_naive(const QuantizedExpertWeights& qw) { return dequant(qw, 0); }
HalfTensor3 dequantize_fast(const QuantizedExpertWeights& qw) { return dequant(qw, 1); }

void dequantize_fast_expert(const QuantizedExpertWeights& qw, size_t ei, Half* dst) {
  require(ei < qw.e, "dequantize: expert index out of range");
  QuantizedExpertWeights one;
  one.bits = qw.bits;
  one.e = 1;
  one.m = qw.m;
  one.n = qw.n;
  const auto slab = qw.expert_packed(ei);
  one.packed.assign(slab.begin(), slab.end());
  one.scales.assign(qw.scales.begin() + ei * qw.n, qw.scales.begin() + (ei + 1) * qw.n);
  const HalfTensor3 t = dequantize_fast(one);
  std::memcpy(dst, t.data.data(), t.size() * 2);
}

// ------------------------------------------------------------------- routing
std::vector<GateDecision> gate_top1(std::span<const float> logits, size_t rows,
                                    size_t n_experts) {
  require(rows > 0 && n_experts > 0, "gate_top1: empty input");
  require(logits.size() == rows * n_experts, "gate_top1: logits shape mismatch");
  Dev dl(logits.data(), logits.size() * 4), de(rows * 4), ds(rows * 2);
  check(moe_gate_topk(dl.as<float>(), rows, n_experts, 1, de.as<uint32_t>(), ds.as<uint16_t>(),
                      nullptr));
  std::vector<uint32_t> ex(rows);
  std::vector<uint16_t> sc(rows);
  de.down(ex.data(), rows * 4);
  ds.down(sc.data(), rows * 2);
  std::vector<GateDecision> out(rows);
  for (size_t r = 0; r < rows; ++r) out[r] = {static_cast<uint32_t>(r), ex[r], Half(sc[r])};
  return out;
}

RoutingPlan build_routing_plan(std::span<const GateDecision> decisions,
                               std::span<const uint8_t> finished, size_t n_experts) {
  const size_t t = decisions.size();
  require(t > 0, "build_routing_plan: no rows");
  require(finished.size() == t, "build_routing_plan: finished size mismatch");
  std::vector<uint32_t> ex(t);
  for (size_t r = 0; r < t; ++r) ex[r] = decisions[r].expert;
  Dev de(ex.data(), t * 4), df(finished.data(), t), dperm(t * 4), dinv(t * 4),
      doff((n_experts + 1) * 4), dact(4);
  check(moe_routing_plan(de.as<uint32_t>(), df.as<uint8_t>(), t, 1, n_experts,
                         dperm.as<uint32_t>(), dinv.as<uint32_t>(), doff.as<uint32_t>(), nullptr,
                         dact.as<uint32_t>(), nullptr));
  RoutingPlan p;
  p.permutation.resize(t);
  p.inverse_permutation.resize(t);
  p.expert_offsets.resize(n_experts + 1);
  dperm.down(p.permutation.data(), t * 4);
  dinv.down(p.inverse_permutation.data(), t * 4);
  doff.down(p.expert_offsets.data(), (n_experts + 1) * 4);
  dact.down(&p.active_rows, 4);
  return p;
}

HalfMat permute_rows(const HalfMat& x, const RoutingPlan& plan) {
  require(x.rows == plan.permutation.size(), "permute_rows: row count mismatch");
  HalfMat out(x.rows, x.cols);
  if (x.size() == 0) return out;
  Dev dx(x.data.data(), x.size() * 2), dperm(plan.permutation.data(), x.rows * 4),
      dout(x.size() * 2);
  check(moe_permute_rows(dx.as<uint16_t>(), x.cols, dperm.as<uint32_t>(), x.rows, 1,
                         dout.as<uint16_t>(), nullptr));
  dout.down(out.data.data(), out.size() * 2);
  return out;
}

HalfMat unpermute_and_scale(const HalfMat& y_perm, const RoutingPlan& plan,
                            std::span<const GateDecision> decisions) {
  require(y_perm.rows == plan.permutation.size(), "unpermute_and_scale: row count mismatch");
  require(decisions.size() == y_perm.rows, "unpermute_and_scale: decision count mismatch");
  HalfMat out(y_perm.rows, y_perm.cols);
  if (y_perm.size() == 0) return out;
  std::vector<uint16_t> sc(decisions.size());
  for (size_t r = 0; r < decisions.size(); ++r) sc[r] = decisions[r].scale.bits;
  Dev dy(y_perm.data.data(), y_perm.size() * 2), dperm(plan.permutation.data(), y_perm.rows * 4),
      dact(&plan.active_rows, 4), dsc(sc.data(), sc.size() * 2), dout(out.size() * 2);
  check(moe_unpermute_scale(dy.as<uint16_t>(), y_perm.rows, y_perm.cols, dperm.as<uint32_t>(),
                            dact.as<uint32_t>(), dsc.as<uint16_t>(), dout.as<uint16_t>(),
                            nullptr));
  dout.down(out.data.data(), out.size() * 2);
  return out;
}

// ------------------------------------------------------------------ grouped
std::vector<GroupedProblem> make_grouped_problems(const RoutingPlan& plan) {
  std::vector<GroupedProblem> out;
  for (size_t e = 0; e + 1 < plan.expert_offsets.size(); ++e)
    if (plan.expert_offsets[e + 1] > plan.expert_offsets[e])
      out.push_back({static_cast<uint32_t>(e), plan.expert_offsets[e], plan.expert_offsets[e + 1]});
  return out;
}

HalfMat grouped_gemm_f16(const HalfMat& x_perm, std::span<const GroupedProblem> problems,
                         const HalfTensor3& w, const HalfMat& bias, Activation act,
                         TrafficCounter* tc, int /*threads*/) {
  validate_problems(x_perm, problems, w.e, w.m);
  require(bias.rows == w.e && bias.cols == w.n, "grouped_gemm_f16: bias shape mismatch");
  HalfMat out = run_grouped(x_perm, problems, 16, w.data.data(), w.size() * 2, nullptr, w.e, w.m,
                            w.n, bias, act);
  if (tc != nullptr)
    for (const auto& p : problems) {
      const uint64_t rows = p.row_end - p.row_begin;
      tc->weight_bytes_read += w.m * w.n * 2;
      tc->activation_bytes_read += (rows * w.m + w.n) * 2;
      tc->bytes_written += rows * w.n * 2;
    }
  return out;
}

HalfMat grouped_gemm_quant(const HalfMat& x_perm, std::span<const GroupedProblem> problems,
                           const QuantizedExpertWeights& qw, const HalfMat& bias, Activation act,
                           TrafficCounter* tc, int /*threads*/, DequantMode mode) {
  validate_problems(x_perm, problems, qw.e, qw.m);
  require(bias.rows == qw.e && bias.cols == qw.n, "grouped_gemm_quant: bias shape mismatch");
  require(qw.scales.size() == qw.e * qw.n, "grouped_gemm_quant: scale count mismatch");
  const size_t code_bytes = qw.bits == QuantBits::b8 ? qw.m * qw.n : qw.m * qw.n / 2;
  require(qw.packed.size() == code_bytes * qw.e, "grouped_gemm_quant: packed size mismatch");
  // fused and separate-pass are numerically identical (grouped_gemm.cpp:191-200);
  // the device always dequantises in-kernel, the counters follow `mode`.
  HalfMat out = run_grouped(x_perm, problems, static_cast<int>(qw.bits), qw.packed.data(),
                            qw.packed.size(), &qw.scales, qw.e, qw.m, qw.n, bias, act);
  if (tc != nullptr)
    for (const auto& p : problems) {
      const uint64_t rows = p.row_end - p.row_begin, wdq = qw.m * qw.n * 2;
      tc->weight_bytes_read += code_bytes + qw.n * 2;
      tc->activation_bytes_read += (rows * qw.m + qw.n) * 2;
      tc->bytes_written += rows * qw.n * 2;
      if (mode == DequantMode::separate_pass) {
        tc->weight_bytes_read += wdq;
        tc->bytes_written += wdq;
      }
    }
  return out;
}

// --------------------------------------------------------------------- model
HalfMat layer_norm(const HalfMat& x, const LayerNormWeights& ln) {
  require(ln.gamma.size() == x.cols && ln.beta.size() == x.cols,
          "layer_norm: parameter size mismatch");
  HalfMat out(x.rows, x.cols);
  if (x.size() == 0) return out;
  Dev dx(x.data.data(), x.size() * 2), dg(ln.gamma.data(), x.cols * 2),
      db(ln.beta.data(), x.cols * 2), dout(x.size() * 2);
  check(moe_layer_norm(dx.as<uint16_t>(), x.rows, x.cols, dg.as<uint16_t>(), db.as<uint16_t>(),
                       dout.as<uint16_t>(), nullptr));
  dout.down(out.data.data(), out.size() * 2);
  return out;
}

std::vector<float> gate_logits_f32(const HalfMat& xn, const HalfMat& gate_w,
                                   std::span<const Half> gate_b, TrafficCounter* tc) {
  require(xn.cols == gate_w.rows, "gate: dimension mismatch");
  require(gate_b.size() == gate_w.cols, "gate: bias size mismatch");
  const size_t t = xn.rows, e = gate_w.cols;
  std::vector<float> out(t * e);
  if (t > 0 && e > 0) {
    Dev dx(xn.data.data(), xn.size() * 2), dw(gate_w.data.data(), gate_w.size() * 2),
        db(gate_b.data(), e * 2), dout(t * e * 4);
    check(moe_gate_logits(dx.as<uint16_t>(), t, xn.cols, dw.as<uint16_t>(), db.as<uint16_t>(), e,
                          dout.as<float>(), nullptr));
    dout.down(out.data(), out.size() * 4);
  }
  if (tc != nullptr) {
    tc->weight_bytes_read += gate_w.size() * 2;
    tc->activation_bytes_read += (t * xn.cols + e) * 2;
    tc->bytes_written += t * e * 4;
  }
  return out;
}

HalfMat moe_ffn_forward(const HalfMat& x, const MoeFfn& w, std::span<const uint8_t> finished,
                        ModelTraffic* tr, int /*threads*/) {
  require(finished.size() == x.rows, "moe_ffn: finished flag count mismatch");
  cuda::DeviceMoeFfn dev(w);
  HalfMat out = dev.forward(x, finished, 1, cuda::numerics());
  if (tr != nullptr) *tr += dev.last_traffic();
  return out;
}

MoeFfn quantize_moe_ffn(const MoeFfn& w, QuantBits bits, int threads) {
  require(!w.quantized(), "quantize_model: model is already quantized");
  MoeFfn q = w;
  q.qw1 = quantize(w.w1, bits, threads);
  q.qw2 = quantize(w.w2, bits, threads);
  q.w1 = HalfTensor3();
  q.w2 = HalfTensor3();
  return q;
}

MoeModel quantize_model(const MoeModel& m, QuantBits bits, int threads) {
  require(m.precision == Precision::f16, "quantize_model: source must be an fp16 model");
  MoeModel out;
  out.precision = bits == QuantBits::b8 ? Precision::int8 : Precision::int4;
  out.blocks.reserve(m.blocks.size());
  for (const MoeFfn& b : m.blocks) out.blocks.push_back(quantize_moe_ffn(b, bits, threads));
  return out;
}

// ---------------------------------------------------------------- device API
namespace cuda {

static Numerics g_numerics = Numerics::exact;
void set_numerics(Numerics n) { g_numerics = n; }
Numerics numerics() { return g_numerics; }

DeviceMoeFfn::DeviceMoeFfn(const MoeFfn& w) {
  const size_t d = w.gate_w.rows, E = w.gate_w.cols;
  require(d > 0 && E > 0, "moe_ffn: empty gate");
  require(w.ln.gamma.size() == d && w.ln.beta.size() == d, "layer_norm: parameter size mismatch");
  require(w.gate_b.size() == E, "gate: bias size mismatch");
  moe_layer_desc D{};
  D.d = static_cast<int64_t>(d);
  D.E = static_cast<int64_t>(E);
  D.ln_g = bits_of(w.ln.gamma);
  D.ln_b = bits_of(w.ln.beta);
  D.gate_w = reinterpret_cast<const uint16_t*>(w.gate_w.data.data());
  D.gate_b = bits_of(w.gate_b);
  D.b1 = reinterpret_cast<const uint16_t*>(w.b1.data.data());
  D.b2 = reinterpret_cast<const uint16_t*>(w.b2.data.data());
  if (w.quantized()) {
    const auto& q1 = *w.qw1;
    const auto& q2 = *w.qw2;
    require(q1.e == E && q1.m == d && q2.e == E && q2.n == d && q2.m == q1.n,
            "moe_ffn: expert shapes inconsistent with the gate");
    D.f = static_cast<int64_t>(q1.n);
    D.bits = static_cast<int>(q1.bits);
    D.q1 = q1.packed.data();
    D.q2 = q2.packed.data();
    D.s1 = bits_of(q1.scales);
    D.s2 = bits_of(q2.scales);
  } else {
    require(w.w1.e == E && w.w1.m == d && w.w2.e == E && w.w2.n == d && w.w2.m == w.w1.n,
            "moe_ffn: expert shapes inconsistent with the gate");
    D.f = static_cast<int64_t>(w.w1.n);
    D.bits = 16;
    D.w1 = reinterpret_cast<const uint16_t*>(w.w1.data.data());
    D.w2 = reinterpret_cast<const uint16_t*>(w.w2.data.data());
  }
  require(w.b1.rows == E && w.b1.cols == static_cast<size_t>(D.f) && w.b2.rows == E &&
              w.b2.cols == d,
          "moe_ffn: bias shape mismatch");
  check(moe_layer_create(&D, &h_));
  d_ = d;
  e_ = E;
}

DeviceMoeFfn::~DeviceMoeFfn() { moe_layer_destroy(h_); }

HalfMat DeviceMoeFfn::forward(const HalfMat& x, std::span<const uint8_t> finished, int top_k,
                              Numerics n) {
  require(x.cols == d_, "moe_ffn: activation width != d_model");
  require(finished.empty() || finished.size() == x.rows, "moe_ffn: finished flag count mismatch");
  HalfMat out(x.rows, x.cols);
  if (x.rows == 0) return out;
  check(moe_layer_forward_host(h_, reinterpret_cast<const uint16_t*>(x.data.data()),
                               finished.empty() ? nullptr : finished.data(), x.rows, top_k,
                               static_cast<int>(n), reinterpret_cast<uint16_t*>(out.data.data()),
                               nullptr));
  return out;
}

void DeviceMoeFfn::forward_device(const uint16_t* x, const uint8_t* finished, int64_t T, int top_k,
                                  Numerics n, uint16_t* out, void* stream) {
  check(moe_layer_forward(h_, x, finished, T, top_k, static_cast<int>(n), out, stream));
}

ModelTraffic DeviceMoeFfn::last_traffic() {
  uint64_t t[6] = {};
  check(moe_layer_traffic(h_, t, nullptr));
  ModelTraffic m;
  m.expert = {t[0], t[1], t[2]};
  m.other = {t[3], t[4], t[5]};
  return m;
}

}  // namespace cuda
}  // namespace moe
