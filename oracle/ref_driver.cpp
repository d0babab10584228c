// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE ONLY (never shipped, never on
// the product path).
//
// A flat extern "C" face over the *unmodified* reference engine
// (/root/reference/proj, C++20, compiled from its own sources by
// oracle/Makefile into oracle/_ref/libmoeref.so).  Python tests, the golden
// fixture generator and bench.py's `--impl reference` / cpu_baseline legs load
// it with ctypes.  Every function here only marshals raw buffers into the
// reference's value types and calls the reference's public API:
//
//   quantize                 proj/include/moeinfer/quantize.hpp:56-57
//   dequantize_naive/fast    proj/include/moeinfer/dequant.hpp:73-74
//   gate_top1                proj/include/moeinfer/routing.hpp:40-41
//   build_routing_plan       proj/include/moeinfer/routing.hpp:43-45
//   permute_rows             proj/include/moeinfer/routing.hpp:48
//   unpermute_and_scale      proj/include/moeinfer/routing.hpp:53-54
//   grouped_gemm_f16/quant   proj/include/moeinfer/grouped_gemm.hpp:65-82
//   layer_norm               proj/include/moeinfer/model.hpp:139-140
//   gate_logits_f32          proj/include/moeinfer/model.hpp:159-161
//   moe_ffn_forward          proj/include/moeinfer/model.hpp:154-156
//   ref::moe_per_token       proj/include/moeinfer/reference.hpp:62-63
//   ref::quantize            proj/include/moeinfer/reference.hpp:41
//   random_model / quantize_model / save_model / load_model
//                            proj/include/moeinfer/model.hpp:114-118,
//                            proj/include/moeinfer/checkpoint.hpp:41-42
//
// The one thing the reference lacks is top-k>1 gating.
// ref_moe_ffn_forward_topk composes the reference's own primitives
// (layer_norm, gate_logits_f32, grouped_gemm_*, half arithmetic) around the
// top-k extension documented in DESIGN.md §3 so the CPU baseline can time the
// same top-2 workload the GPU runs; for k == 1 it is bit-identical to
// moe_ffn_forward (checked in tests/test_oracle_vs_ref.py).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "moeinfer/checkpoint.hpp"
#include "moeinfer/dequant.hpp"
#include "moeinfer/grouped_gemm.hpp"
#include "moeinfer/model.hpp"
#include "moeinfer/quantize.hpp"
#include "moeinfer/reference.hpp"
#include "moeinfer/routing.hpp"

using namespace moe;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

HalfMat mat(const uint16_t* p, size_t r, size_t c) {
  HalfMat m(r, c);
  if (p != nullptr) std::memcpy(m.data.data(), p, r * c * 2);
  return m;
}
HalfTensor3 t3(const uint16_t* p, size_t e, size_t m, size_t n) {
  HalfTensor3 t(e, m, n);
  std::memcpy(t.data.data(), p, e * m * n * 2);
  return t;
}
std::vector<Half> vec(const uint16_t* p, size_t n) {
  std::vector<Half> v(n);
  std::memcpy(v.data(), p, n * 2);
  return v;
}
void out_mat(const HalfMat& m, uint16_t* dst) {
  std::memcpy(dst, m.data.data(), m.data.size() * 2);
}
QuantizedExpertWeights qw_from(const uint8_t* packed, const uint16_t* scales,
                               size_t e, size_t m, size_t n, int bits) {
  QuantizedExpertWeights q;
  q.bits = bits == 4 ? QuantBits::b4 : QuantBits::b8;
  q.e = e;
  q.m = m;
  q.n = n;
  const size_t nb = bits == 4 ? e * m * n / 2 : e * m * n;
  q.packed.assign(packed, packed + nb);
  q.scales = vec(scales, e * n);
  return q;
}
std::vector<GroupedProblem> problems_from(const uint32_t* p, size_t np) {
  std::vector<GroupedProblem> ps(np);
  for (size_t i = 0; i < np; ++i) ps[i] = {p[3 * i], p[3 * i + 1], p[3 * i + 2]};
  return ps;
}
void traffic_out(const TrafficCounter& tc, uint64_t* t) {
  if (t) {
    t[0] = tc.weight_bytes_read;
    t[1] = tc.activation_bytes_read;
    t[2] = tc.bytes_written;
  }
}

struct Layer {
  MoeFfn w;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_quantize(const uint16_t* w, size_t e, size_t m, size_t n, int bits,
                 int threads, uint8_t* packed, uint16_t* scales) {
  return guarded([&] {
    if (bits != 4 && bits != 8) throw std::invalid_argument("bits must be 4 or 8");
    const auto q = quantize(t3(w, e, m, n), bits == 4 ? QuantBits::b4 : QuantBits::b8,
                            threads);
    std::memcpy(packed, q.packed.data(), q.packed.size());
    std::memcpy(scales, q.scales.data(), q.scales.size() * 2);
  });
}

// moe::ref::quantize (reference.hpp:41): logical codes + scales as doubles.
int ref_ref_quantize(const uint16_t* w, size_t e, size_t m, size_t n, int bits,
                     uint8_t* stored, double* scales) {
  return guarded([&] {
    const auto r = ref::quantize(t3(w, e, m, n), bits == 4 ? QuantBits::b4 : QuantBits::b8);
    std::memcpy(stored, r.stored.data(), r.stored.size());
    std::memcpy(scales, r.scales.data(), r.scales.size() * sizeof(double));
  });
}

int ref_pack_int4(const uint8_t* v, size_t count, uint8_t* out) {
  return guarded([&] {
    const auto p = pack_int4_interleaved(std::span<const uint8_t>(v, count));
    std::memcpy(out, p.data(), p.size());
  });
}

int ref_dequantize(const uint8_t* packed, const uint16_t* scales, size_t e,
                   size_t m, size_t n, int bits, int fast, uint16_t* out) {
  return guarded([&] {
    const auto q = qw_from(packed, scales, e, m, n, bits);
    const auto t = fast ? dequantize_fast(q) : dequantize_naive(q);
    std::memcpy(out, t.data.data(), t.data.size() * 2);
  });
}

int ref_gate_top1(const float* logits, size_t rows, size_t E, uint32_t* expert,
                  uint16_t* scale) {
  return guarded([&] {
    const auto d = gate_top1(std::span<const float>(logits, rows * E), rows, E);
    for (size_t r = 0; r < rows; ++r) {
      expert[r] = d[r].expert;
      scale[r] = d[r].scale.bits;
    }
  });
}

int ref_build_plan(const uint32_t* expert, const uint8_t* finished, size_t T,
                   size_t E, uint32_t* perm, uint32_t* inv, uint32_t* offsets,
                   uint32_t* active) {
  return guarded([&] {
    std::vector<GateDecision> d(T);
    for (size_t r = 0; r < T; ++r) d[r] = {uint32_t(r), expert[r], kHalfOne};
    const auto p = build_routing_plan(d, std::span<const uint8_t>(finished, T), E);
    std::memcpy(perm, p.permutation.data(), T * 4);
    std::memcpy(inv, p.inverse_permutation.data(), T * 4);
    std::memcpy(offsets, p.expert_offsets.data(), (E + 1) * 4);
    *active = p.active_rows;
  });
}

int ref_layer_norm(const uint16_t* x, size_t T, size_t d, const uint16_t* g,
                   const uint16_t* b, uint16_t* out) {
  return guarded([&] {
    LayerNormWeights ln{vec(g, d), vec(b, d)};
    out_mat(layer_norm(mat(x, T, d), ln), out);
  });
}

int ref_gate_logits(const uint16_t* xn, size_t T, size_t d, const uint16_t* gw,
                    const uint16_t* gb, size_t E, float* logits) {
  return guarded([&] {
    const auto l = gate_logits_f32(mat(xn, T, d), mat(gw, d, E), vec(gb, E));
    std::memcpy(logits, l.data(), l.size() * 4);
  });
}

// unpermute_and_scale over a top-1 plan built from (expert, finished).
int ref_unpermute(const uint16_t* y, size_t T, size_t cols, const uint32_t* expert,
                  const uint16_t* scale, const uint8_t* finished, size_t E,
                  uint16_t* out) {
  return guarded([&] {
    std::vector<GateDecision> d(T);
    for (size_t r = 0; r < T; ++r) d[r] = {uint32_t(r), expert[r], Half(scale[r])};
    const auto p = build_routing_plan(d, std::span<const uint8_t>(finished, T), E);
    out_mat(unpermute_and_scale(mat(y, T, cols), p, d), out);
  });
}

int ref_permute(const uint16_t* x, size_t T, size_t cols, const uint32_t* expert,
                const uint8_t* finished, size_t E, uint16_t* out) {
  return guarded([&] {
    std::vector<GateDecision> d(T);
    for (size_t r = 0; r < T; ++r) d[r] = {uint32_t(r), expert[r], kHalfOne};
    const auto p = build_routing_plan(d, std::span<const uint8_t>(finished, T), E);
    out_mat(permute_rows(mat(x, T, cols), p), out);
  });
}

// problems: np triples (expert, row_begin, row_end).
int ref_grouped_gemm_f16(const uint16_t* x, size_t rows, size_t m,
                         const uint32_t* problems, size_t np, const uint16_t* w,
                         size_t E, size_t n, const uint16_t* bias, int relu,
                         int threads, uint16_t* out, uint64_t* traffic) {
  return guarded([&] {
    TrafficCounter tc;
    const auto y = grouped_gemm_f16(mat(x, rows, m), problems_from(problems, np),
                                    t3(w, E, m, n), mat(bias, E, n),
                                    relu ? Activation::relu : Activation::none, &tc,
                                    threads);
    out_mat(y, out);
    traffic_out(tc, traffic);
  });
}

int ref_grouped_gemm_quant(const uint16_t* x, size_t rows, size_t m,
                           const uint32_t* problems, size_t np,
                           const uint8_t* packed, const uint16_t* scales, int bits,
                           size_t E, size_t n, const uint16_t* bias, int relu,
                           int fused, int threads, uint16_t* out,
                           uint64_t* traffic) {
  return guarded([&] {
    TrafficCounter tc;
    const auto y = grouped_gemm_quant(
        mat(x, rows, m), problems_from(problems, np),
        qw_from(packed, scales, E, m, n, bits), mat(bias, E, n),
        relu ? Activation::relu : Activation::none, &tc, threads,
        fused ? DequantMode::fused : DequantMode::separate_pass);
    out_mat(y, out);
    traffic_out(tc, traffic);
  });
}

// ---- whole-layer handles ---------------------------------------------------
// bits: 16 (fp16 experts), 8 or 4 (quantized by the reference quantizer).
void* ref_layer_create(size_t d, size_t f, size_t E, const uint16_t* ln_g,
                       const uint16_t* ln_b, const uint16_t* gw, const uint16_t* gb,
                       const uint16_t* w1, const uint16_t* b1, const uint16_t* w2,
                       const uint16_t* b2, int bits, int threads) {
  Layer* L = nullptr;
  const int st = guarded([&] {
    L = new Layer;
    L->w.ln = {vec(ln_g, d), vec(ln_b, d)};
    L->w.gate_w = mat(gw, d, E);
    L->w.gate_b = vec(gb, E);
    L->w.b1 = mat(b1, E, f);
    L->w.b2 = mat(b2, E, d);
    HalfTensor3 W1 = t3(w1, E, d, f), W2 = t3(w2, E, f, d);
    if (bits == 16) {
      L->w.w1 = std::move(W1);
      L->w.w2 = std::move(W2);
    } else {
      const QuantBits qb = bits == 4 ? QuantBits::b4 : QuantBits::b8;
      L->w.qw1 = quantize(W1, qb, threads);
      L->w.qw2 = quantize(W2, qb, threads);
    }
  });
  if (st != 0) {
    delete L;
    return nullptr;
  }
  return L;
}

// Same, from already-quantized payloads (reference layout) -- lets tests hand
// the exact GPU-quantized codes to the reference.
void* ref_layer_create_quant(size_t d, size_t f, size_t E, const uint16_t* ln_g,
                             const uint16_t* ln_b, const uint16_t* gw,
                             const uint16_t* gb, const uint8_t* q1,
                             const uint16_t* s1, const uint16_t* b1,
                             const uint8_t* q2, const uint16_t* s2,
                             const uint16_t* b2, int bits) {
  Layer* L = nullptr;
  const int st = guarded([&] {
    L = new Layer;
    L->w.ln = {vec(ln_g, d), vec(ln_b, d)};
    L->w.gate_w = mat(gw, d, E);
    L->w.gate_b = vec(gb, E);
    L->w.b1 = mat(b1, E, f);
    L->w.b2 = mat(b2, E, d);
    L->w.qw1 = qw_from(q1, s1, E, d, f, bits);
    L->w.qw2 = qw_from(q2, s2, E, f, d, bits);
  });
  if (st != 0) {
    delete L;
    return nullptr;
  }
  return L;
}

void ref_layer_destroy(void* h) { delete static_cast<Layer*>(h); }

// Exports the reference-quantized payload of a layer (bits 4/8 only).
int ref_layer_export_quant(void* h, uint8_t* q1, uint16_t* s1, uint8_t* q2,
                           uint16_t* s2) {
  return guarded([&] {
    const Layer* L = static_cast<Layer*>(h);
    if (!L->w.quantized()) throw std::invalid_argument("layer is not quantized");
    std::memcpy(q1, L->w.qw1->packed.data(), L->w.qw1->packed.size());
    std::memcpy(s1, L->w.qw1->scales.data(), L->w.qw1->scales.size() * 2);
    std::memcpy(q2, L->w.qw2->packed.data(), L->w.qw2->packed.size());
    std::memcpy(s2, L->w.qw2->scales.data(), L->w.qw2->scales.size() * 2);
  });
}

// moe::moe_ffn_forward (model.cpp:299-349), top-1, unmodified.
int ref_layer_forward(void* h, const uint16_t* x, size_t T, size_t d,
                      const uint8_t* finished, int threads, uint16_t* out,
                      uint64_t* traffic6) {
  return guarded([&] {
    const Layer* L = static_cast<Layer*>(h);
    ModelTraffic tr;
    const auto y = moe_ffn_forward(mat(x, T, d), L->w,
                                   std::span<const uint8_t>(finished, T), &tr, threads);
    out_mat(y, out);
    if (traffic6) {
      traffic_out(tr.expert, traffic6);
      traffic_out(tr.other, traffic6 + 3);
    }
  });
}

// moe::ref::moe_per_token (reference.cpp:167-239), top-1.
int ref_layer_per_token(void* h, const uint16_t* x, size_t T, size_t d,
                        const uint8_t* finished, uint16_t* out) {
  return guarded([&] {
    const Layer* L = static_cast<Layer*>(h);
    out_mat(ref::moe_per_token(mat(x, T, d), L->w, std::span<const uint8_t>(finished, T)),
            out);
  });
}

// Top-k MoE layer built from the reference's primitives (see header note).
int ref_layer_forward_topk(void* h, const uint16_t* x, size_t T, size_t d,
                           const uint8_t* finished, int k, int threads,
                           uint16_t* out) {
  return guarded([&] {
    const Layer* L = static_cast<Layer*>(h);
    const MoeFfn& w = L->w;
    const size_t E = w.gate_w.cols;
    if (k < 1 || static_cast<size_t>(k) > E) throw std::invalid_argument("bad k");
    const HalfMat xm = mat(x, T, d);
    const HalfMat xn = layer_norm(xm, w.ln);
    const auto logits = gate_logits_f32(xn, w.gate_w, w.gate_b);
    const size_t S = T * k;
    std::vector<uint32_t> ex(S);
    std::vector<Half> sc(S);
    for (size_t r = 0; r < T; ++r) {
      const float* l = logits.data() + r * E;
      for (size_t j = 0; j < E; ++j)
        if (!std::isfinite(l[j])) throw std::invalid_argument("gate: non-finite logit");
      std::vector<char> taken(E, 0);
      for (int s = 0; s < k; ++s) {
        size_t best = E;
        for (size_t j = 0; j < E; ++j) {
          if (taken[j]) continue;
          if (best == E || l[j] > l[best]) best = j;
        }
        taken[best] = 1;
        ex[r * k + s] = static_cast<uint32_t>(best);
      }
      const float mx = l[ex[r * k]];
      float sum = 0.0f;
      for (size_t j = 0; j < E; ++j) sum += std::exp(l[j] - mx);
      for (int s = 0; s < k; ++s)
        sc[r * k + s] = f32_to_half(std::exp(l[ex[r * k + s]] - mx) / sum);
    }
    // Stable counting sort over slots (slot = r*k + s), finished -> key E.
    std::vector<uint32_t> counts(E + 1, 0), cursor(E + 1, 0);
    auto key = [&](size_t i) { return finished[i / k] ? E : ex[i]; };
    for (size_t i = 0; i < S; ++i) ++counts[key(i)];
    RoutingPlan plan;
    plan.expert_offsets.resize(E + 1);
    uint32_t run = 0;
    for (size_t e = 0; e <= E; ++e) {
      if (e < E) plan.expert_offsets[e] = run;
      cursor[e] = run;
      run += counts[e];
    }
    plan.active_rows = run - counts[E];
    plan.expert_offsets[E] = plan.active_rows;
    plan.permutation.assign(S, 0);
    plan.inverse_permutation.assign(S, 0);
    for (size_t i = 0; i < S; ++i) {
      const uint32_t pos = cursor[key(i)]++;
      plan.permutation[pos] = static_cast<uint32_t>(i);
      plan.inverse_permutation[i] = pos;
    }
    HalfMat xp(S, d);
    for (size_t p = 0; p < S; ++p) {
      const auto src = xn.row(plan.permutation[p] / k);
      std::copy(src.begin(), src.end(), xp.row(p).begin());
    }
    const auto problems = make_grouped_problems(plan);
    HalfMat hmid, y;
    if (w.quantized()) {
      hmid = grouped_gemm_quant(xp, problems, *w.qw1, w.b1, Activation::relu, nullptr, threads);
      y = grouped_gemm_quant(hmid, problems, *w.qw2, w.b2, Activation::none, nullptr, threads);
    } else {
      hmid = grouped_gemm_f16(xp, problems, w.w1, w.b1, Activation::relu, nullptr, threads);
      y = grouped_gemm_f16(hmid, problems, w.w2, w.b2, Activation::none, nullptr, threads);
    }
    HalfMat o(T, d);
    for (size_t r = 0; r < T; ++r) {
      auto orow = o.row(r);
      const auto xr = xm.row(r);
      std::copy(xr.begin(), xr.end(), orow.begin());
      if (finished[r]) continue;
      for (int s = 0; s < k; ++s) {
        const auto yr = y.row(plan.inverse_permutation[r * k + s]);
        for (size_t c = 0; c < d; ++c)
          orow[c] = half_add(orow[c], half_mul(yr[c], sc[r * k + s]));
      }
    }
    out_mat(o, out);
  });
}


// Write a .moec checkpoint of random_model(cfg, seed), quantized to `bits`
// (16 = FP16) by quantize_model -- the reference's own writer
// (checkpoint.cpp:390-415), for the loader fixtures.
int ref_make_moec(const char* path, const uint32_t* cfg9, int bits, uint64_t seed) {
  return guarded([&] {
    ModelConfig c;
    uint32_t* f[] = {&c.d_model, &c.d_ffn, &c.n_enc_layers, &c.n_dec_layers, &c.n_experts,
                     &c.n_heads, &c.vocab_size, &c.moe_every, &c.max_seq_len};
    for (int i = 0; i < 9; ++i) *f[i] = cfg9[i];
    Model m = random_model(c, seed);
    if (bits != 16) m = quantize_model(m, bits == 8 ? QuantBits::b8 : QuantBits::b4, 1);
    save_model(m, path);
  });
}

// moe_ffn_forward of the i-th MoE block (file order: encoder, then decoder)
// of a loaded .moec (load_model, checkpoint.cpp:419-483).
int ref_moec_block_forward(const char* path, int block, const uint16_t* x, size_t T,
                           const uint8_t* finished, uint16_t* out) {
  return guarded([&] {
    const Model m = load_model(path);
    std::vector<const MoeFfn*> blocks;
    for (const auto& l : m.encoder)
      if (const auto* b = std::get_if<MoeFfn>(&l.ffn)) blocks.push_back(b);
    for (const auto& l : m.decoder)
      if (const auto* b = std::get_if<MoeFfn>(&l.ffn)) blocks.push_back(b);
    if (block < 0 || block >= (int)blocks.size()) throw std::out_of_range("block");
    const auto y = moe_ffn_forward(mat(x, T, m.config.d_model), *blocks[block],
                                   std::span<const uint8_t>(finished, T), nullptr, 1);
    out_mat(y, out);
  });
}

// encoder_forward (model.cpp:351-398) of a loaded .moec over `batch`
// sentences of `len` token ids: embeddings, every encoder layer (attention,
// then the MoE or dense FFN), final LayerNorm -> out (batch * len, d).
int ref_encoder_forward(const char* path, const int32_t* tokens, size_t batch, size_t len,
                        uint16_t* out) {
  return guarded([&] {
    const Model m = load_model(path);
    std::vector<std::vector<int32_t>> src(batch, std::vector<int32_t>(len));
    for (size_t s = 0; s < batch; ++s)
      for (size_t p = 0; p < len; ++p) src[s][p] = tokens[s * len + p];
    out_mat(encoder_forward(m, src, nullptr, 1), out);
  });
}

// a loaded model kept across calls (timing encoder_forward without the load)
void* ref_model_load(const char* path) {
  try {
    return new Model(load_model(path));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void ref_model_free(void* h) { delete static_cast<Model*>(h); }
int ref_model_encoder(void* h, const int32_t* tokens, size_t batch, size_t len, int threads,
                      uint16_t* out) {
  return guarded([&] {
    const Model& m = *static_cast<Model*>(h);
    std::vector<std::vector<int32_t>> src(batch, std::vector<int32_t>(len));
    for (size_t s = 0; s < batch; ++s)
      for (size_t p = 0; p < len; ++p) src[s][p] = tokens[s * len + p];
    out_mat(encoder_forward(m, src, nullptr, threads), out);
  });
}

}  // extern "C"
