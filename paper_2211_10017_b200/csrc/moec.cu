// moec.cu -- `.moec` checkpoint -> device MoE layers.
//
// Reads the reference's checkpoint format (proj/src/checkpoint.cpp:
// Writer/Reader :35-240, record walk :242-300, header :390-446): magic
// "MOEC", version 1, nine u32 config fields, precision tag, record count,
// length-prefixed records {name u16+bytes, dtype u8 (0 f16, 1 u8, 2 u4),
// layout u8 (0 dense, 1 interleaved), ndim u8, dims u64...; payload; for
// quantized records a u64 scale count + fp16 scales}, FNV-1a-64 of
// everything before the trailing checksum.  Every record is validated in
// the reference's serialization order with the reference's messages
// ("checkpoint: ..."); the records of each MoE block (enc.i.ffn /
// dec.i.ffn with i % moe_every == 0) are handed to moe_layer_create
// straight from the file image -- int4 / int8 payloads in the reference's
// packing and fp16 scales go to the device as stored (no host dequant) and
// are re-tiled on the device into the tcgen05/TMA weight layout.
// Attention, dense-FFN, embedding and projection records are checked and
// skipped (outside the hot path).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "encoder.cuh"

namespace {

constexpr uint32_t kVersion = 1;

uint64_t fnv1a(const uint8_t* p, size_t n) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

struct Fail {
  std::string what;
};

struct Rd {
  const std::vector<uint8_t>& in;
  size_t pos = 0;
  size_t end;
  void need(size_t n) const {
    if (pos + n > end) throw Fail{"truncated file"};
  }
  uint64_t uint(int bytes) {
    need(bytes);
    uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= (uint64_t)in[pos++] << (8 * i);
    return v;
  }
  const uint8_t* take(size_t n) {
    need(n);
    const uint8_t* p = in.data() + pos;
    pos += n;
    return p;
  }
  // one record header; returns a pointer to its payload
  const uint8_t* record(const std::string& name, uint8_t dtype, uint8_t layout,
                        std::initializer_list<uint64_t> dims, size_t payload) {
    const uint64_t len = uint(2);
    need(len);
    const std::string got(reinterpret_cast<const char*>(in.data() + pos), len);
    pos += len;
    if (got != name) throw Fail{"unexpected record '" + got + "', wanted '" + name + "'"};
    const uint8_t dt = (uint8_t)uint(1), ly = (uint8_t)uint(1);
    if (dt != dtype || ly != layout) throw Fail{"record '" + name + "' has wrong dtype"};
    if (uint(1) != dims.size()) throw Fail{"record rank mismatch"};
    for (uint64_t w : dims)
      if (uint(8) != w) throw Fail{"record shape mismatch"};
    return take(payload);
  }
  const uint16_t* f16(const std::string& name, std::initializer_list<uint64_t> dims) {
    uint64_t n = 1;
    for (uint64_t v : dims) n *= v;
    return reinterpret_cast<const uint16_t*>(record(name, 0, 0, dims, n * 2));
  }
};

struct Cfg {
  uint32_t d, f, nenc, ndec, E, heads, vocab, every, maxlen;
};

}  // namespace

struct moe_moec {
  Cfg cfg{};
  int precision = 0;
  std::vector<std::string> names;
  std::vector<moe_layer*> layers;
  std::unique_ptr<moecu::EncoderDev> enc;  // attention / dense-FFN weights (create_layers)
  ~moe_moec() {
    enc.reset();
    for (moe_layer* L : layers) moe_layer_destroy(L);
  }
};

namespace moecu {
EncoderDev* moec_encoder(moe_moec* M) { return M->enc.get(); }
moe_layer* moec_layer(moe_moec* M, int i) { return M->layers[i]; }
}  // namespace moecu

using namespace moecu;

namespace {

// Walk the file in the reference's order (checkpoint.cpp:242-300); for each
// MoE block fill a descriptor and (create) build its device layer.
int walk(const std::vector<uint8_t>& bytes, moe_moec* M, bool create) {
  try {
    if (bytes.size() < 12) throw Fail{"truncated file"};
    const size_t body = bytes.size() - 8;
    uint64_t stored = 0;
    for (int i = 0; i < 8; ++i) stored |= (uint64_t)bytes[body + i] << (8 * i);
    if (stored != fnv1a(bytes.data(), body)) throw Fail{"checksum mismatch"};
    Rd r{bytes, 0, body};
    if (std::memcmp(r.take(4), "MOEC", 4) != 0) throw Fail{"bad magic"};
    if (r.uint(4) != kVersion) throw Fail{"unsupported version"};
    Cfg& c = M->cfg;
    for (uint32_t* f : {&c.d, &c.f, &c.nenc, &c.ndec, &c.E, &c.heads, &c.vocab, &c.every, &c.maxlen})
      *f = (uint32_t)r.uint(4);
    // ModelConfig::validate (proj/src/model.cpp:15-27)
    if (!(c.d > 0 && c.heads > 0 && c.d % c.heads == 0))
      return set_error(MOE_EINVAL, "config: d_model must be a positive multiple of n_heads");
    if (!(c.f > 0 && c.f % 8 == 0)) return set_error(MOE_EINVAL, "config: d_ffn must be a positive multiple of 8");
    if (c.d % 8 != 0) return set_error(MOE_EINVAL, "config: d_model must be a multiple of 8");
    if (!(c.nenc > 0 && c.ndec > 0)) return set_error(MOE_EINVAL, "config: need layers");
    if (c.E == 0) return set_error(MOE_EINVAL, "config: need at least one expert");
    if (c.vocab < 4) return set_error(MOE_EINVAL, "config: vocab must cover BOS, EOS and payload");
    if (c.every < 1) return set_error(MOE_EINVAL, "config: moe_every must be >= 1");
    if (c.maxlen < 2) return set_error(MOE_EINVAL, "config: max_seq_len too small");
    const uint8_t prec = (uint8_t)r.uint(1);
    if (prec > 2) throw Fail{"bad precision tag"};
    M->precision = prec;
    const uint32_t n_records = (uint32_t)r.uint(4);
    const uint64_t d = c.d, f = c.f, E = c.E;
    uint64_t count = 0;
    // attention records; encoder layers' go to the device (encoder_forward)
    auto attn = [&](const std::string& p, EncLayerDev* dev) -> int {
      const uint16_t* g = r.f16(p + ".ln_g", {d});
      const uint16_t* b = r.f16(p + ".ln_b", {d});
      const uint16_t* wv[4];
      const uint16_t* bv[4];
      int i = 0;
      for (const char* w : {"q", "k", "v", "o"}) {
        wv[i] = r.f16(p + ".w" + w, {d, d});
        bv[i] = r.f16(p + ".b" + w, {d});
        ++i;
      }
      if (dev) {
        // W_q | W_k | W_v column-concatenated: one (d, 3d) projection
        std::vector<uint16_t> w3((size_t)d * 3 * d), b3((size_t)3 * d);
        for (uint64_t row = 0; row < d; ++row)
          for (int m = 0; m < 3; ++m)
            std::memcpy(&w3[row * 3 * d + m * d], wv[m] + row * d, d * 2);
        for (int m = 0; m < 3; ++m) std::memcpy(&b3[m * d], bv[m], d * 2);
        TRY(enc_linear(M->enc.get(), w3.data(), b3.data(), (int64_t)d, (int64_t)(3 * d), &dev->qkv));
        TRY(enc_linear(M->enc.get(), wv[3], bv[3], (int64_t)d, (int64_t)d, &dev->o));
      }
      if (dev) {
        TRY(enc_upload(M->enc.get(), g, (int64_t)d, &dev->ln_g));
        TRY(enc_upload(M->enc.get(), b, (int64_t)d, &dev->ln_b));
      }
      count += 10;
      return MOE_OK;
    };
    auto quant = [&](const std::string& name, uint64_t m, uint64_t n, const uint8_t** packed,
                     const uint16_t** scales) {
      const bool is4 = prec == 2;
      *packed = r.record(name, is4 ? 2 : 1, is4 ? 1 : 0, {E, m, n}, is4 ? E * m * n / 2 : E * m * n);
      if (r.uint(8) != E * n) throw Fail{"record '" + name + "' has wrong scale count"};
      *scales = reinterpret_cast<const uint16_t*>(r.take(E * n * 2));
    };
    auto ffn = [&](const std::string& p, uint32_t idx, EncLayerDev* dev) -> int {
      if (idx % c.every != 0) {  // dense FFN block
        const uint16_t* g = r.f16(p + ".ln_g", {d});
        const uint16_t* b = r.f16(p + ".ln_b", {d});
        const uint16_t* w1 = r.f16(p + ".w1", {d, f});
        const uint16_t* b1 = r.f16(p + ".b1", {f});
        const uint16_t* w2 = r.f16(p + ".w2", {f, d});
        const uint16_t* b2 = r.f16(p + ".b2", {d});
        if (dev) {
          TRY(enc_upload(M->enc.get(), g, (int64_t)d, &dev->fln_g));
          TRY(enc_upload(M->enc.get(), b, (int64_t)d, &dev->fln_b));
          TRY(enc_linear(M->enc.get(), w1, b1, (int64_t)d, (int64_t)f, &dev->w1));
          TRY(enc_linear(M->enc.get(), w2, b2, (int64_t)f, (int64_t)d, &dev->w2));
        }
        count += 6;
        return MOE_OK;
      }
      if (dev) dev->moe_block = (int)M->names.size();
      moe_layer_desc D{};
      D.d = (int64_t)d;
      D.f = (int64_t)f;
      D.E = (int64_t)E;
      D.bits = prec == 0 ? 16 : prec == 1 ? 8 : 4;
      D.ln_g = r.f16(p + ".ln_g", {d});
      D.ln_b = r.f16(p + ".ln_b", {d});
      D.gate_w = r.f16(p + ".gate_w", {d, E});
      D.gate_b = r.f16(p + ".gate_b", {E});
      if (prec == 0) {
        D.w1 = r.f16(p + ".w1", {E, d, f});
        D.w2 = r.f16(p + ".w2", {E, f, d});
      } else {
        quant(p + ".w1", d, f, &D.q1, &D.s1);
        quant(p + ".w2", f, d, &D.q2, &D.s2);
      }
      D.b1 = r.f16(p + ".b1", {E, f});
      D.b2 = r.f16(p + ".b2", {E, d});
      count += 8;
      M->names.push_back(p);
      if (create) {
        moe_layer* L = nullptr;
        const int st = moe_layer_create(&D, &L);
        if (st != MOE_OK) return st;
        M->layers.push_back(L);
      }
      return MOE_OK;
    };
    const uint16_t* tok = r.f16("tok_embed", {c.vocab, d});
    const uint16_t* pos = r.f16("pos_embed", {c.maxlen, d});
    count += 2;
    if (create) {
      M->enc = std::make_unique<EncoderDev>();
      EncoderDev* E = M->enc.get();
      E->d = d;
      E->f = f;
      E->heads = c.heads;
      E->vocab = c.vocab;
      E->maxlen = c.maxlen;
      E->layers.resize(c.nenc);
      TRY(enc_upload(E, tok, (int64_t)c.vocab * d, &E->tok));
      TRY(enc_upload(E, pos, (int64_t)c.maxlen * d, &E->pos));
    }
    for (uint32_t i = 0; i < c.nenc; ++i) {
      const std::string p = "enc." + std::to_string(i);
      EncLayerDev* dev = create ? &M->enc->layers[i] : nullptr;
      TRY(attn(p + ".attn", dev));
      TRY(ffn(p + ".ffn", i, dev));
    }
    for (uint32_t i = 0; i < c.ndec; ++i) {
      const std::string p = "dec." + std::to_string(i);
      TRY(attn(p + ".self", nullptr));
      TRY(attn(p + ".cross", nullptr));
      TRY(ffn(p + ".ffn", i, nullptr));
    }
    for (const char* nm : {"enc_ln_g", "enc_ln_b", "dec_ln_g", "dec_ln_b"}) {
      const uint16_t* v = r.f16(nm, {d});
      if (create && std::strcmp(nm, "enc_ln_g") == 0) TRY(enc_upload(M->enc.get(), v, (int64_t)d, &M->enc->ln_g));
      if (create && std::strcmp(nm, "enc_ln_b") == 0) TRY(enc_upload(M->enc.get(), v, (int64_t)d, &M->enc->ln_b));
    }
    r.f16("out_w", {d, c.vocab});
    r.f16("out_b", {c.vocab});
    count += 6;
    if (n_records != count) throw Fail{"record count mismatch"};
    if (r.pos != body) throw Fail{"trailing bytes"};
    return MOE_OK;
  } catch (const Fail& e) {
    return set_error(MOE_EIO, "checkpoint: %s", e.what.c_str());
  }
}

int read_file(const char* path, std::vector<uint8_t>* out) {
  FILE* fp = std::fopen(path, "rb");
  if (!fp) return set_error(MOE_EIO, "checkpoint: cannot open '%s'", path);
  std::fseek(fp, 0, SEEK_END);
  const long n = std::ftell(fp);
  std::fseek(fp, 0, SEEK_SET);
  out->resize(n > 0 ? (size_t)n : 0);
  const size_t got = n > 0 ? std::fread(out->data(), 1, (size_t)n, fp) : 0;
  std::fclose(fp);
  if ((long)got != n) return set_error(MOE_EIO, "checkpoint: read from '%s' failed", path);
  return MOE_OK;
}

}  // namespace

extern "C" {

int moe_moec_load(const char* path, int create_layers, moe_moec** out) {
  if (!path || !out) return set_error(MOE_EINVAL, "checkpoint: null argument");
  std::vector<uint8_t> bytes;
  TRY(read_file(path, &bytes));
  auto M = std::make_unique<moe_moec>();
  TRY(walk(bytes, M.get(), create_layers != 0));
  *out = M.release();
  return MOE_OK;
}

int moe_moec_info(const moe_moec* M, uint32_t* cfg9, int* precision, int* n_moe_blocks) {
  if (!M) return set_error(MOE_EINVAL, "checkpoint: null");
  if (cfg9) {
    const Cfg& c = M->cfg;
    const uint32_t v[9] = {c.d, c.f, c.nenc, c.ndec, c.E, c.heads, c.vocab, c.every, c.maxlen};
    std::memcpy(cfg9, v, sizeof v);
  }
  if (precision) *precision = M->precision;
  if (n_moe_blocks) *n_moe_blocks = (int)M->names.size();
  return MOE_OK;
}

int moe_moec_block(const moe_moec* M, int i, moe_layer** layer, char* name, size_t name_len) {
  if (!M || i < 0 || i >= (int)M->names.size())
    return set_error(MOE_ERANGE, "checkpoint: MoE block index out of range");
  if (layer) *layer = i < (int)M->layers.size() ? M->layers[i] : nullptr;
  if (name && name_len) {
    std::snprintf(name, name_len, "%s", M->names[i].c_str());
  }
  return MOE_OK;
}

int moe_moec_destroy(moe_moec* M) {
  delete M;
  return MOE_OK;
}

// A synthetic checkpoint in the reference's format (the records walk()
// reads, in the same order; checkpoint.cpp:390-415 writer layout) for
// benchmarks at model sizes no fixture covers: fp16 tensors ~ N(0, s) with
// random_model-like scales (s = 1/sqrt(fan-in) for projections, 0.02 for
// biases and embeddings, LN gamma 1 + 0.1 N, beta 0.05 N), quantized records
// random codes with per-column scales 1/(7 sqrt(fan-in)).  Deterministic in
// the seed; not a reference model (no parity use).
int moe_moec_write_synthetic(const char* path, const uint32_t* cfg9, int bits, uint64_t seed) {
  if (!path || !cfg9) return set_error(MOE_EINVAL, "checkpoint: null argument");
  if (bits != 4 && bits != 8 && bits != 16) return set_error(MOE_EINVAL, "checkpoint: bits must be 4, 8 or 16");
  FILE* fp = std::fopen(path, "wb");
  if (!fp) return set_error(MOE_EIO, "checkpoint: cannot open '%s'", path);
  uint64_t h = 0xcbf29ce484222325ull, rs = seed * 0x9e3779b97f4a7c15ull + 1;
  std::vector<uint8_t> buf;
  auto flush = [&]() {
    for (uint8_t b : buf) {
      h ^= b;
      h *= 0x100000001b3ull;
    }
    std::fwrite(buf.data(), 1, buf.size(), fp);
    buf.clear();
  };
  auto put = [&](uint64_t v, int n) {
    for (int i = 0; i < n; ++i) buf.push_back((uint8_t)(v >> (8 * i)));
    if (buf.size() > (1u << 24)) flush();
  };
  auto rnd = [&]() {  // xorshift64*
    rs ^= rs >> 12;
    rs ^= rs << 25;
    rs ^= rs >> 27;
    return rs * 0x2545f4914f6cdd1dull;
  };
  auto f2h = [](float f) -> uint16_t {  // RN, |f| well inside the fp16 range
    uint32_t x;
    std::memcpy(&x, &f, 4);
    const uint32_t sign = (x >> 16) & 0x8000u;
    const int e = (int)((x >> 23) & 0xFF) - 112;
    if (e <= 0) return (uint16_t)sign;
    uint32_t m = (x & 0x7FFFFFu), r = ((uint32_t)e << 10) | (m >> 13);
    const uint32_t rem = m & 0x1FFFu;
    if (rem > 0x1000u || (rem == 0x1000u && (r & 1u))) ++r;
    return (uint16_t)(sign | r);
  };
  auto normal = [&]() {  // sum of 4 uniforms, unit variance
    float a = 0.f;
    for (int i = 0; i < 4; ++i) a += (float)(rnd() >> 40) * (1.0f / 16777216.0f) - 0.5f;
    return a * 1.7320508f;
  };
  uint32_t nrec = 0;
  auto header = [&](const std::string& name, int dt, int ly, std::initializer_list<uint64_t> dims) {
    put(name.size(), 2);
    for (char ch : name) put((uint8_t)ch, 1);
    put(dt, 1);
    put(ly, 1);
    put(dims.size(), 1);
    for (uint64_t v : dims) put(v, 8);
    ++nrec;
  };
  auto f16rec = [&](const std::string& name, std::initializer_list<uint64_t> dims, float scale,
                    float offset) {
    header(name, 0, 0, dims);
    uint64_t n = 1;
    for (uint64_t v : dims) n *= v;
    for (uint64_t i = 0; i < n; ++i) put(f2h(offset + scale * normal()), 2);
  };
  const uint32_t d = cfg9[0], f = cfg9[1], nenc = cfg9[2], ndec = cfg9[3], E = cfg9[4];
  const uint32_t vocab = cfg9[6], every = cfg9[7], maxlen = cfg9[8];
  auto qrec = [&](const std::string& name, uint64_t m, uint64_t n) {
    const uint64_t payload = bits == 4 ? E * m * n / 2 : E * m * n;
    header(name, bits == 4 ? 2 : 1, bits == 4 ? 1 : 0, {E, m, n});
    for (uint64_t i = 0; i < payload; i += 8) {
      const uint64_t r = rnd();
      for (uint64_t j = 0; j < 8 && i + j < payload; ++j) put((r >> (8 * j)) & 0xFF, 1);
    }
    put(E * n, 8);
    const uint16_t sc = f2h(1.0f / (7.0f * std::sqrt((float)m)));
    for (uint64_t i = 0; i < E * n; ++i) put(sc, 2);
  };
  auto attn = [&](const std::string& p) {
    f16rec(p + ".ln_g", {d}, 0.1f, 1.0f);
    f16rec(p + ".ln_b", {d}, 0.05f, 0.f);
    for (const char* w : {"q", "k", "v", "o"}) {
      f16rec(p + ".w" + w, {d, d}, 1.0f / std::sqrt((float)d), 0.f);
      f16rec(p + ".b" + w, {d}, 0.02f, 0.f);
    }
  };
  auto ffn = [&](const std::string& p, uint32_t idx) {
    f16rec(p + ".ln_g", {d}, 0.1f, 1.0f);
    f16rec(p + ".ln_b", {d}, 0.05f, 0.f);
    if (idx % every != 0) {
      f16rec(p + ".w1", {d, f}, 1.0f / std::sqrt((float)d), 0.f);
      f16rec(p + ".b1", {f}, 0.02f, 0.f);
      f16rec(p + ".w2", {f, d}, 1.0f / std::sqrt((float)f), 0.f);
      f16rec(p + ".b2", {d}, 0.02f, 0.f);
      return;
    }
    f16rec(p + ".gate_w", {d, E}, 1.0f / std::sqrt((float)d), 0.f);
    f16rec(p + ".gate_b", {E}, 0.02f, 0.f);
    if (bits == 16) {
      f16rec(p + ".w1", {E, d, f}, 1.0f / std::sqrt((float)d), 0.f);
      f16rec(p + ".w2", {E, f, d}, 1.0f / std::sqrt((float)f), 0.f);
    } else {
      qrec(p + ".w1", d, f);
      qrec(p + ".w2", f, d);
    }
    f16rec(p + ".b1", {E, f}, 0.02f, 0.f);
    f16rec(p + ".b2", {E, d}, 0.02f, 0.f);
  };
  // header (the record count is patched in once known: it precedes the
  // records, so count first)
  uint32_t count = 2 + 6;
  for (uint32_t i = 0; i < nenc; ++i) count += 10 + (i % every ? 6 : 8);
  for (uint32_t i = 0; i < ndec; ++i) count += 20 + (i % every ? 6 : 8);
  for (char ch : std::string("MOEC")) put((uint8_t)ch, 1);
  put(kVersion, 4);
  for (int i = 0; i < 9; ++i) put(cfg9[i], 4);
  put(bits == 16 ? 0 : bits == 8 ? 1 : 2, 1);
  put(count, 4);
  f16rec("tok_embed", {vocab, d}, 0.02f, 0.f);
  f16rec("pos_embed", {maxlen, d}, 0.02f, 0.f);
  for (uint32_t i = 0; i < nenc; ++i) {
    const std::string p = "enc." + std::to_string(i);
    attn(p + ".attn");
    ffn(p + ".ffn", i);
  }
  for (uint32_t i = 0; i < ndec; ++i) {
    const std::string p = "dec." + std::to_string(i);
    attn(p + ".self");
    attn(p + ".cross");
    ffn(p + ".ffn", i);
  }
  for (const char* nm : {"enc_ln_g", "enc_ln_b", "dec_ln_g", "dec_ln_b"})
    f16rec(nm, {d}, nm[std::strlen(nm) - 1] == 'g' ? 0.1f : 0.05f, nm[std::strlen(nm) - 1] == 'g' ? 1.0f : 0.f);
  f16rec("out_w", {d, vocab}, 1.0f / std::sqrt((float)d), 0.f);
  f16rec("out_b", {vocab}, 0.02f, 0.f);
  flush();
  const bool ok_count = nrec == count;
  uint64_t hv = h;
  for (int i = 0; i < 8; ++i) std::fputc((int)((hv >> (8 * i)) & 0xFF), fp);
  const bool ok = std::fclose(fp) == 0;
  if (!ok_count) return set_error(MOE_EINVAL, "checkpoint: synthetic record count mismatch");
  return ok ? MOE_OK : set_error(MOE_EIO, "checkpoint: write to '%s' failed", path);
}

}  // extern "C"
