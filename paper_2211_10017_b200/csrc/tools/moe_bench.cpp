// moe_bench -- the reference CLI's `moe bench` (proj/tools/moe_cli.cpp:
// BenchOpts :200-214, cmd_bench :291-394, report schema :54-135) for the
// MoE blocks of a `.moec` checkpoint on the GPU.
//
// One JSONL line per (batch, beam, prune) cell in the reference's
// `moe-bench-v1` schema -- exactly its 21 fields, validated the way
// validate_report_line does before anything is written.  The workload is
// the MoE side of beam-search decoding (moe_decode_run): for
// every decode step, every decoder MoE block (dec.i.ffn) runs one layer
// forward over the batch x beam rows, with the finished rows routed out when
// prune is on (proj/src/decode.cpp:167-169, 216).  What differs from the
// reference, by construction of the hot-path scope:
//   * attention, embeddings and the search are not run: the per-step
//     decoder hidden states are synthetic (seeded normal) and every row's
//     EOS step is seeded uniform in [max_len/4, max_len);
//   * wall_ms is the GPU time of the decode's MoE blocks (CUDA events around
//     one moe_decode_run after a warm-up run), input_tokens_per_second
//     = batch * src_len / wall_ms;
//   * expert_* / other_* are the reference's analytic counters
//     (grouped_gemm.cpp:155-160, 201-211; model.cpp:303-347) summed over
//     every MoE-block forward of the decode (moe_layer_traffic); other_*
//     therefore covers the MoE blocks' LN / gate traffic only;
//   * steps = decode steps until every row finished (<= max_len);
//     generated_tokens = sum over rows of the tokens before EOS + EOS, one
//     hypothesis per sentence (beam rows share their sentence's EOS step).
// The cell seed is the reference's cell_seed (prune not mixed in, so
// --prune both feeds the identical workload to both variants).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "moe_cuda.h"

namespace {

constexpr const char* kSchema = "moe-bench-v1";

struct Opts {
  std::string config, precision = "fp16", prune = "on", out;
  std::vector<uint32_t> batch, beam;
  uint64_t seed = 1;
  uint32_t src_len = 40, max_len = 32;
  int threads = 1;
};

[[noreturn]] void die(const char* what, const char* detail = "") {
  std::fprintf(stderr, "error: %s%s\n", what, detail);
  std::exit(2);
}

void check(int st, const char* what) {
  if (st != MOE_OK) {
    std::fprintf(stderr, "error: %s: %s\n", what, moe_cuda_last_error());
    std::exit(1);
  }
}

uint64_t cell_seed(uint64_t base, uint64_t batch, uint64_t beam) {
  uint64_t h = base + 0x9e3779b97f4a7c15ull;
  for (const uint64_t v : {batch, beam}) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    h *= 0xff51afd7ed558ccdull;
    h ^= h >> 33;
  }
  return h >> 11;  // 53 bits: exact in JSON doubles
}

uint16_t f2h(float f) {  // RN, finite inputs
  uint32_t x;
  std::memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  const int exp = (int)((x >> 23) & 0xFF) - 127 + 15;
  uint32_t man = x & 0x7FFFFFu;
  if (exp >= 31) return (uint16_t)(sign | 0x7C00u);
  if (exp <= 0) {
    if (exp < -10) return (uint16_t)sign;
    man |= 0x800000u;
    const int shift = 14 - exp;
    uint32_t h = man >> shift;
    const uint32_t rem = man & ((1u << shift) - 1), half = 1u << (shift - 1);
    if (rem > half || (rem == half && (h & 1u))) ++h;
    return (uint16_t)(sign | h);
  }
  uint32_t h = ((uint32_t)exp << 10) | (man >> 13);
  const uint32_t rem = man & 0x1FFFu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;
  return (uint16_t)(sign | h);
}

struct Field {
  const char* key;
  char type;  // s string, i integer >= 0, b bool, f float >= 0, o object
  std::string value;
};

// validate_report_line (moe_cli.cpp:76-135): every documented field, in
// order, with its type; config echo with the nine config keys
void validate(const std::vector<Field>& f) {
  static const char* keys[] = {"schema", "config", "precision", "batch", "beam", "prune", "seed",
                               "src_len", "max_len", "threads", "steps", "input_tokens",
                               "generated_tokens", "expert_weight_bytes", "expert_activation_bytes",
                               "expert_bytes_written", "other_weight_bytes", "other_activation_bytes",
                               "other_bytes_written", "wall_ms", "input_tokens_per_second"};
  static const char types[] = "sosiibiiiiiiiiiiiiiff";
  if (f.size() != sizeof(keys) / sizeof(keys[0])) die("report line has wrong field count");
  for (size_t i = 0; i < f.size(); ++i) {
    if (std::strcmp(f[i].key, keys[i]) != 0) die("report line field order: ", f[i].key);
    if (f[i].type != types[i]) die("report field has wrong type: ", f[i].key);
    if ((f[i].type == 'i' || f[i].type == 'f') && !f[i].value.empty() && f[i].value[0] == '-')
      die("report field is negative: ", f[i].key);
  }
  if (f[0].value != std::string("\"") + kSchema + "\"") die("report schema tag mismatch");
}

std::string dump(const std::vector<Field>& f) {
  std::string s = "{";
  for (size_t i = 0; i < f.size(); ++i) {
    if (i) s += ", ";
    s += "\"" + std::string(f[i].key) + "\": " + f[i].value;
  }
  return s + "}";
}

std::vector<uint32_t> parse_list(int& i, int argc, char** argv) {
  std::vector<uint32_t> v;
  while (i + 1 < argc && argv[i + 1][0] != '-') v.push_back((uint32_t)std::strtoul(argv[++i], nullptr, 10));
  if (v.empty()) die("expected at least one value after ", argv[i]);
  return v;
}

void usage() {
  std::printf(
      "usage: moe_bench --config PATH.moec [--precision fp16|int8|int4] [--batch N ...]\n"
      "                 [--beam N ...] [--prune on|off|both] [--seed S] [--src-len L]\n"
      "                 [--max-len M] [--threads T] [--out REPORT.jsonl]\n"
      "MoE blocks of the checkpoint's decoder, beam-search decode shape, on cuda:0;\n"
      "one moe-bench-v1 JSONL line per (batch, beam, prune) cell.\n");
}

}  // namespace

int main(int argc, char** argv) {
  Opts o;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    auto val = [&]() -> const char* {
      if (i + 1 >= argc) die("missing value after ", argv[i]);
      return argv[++i];
    };
    if (a == "-h" || a == "--help") {
      usage();
      return 0;
    } else if (a == "--config") o.config = val();
    else if (a == "--precision") o.precision = val();
    else if (a == "--batch") o.batch = parse_list(i, argc, argv);
    else if (a == "--beam") o.beam = parse_list(i, argc, argv);
    else if (a == "--prune") o.prune = val();
    else if (a == "--seed") o.seed = std::strtoull(val(), nullptr, 10);
    else if (a == "--src-len") o.src_len = (uint32_t)std::strtoul(val(), nullptr, 10);
    else if (a == "--max-len") o.max_len = (uint32_t)std::strtoul(val(), nullptr, 10);
    else if (a == "--threads") o.threads = std::atoi(val());
    else if (a == "--out") o.out = val();
    else die("unknown option ", a.c_str());
  }
  if (o.config.empty()) {
    usage();
    die("--config is required");
  }
  if (o.batch.empty()) o.batch = {8};
  if (o.beam.empty()) o.beam = {1};
  std::vector<int> prunes;
  if (o.prune == "on") prunes = {1};
  else if (o.prune == "off") prunes = {0};
  else if (o.prune == "both") prunes = {0, 1};
  else die("--prune must be on, off or both");
  if (o.max_len < 2) die("--max-len out of range");

  moe_moec* M = nullptr;
  check(moe_moec_load(o.config.c_str(), 1, &M), "load");
  uint32_t cfg[9];
  int prec = 0, nblk = 0;
  check(moe_moec_info(M, cfg, &prec, &nblk), "info");
  static const char* pname[] = {"fp16", "int8", "int4"};
  if (o.precision != pname[prec]) {
    std::fprintf(stderr, "error: checkpoint %s holds %s weights but --precision says %s\n",
                 o.config.c_str(), pname[prec], o.precision.c_str());
    return 2;
  }
  if (o.src_len == 0 || o.src_len > cfg[8]) die("--src-len out of range");
  const int64_t d = cfg[0];
  std::vector<moe_layer*> dec;  // decoder MoE blocks, in stack order
  for (int i = 0; i < nblk; ++i) {
    moe_layer* L = nullptr;
    char name[64];
    check(moe_moec_block(M, i, &L, name, sizeof name), "block");
    if (std::strncmp(name, "dec.", 4) == 0) dec.push_back(L);
  }
  if (dec.empty()) die("checkpoint has no decoder MoE block");
  const char* cfg_keys[] = {"d_model", "d_ffn", "n_enc_layers", "n_dec_layers", "n_experts",
                            "n_heads", "vocab_size", "moe_every", "max_seq_len"};
  std::string cfg_json = "{";
  for (int i = 0; i < 9; ++i)
    cfg_json += std::string(i ? ", " : "") + "\"" + cfg_keys[i] + "\": " + std::to_string(cfg[i]);
  cfg_json += "}";

  std::vector<std::string> lines;
  std::printf("%-5s %6s %5s %6s %6s %8s %9s %14s %14s %10s %9s\n", "prec", "batch", "beam", "prune",
              "steps", "in_tok", "gen_tok", "exp_wt_bytes", "exp_act_bytes", "tok/s", "wall_ms");
  cudaStream_t st;
  cudaStreamCreate(&st);
  for (const uint32_t batch : o.batch)
    for (const uint32_t beam : o.beam)
      for (const int prune : prunes) {
        const uint64_t seed = cell_seed(o.seed, batch, beam);
        const int64_t rows = (int64_t)batch * beam;
        std::mt19937_64 rng(seed);
        std::vector<uint32_t> eos(batch);  // per sentence, shared by its beam rows
        uint32_t steps = 0;
        for (auto& e : eos) {
          e = o.max_len / 4 + (uint32_t)(rng() % (o.max_len - o.max_len / 4));
          steps = std::max(steps, e + 1);
        }
        steps = std::min(steps, o.max_len);
        std::vector<uint16_t> x((size_t)steps * rows * d);
        for (auto& v : x) {  // Box-Muller normals
          const double u1 = 1.0 - (double)(rng() >> 11) * 0x1.0p-53, u2 = (double)(rng() >> 11) * 0x1.0p-53;
          v = f2h((float)(std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2)));
        }
        std::vector<uint8_t> fin((size_t)steps * rows);
        uint64_t generated = 0;
        for (uint32_t b = 0; b < batch; ++b) generated += std::min(eos[b] + 1, steps);
        for (uint32_t s = 0; s < steps; ++s)
          for (int64_t r = 0; r < rows; ++r) fin[(size_t)s * rows + r] = s > eos[r / beam] ? 1 : 0;
        uint16_t *dx = nullptr, *dout = nullptr, *dwork = nullptr;
        uint8_t* dfin = nullptr;
        cudaMalloc(&dx, x.size() * 2);
        cudaMalloc(&dout, x.size() * 2);
        cudaMalloc(&dwork, (size_t)rows * d * 2);
        cudaMalloc(&dfin, fin.size());
        cudaMemcpy(dx, x.data(), x.size() * 2, cudaMemcpyHostToDevice);
        cudaMemcpy(dfin, fin.data(), fin.size(), cudaMemcpyHostToDevice);
        // analytic counters: every MoE-block forward of the decode, in order
        uint64_t cnt[6] = {0, 0, 0, 0, 0, 0};
        for (uint32_t s = 0; s < steps; ++s) {
          const uint16_t* in = dx + (size_t)s * rows * d;
          for (size_t l = 0; l < dec.size(); ++l) {
            uint16_t* dst = (l & 1) ? dwork : dout;
            check(moe_layer_forward(dec[l], in, prune ? dfin + (size_t)s * rows : nullptr, rows, 1,
                                    MOE_MODE_FAST, dst, st),
                  "forward");
            uint64_t t6[6];
            check(moe_layer_traffic(dec[l], t6, st), "traffic");
            for (int q = 0; q < 6; ++q) cnt[q] += t6[q];
            in = dst;
          }
        }
        // timing: one warm-up decode, then one timed decode (CUDA events)
        auto run = [&]() {
          check(moe_decode_run(dec.data(), (int)dec.size(), dx, dfin, (int)steps, rows, 1,
                               MOE_MODE_FAST, prune, dout, dwork, st),
                "decode");
        };
        run();
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        run();
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        check(cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ECUDA, "cuda");
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFree(dx);
        cudaFree(dout);
        cudaFree(dwork);
        cudaFree(dfin);
        const uint64_t in_tok = (uint64_t)batch * o.src_len;
        const double tps = ms > 0.f ? 1000.0 * (double)in_tok / ms : 0.0;
        char fbuf[64], tbuf[64];
        std::snprintf(fbuf, sizeof fbuf, "%.6f", (double)ms);
        std::snprintf(tbuf, sizeof tbuf, "%.3f", tps);
        std::vector<Field> f = {
            {"schema", 's', std::string("\"") + kSchema + "\""},
            {"config", 'o', cfg_json},
            {"precision", 's', "\"" + o.precision + "\""},
            {"batch", 'i', std::to_string(batch)},
            {"beam", 'i', std::to_string(beam)},
            {"prune", 'b', prune ? "true" : "false"},
            {"seed", 'i', std::to_string(seed)},
            {"src_len", 'i', std::to_string(o.src_len)},
            {"max_len", 'i', std::to_string(o.max_len)},
            {"threads", 'i', std::to_string(o.threads)},
            {"steps", 'i', std::to_string(steps)},
            {"input_tokens", 'i', std::to_string(in_tok)},
            {"generated_tokens", 'i', std::to_string(generated)},
            {"expert_weight_bytes", 'i', std::to_string(cnt[0])},
            {"expert_activation_bytes", 'i', std::to_string(cnt[1])},
            {"expert_bytes_written", 'i', std::to_string(cnt[2])},
            {"other_weight_bytes", 'i', std::to_string(cnt[3])},
            {"other_activation_bytes", 'i', std::to_string(cnt[4])},
            {"other_bytes_written", 'i', std::to_string(cnt[5])},
            {"wall_ms", 'f', fbuf},
            {"input_tokens_per_second", 'f', tbuf},
        };
        validate(f);
        lines.push_back(dump(f));
        std::printf("%-5s %6u %5u %6s %6u %8llu %9llu %14llu %14llu %10.0f %9.3f\n", o.precision.c_str(),
                    batch, beam, prune ? "on" : "off", steps, (unsigned long long)in_tok,
                    (unsigned long long)generated, (unsigned long long)cnt[0],
                    (unsigned long long)cnt[1], tps, (double)ms);
      }
  cudaStreamDestroy(st);
  if (!o.out.empty()) {
    FILE* fp = std::fopen(o.out.c_str(), "w");
    if (!fp) die("cannot write ", o.out.c_str());
    for (const auto& l : lines) std::fprintf(fp, "%s\n", l.c_str());
    std::fclose(fp);
  }
  moe_moec_destroy(M);
  return 0;
}
