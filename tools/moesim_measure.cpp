// moesim_measure -- the reference CLI's `simulate` report (latency.csv,
// memory.csv, comm.csv, cache.csv, summary.csv, manifest.json; schemas of
// proj/tools/moesim.cpp:342-423) filled with MEASURED B200 numbers instead of
// the analytic cost model.
//
// A synthetic trace (moesim::gen_synthetic_trace, bit-identical to the
// reference generator) or the layer's own gate drives the GPU MoE layer
// through the C++ host API (include/moesim/gpu_layer.hpp); every batch is
// timed per stage with CUDA events inside the library.  Single GPU: the
// all-to-all components are zero.
//
//   moesim_measure --experts 128 --topk 2 --tokens 6144 --batches 8
//       --token-dim 2048 --hidden-dim 8192 --mode both --capacity-factor 1
//       --zipf 1.2 --persist 0.9 --active-frac 0.75 --cache-size 0 --out out/
//   --gate        route with the layer's gate instead of the trace
//   --trace F     replay the routing of a JSON Lines trace file (reference
//                 format, load_token_trace); E, k and the batches come from it
//   --save-trace F  write the routing trace used (generated or loaded)
//   --verify N    check N tokens of the first batch (dynamic mode) against an
//                 fp32 host reference
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "moesim/gating.hpp"
#include "moesim/gpu_layer.hpp"
#include "moesim/trace.hpp"

namespace fs = std::filesystem;
using namespace moesim;

namespace {

struct Options {
  int experts = 16, topk = 2, tokens = 512, batches = 4, token_dim = 256, hidden_dim = 512;
  std::string mode = "both";
  double capacity_factor = 1.0, zipf = 1.2, persist = 0.9, active_frac = 0.75;
  int cache_size = 0;
  std::uint64_t seed = 7;
  std::string out = "measure_out";
  bool gate = false;
  int verify = 0;
  std::string trace, save_trace;
};

[[noreturn]] void usage(const std::string& msg) {
  std::cerr << "moesim_measure: " << msg << "\n";
  std::exit(2);
}

Options parse(int argc, char** argv) {
  Options o;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) usage("missing value for " + a);
      return argv[++i];
    };
    if (a == "--experts") o.experts = std::stoi(val());
    else if (a == "--topk") o.topk = std::stoi(val());
    else if (a == "--tokens") o.tokens = std::stoi(val());
    else if (a == "--batches") o.batches = std::stoi(val());
    else if (a == "--token-dim") o.token_dim = std::stoi(val());
    else if (a == "--hidden-dim") o.hidden_dim = std::stoi(val());
    else if (a == "--mode") o.mode = val();
    else if (a == "--capacity-factor") o.capacity_factor = std::stod(val());
    else if (a == "--zipf") o.zipf = std::stod(val());
    else if (a == "--persist") o.persist = std::stod(val());
    else if (a == "--active-frac") o.active_frac = std::stod(val());
    else if (a == "--cache-size") o.cache_size = std::stoi(val());
    else if (a == "--seed") o.seed = std::stoull(val());
    else if (a == "--out") o.out = val();
    else if (a == "--gate") o.gate = true;
    else if (a == "--verify") o.verify = std::stoi(val());
    else if (a == "--trace") o.trace = val();
    else if (a == "--save-trace") o.save_trace = val();
    else usage("unknown option " + a);
  }
  if (o.mode != "static" && o.mode != "dynamic" && o.mode != "both")
    usage("--mode expects static, dynamic or both");
  return o;
}

// %.12g, the reference's CSV number format (proj/src/csv.cpp:8-12)
std::string num(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%.12g", v);
  return b;
}

struct Csv {
  std::ofstream f;
  explicit Csv(const fs::path& p) : f(p, std::ios::binary) {
    if (!f) throw std::runtime_error("cannot write " + p.string());
  }
  template <class... T>
  void row(const T&... cols) {
    bool first = true;
    ((f << (first ? "" : ",") << cell(cols), first = false), ...);
    f << '\n';
  }
  static std::string cell(const std::string& s) { return s; }
  static std::string cell(const char* s) { return s; }
  static std::string cell(double v) { return num(v); }
  static std::string cell(std::int64_t v) { return std::to_string(v); }
  static std::string cell(int v) { return std::to_string(v); }
};

float bf16_to_float(std::uint16_t h) {
  std::uint32_t u = static_cast<std::uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

struct ModeResult {
  double gate = 0, reorder = 0, compute = 0, transfer = 0, total = 0;
  double static_bytes = 0, dynamic_bytes = 0;
};

}  // namespace

int main(int argc, char** argv) {
  Options o = parse(argc, argv);
  try {
    // a replayed trace fixes E, k, the batch count and the tokens per batch
    TokenTrace trace;
    std::vector<int> seq;
    if (!o.trace.empty()) {
      if (o.gate) usage("--trace and --gate are exclusive");
      trace = load_token_trace(o.trace);
      o.experts = trace.num_experts;
      o.topk = trace.top_k;
      o.batches = trace.num_batches();
      o.tokens = 0;
      for (const Batch& b : trace.batches) o.tokens = std::max(o.tokens, b.seq_len());
    }
    const fs::path out_dir(o.out);
    fs::create_directories(out_dir);
    gpu::Context ctx(0);
    gpu::Stream stream(ctx);
    const int S = o.tokens, k = o.topk, E = o.experts, TD = o.token_dim, HD = o.hidden_dim;
    const std::size_t wbytes = static_cast<std::size_t>(E) * HD * TD * 2;

    // weights and tokens (counter-based synthetic, on the device)
    gpu::DeviceBuffer Wg(ctx, static_cast<std::size_t>(E) * TD * 2), W1(ctx, wbytes), W2(ctx, wbytes);
    gpu::DeviceBuffer X(ctx, static_cast<std::size_t>(S) * TD * 2), Y(ctx, static_cast<std::size_t>(S) * TD * 2);
    const float r3 = std::sqrt(3.0f);
    gpu::fill_uniform_bf16(ctx, Wg.get(), static_cast<std::int64_t>(E) * TD, o.seed, 2, r3 / std::sqrt(float(TD)));
    gpu::fill_uniform_bf16(ctx, W1.get(), static_cast<std::int64_t>(wbytes / 2), o.seed, 3,
                           r3 * std::sqrt(2.0f / TD));
    gpu::fill_uniform_bf16(ctx, W2.get(), static_cast<std::int64_t>(wbytes / 2), o.seed, 4,
                           r3 / std::sqrt(float(HD)));
    gpu::fill_uniform_bf16(ctx, X.get(), static_cast<std::int64_t>(S) * TD, o.seed, 1, r3);

    // routing trace (reference generator or file) -> device idx / w per batch
    if (!o.gate && o.trace.empty()) {
      SyntheticSpec spec;
      spec.num_experts = E;
      spec.top_k = k;
      spec.num_batches = o.batches;
      spec.seq_len = S;
      spec.zipf_skew = o.zipf;
      spec.persistence = o.persist;
      spec.active_fraction = o.active_frac;
      spec.seed = o.seed;
      trace = gen_synthetic_trace(spec);
    }
    for (int b = 0; b < o.batches; ++b)
      seq.push_back(o.gate ? S : trace.batches[static_cast<std::size_t>(b)].seq_len());
    if (!o.save_trace.empty() && !o.gate) save_token_trace(trace, o.save_trace);
    gpu::DeviceBuffer idx(ctx, static_cast<std::size_t>(o.batches) * S * k * 4);
    gpu::DeviceBuffer wts(ctx, static_cast<std::size_t>(o.batches) * S * k * 4);
    if (!o.gate) {
      std::vector<std::int32_t> hi(static_cast<std::size_t>(o.batches) * S * k);
      std::vector<float> hw(hi.size());
      for (std::size_t b = 0; b < trace.batches.size(); ++b) {
        std::size_t i = b * static_cast<std::size_t>(S) * k;  // batch b at a fixed stride
        for (const TokenAssignment& ta : trace.batches[b].tokens)
          for (int j = 0; j < k; ++j, ++i) {
            hi[i] = ta.experts[static_cast<std::size_t>(j)];
            hw[i] = static_cast<float>(ta.weights[static_cast<std::size_t>(j)]);
          }
      }
      gpu::copy(ctx, idx.get(), hi.data(), hi.size() * 4, gpu::CopyKind::kHostToDevice);
      gpu::copy(ctx, wts.get(), hw.data(), hw.size() * 4, gpu::CopyKind::kHostToDevice);
    }
    auto batch_idx = [&](int b) {
      return static_cast<const std::int32_t*>(idx.get()) + static_cast<std::size_t>(b) * S * k;
    };
    auto batch_w = [&](int b) {
      return static_cast<const float*>(wts.get()) + static_cast<std::size_t>(b) * S * k;
    };

    std::vector<std::string> modes;
    if (o.mode != "dynamic") modes.push_back("static");
    if (o.mode != "static") modes.push_back("dynamic");
    std::map<std::string, ModeResult> res;
    std::map<std::string, std::vector<int>> cache_rows;  // accesses, hits, misses per batch
    double verify_err = -1.0;

    for (const std::string& mode : modes) {
      GatingConfig gc{E, k, o.capacity_factor,
                      mode == "static" ? GatingMode::kStatic : GatingMode::kDynamic};
      gpu::MoeLayer layer(ctx, {TD, HD, E, k}, S, gc, Wg.get(), W1.get(), W2.get());
      ModeResult r;
      layer.enable_timing(o.batches);
      auto run = [&](int b) {
        if (o.gate) layer.forward(X.get(), S, Y.get(), stream.get());
        else layer.forward_routed(X.get(), batch_idx(b), batch_w(b), seq[static_cast<std::size_t>(b)], Y.get(),
                                  stream.get());
      };
      run(0);  // warm-up
      stream.synchronize();
      layer.enable_timing(o.batches);
      for (int b = 0; b < o.batches; ++b) run(b);
      stream.synchronize();
      layer.check_errors(stream.get());
      for (int b = 0; b < o.batches; ++b) {
        const gpu::StageTimes t = layer.stage_times(b);
        r.gate += t.gate * 1e-3;
        r.reorder += (t.route + t.gather) * 1e-3;
        r.compute += (t.ffn1 + t.ffn2 + t.combine) * 1e-3;
        r.total += t.total() * 1e-3;
      }
      const moe_layer_view v = layer.view();
      const double rows = v.rows;
      r.static_bytes = 2.0 * static_cast<double>(wbytes) + static_cast<double>(E) * TD * 2;
      r.dynamic_bytes = rows * (2.0 * TD + HD) * 2 + static_cast<double>(S) * k * 16;

      if (o.verify > 0 && mode == "dynamic") {
        // fp32 host reference for the first tokens of the last batch run,
        // with the routing the GPU used
        run(0);
        stream.synchronize();
        const moe_layer_view vv = layer.view();
        const int n = std::min(o.verify, seq[0]);
        std::vector<std::int32_t> hidx(static_cast<std::size_t>(n) * k);
        std::vector<float> hw(hidx.size());
        gpu::copy(ctx, hidx.data(), o.gate ? vv.idx : batch_idx(0), hidx.size() * 4,
                  gpu::CopyKind::kDeviceToHost);
        gpu::copy(ctx, hw.data(), o.gate ? vv.w : batch_w(0), hw.size() * 4,
                  gpu::CopyKind::kDeviceToHost);
        std::vector<std::uint16_t> hx(static_cast<std::size_t>(n) * TD), hy(hx.size());
        gpu::copy(ctx, hx.data(), X.get(), hx.size() * 2, gpu::CopyKind::kDeviceToHost);
        gpu::copy(ctx, hy.data(), Y.get(), hy.size() * 2, gpu::CopyKind::kDeviceToHost);
        std::vector<std::uint16_t> w1(static_cast<std::size_t>(HD) * TD), w2(w1.size());
        double num2 = 0, den2 = 0;
        std::vector<double> ref(static_cast<std::size_t>(n) * TD, 0.0);
        for (int t = 0; t < n; ++t)
          for (int j = 0; j < k; ++j) {
            const int e = hidx[static_cast<std::size_t>(t) * k + j];
            gpu::copy(ctx, w1.data(), static_cast<const char*>(W1.get()) + static_cast<std::size_t>(e) * HD * TD * 2,
                      w1.size() * 2, gpu::CopyKind::kDeviceToHost);
            gpu::copy(ctx, w2.data(), static_cast<const char*>(W2.get()) + static_cast<std::size_t>(e) * HD * TD * 2,
                      w2.size() * 2, gpu::CopyKind::kDeviceToHost);
            std::vector<double> h(static_cast<std::size_t>(HD));
            for (int o2 = 0; o2 < HD; ++o2) {
              double acc = 0;
              for (int i = 0; i < TD; ++i)
                acc += double(bf16_to_float(hx[static_cast<std::size_t>(t) * TD + i])) *
                       bf16_to_float(w1[static_cast<std::size_t>(o2) * TD + i]);
              h[static_cast<std::size_t>(o2)] = std::max(acc, 0.0);
            }
            for (int o2 = 0; o2 < TD; ++o2) {
              double acc = 0;
              for (int i = 0; i < HD; ++i)
                acc += h[static_cast<std::size_t>(i)] * bf16_to_float(w2[static_cast<std::size_t>(o2) * HD + i]);
              ref[static_cast<std::size_t>(t) * TD + o2] += hw[static_cast<std::size_t>(t) * k + j] * acc;
            }
          }
        for (std::size_t i = 0; i < ref.size(); ++i) {
          const double d = bf16_to_float(hy[i]) - ref[i];
          num2 += d * d;
          den2 += ref[i] * ref[i];
        }
        verify_err = std::sqrt(num2 / std::max(den2, 1e-300));
      }

      if (mode == "dynamic" && o.cache_size > 0) {
        // expert buffering: all experts in pinned host memory, cache_size on the GPU
        gpu::DeviceBuffer h1(ctx, wbytes, true), h2(ctx, wbytes, true);
        gpu::copy(ctx, h1.get(), W1.get(), wbytes, gpu::CopyKind::kDeviceToHost);
        gpu::copy(ctx, h2.get(), W2.get(), wbytes, gpu::CopyKind::kDeviceToHost);
        gpu::MoeLayer clayer(ctx, {TD, HD, E, k}, S, gc, Wg.get(), W1.get(), W2.get());
        gpu::ExpertCache cache(clayer, h1.get(), h2.get(), o.cache_size);
        double cached_total = 0;
        for (int b = 0; b < o.batches; ++b) {
          const auto t0 = std::chrono::steady_clock::now();
          if (o.gate) cache.forward(X.get(), S, Y.get(), stream.get());
          else cache.forward_routed(X.get(), batch_idx(b), batch_w(b), seq[static_cast<std::size_t>(b)], Y.get(),
                                    stream.get());
          stream.synchronize();
          cached_total += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
          const auto st = cache.stats();
          cache_rows[mode].insert(cache_rows[mode].end(), {st.last_accesses, st.last_hits, st.last_misses});
        }
        r.transfer = std::max(0.0, cached_total - r.total);
        r.total = cached_total;
        r.static_bytes = static_cast<double>(o.cache_size) * 2.0 * HD * TD * 2 + static_cast<double>(E) * TD * 2;
      }
      res[mode] = r;
    }

    std::vector<std::string> outputs;
    {
      Csv csv(out_dir / "latency.csv");
      csv.row("component", "seconds");
      for (const auto& [mode, r] : res) {
        csv.row(mode + ".gate", r.gate);
        csv.row(mode + ".reorder", r.reorder);
        csv.row(mode + ".a2a_size", 0.0);
        csv.row(mode + ".a2a_payload", 0.0);
        csv.row(mode + ".expert_compute", r.compute);
        csv.row(mode + ".cpu_gpu_transfer", r.transfer);
        csv.row(mode + ".total", r.total);
      }
      outputs.push_back("latency.csv");
    }
    {
      Csv csv(out_dir / "memory.csv");
      csv.row("component", "bytes");
      for (const auto& [mode, r] : res) {
        csv.row(mode + ".static", r.static_bytes);
        csv.row(mode + ".dynamic", r.dynamic_bytes);
        csv.row(mode + ".peak", r.static_bytes + r.dynamic_bytes);
      }
      outputs.push_back("memory.csv");
    }
    {
      Csv csv(out_dir / "comm.csv");
      csv.row("phase", "src", "dst", "bytes");
      for (const auto& [mode, r] : res) csv.row(mode + ".payload", 0, 0, static_cast<std::int64_t>(0));
      outputs.push_back("comm.csv");
    }
    if (!cache_rows.empty()) {
      Csv csv(out_dir / "cache.csv");
      csv.row("device", "accesses", "hits", "misses", "miss_rate", "worst_batch_miss_rate",
              "transfer_seconds");
      const auto& v = cache_rows["dynamic"];
      std::int64_t acc = 0, hit = 0, mis = 0;
      double worst = 0;
      for (std::size_t i = 0; i + 2 < v.size(); i += 3) {
        acc += v[i];
        hit += v[i + 1];
        mis += v[i + 2];
        if (v[i] > 0) worst = std::max(worst, double(v[i + 2]) / v[i]);
      }
      const double rate = acc > 0 ? double(mis) / acc : 0.0;
      csv.row(std::string("0"), acc, hit, mis, rate, worst, res["dynamic"].transfer);
      csv.row(std::string("global"), acc, hit, mis, rate, worst, res["dynamic"].transfer);
      outputs.push_back("cache.csv");
    }
    std::int64_t total_tokens = 0;
    for (int n : seq) total_tokens += n;
    {
      Csv csv(out_dir / "summary.csv");
      csv.row("metric", "value");
      csv.row("waste_factor", waste_factor(E, o.capacity_factor, k).value);
      csv.row("capacity", static_cast<std::int64_t>(expert_capacity(o.capacity_factor, S)));
      csv.row("num_batches", static_cast<std::int64_t>(o.batches));
      csv.row("total_tokens", total_tokens);
      for (const auto& [mode, r] : res) {
        csv.row("total_latency_" + mode, r.total);
        csv.row("throughput_" + mode, total_tokens / r.total);
        csv.row("payload_bytes_" + mode, static_cast<std::int64_t>(0));
        csv.row("peak_memory_" + mode, r.static_bytes + r.dynamic_bytes);
      }
      if (verify_err >= 0) csv.row("verify_rel_fro", verify_err);
      outputs.push_back("summary.csv");
    }
    {
      std::ofstream m(out_dir / "manifest.json", std::ios::binary);
      m << "{\n  \"artifact\": \"moesim-b200\",\n  \"version\": \"0.1.0\",\n  \"command\": \"measure\",\n"
        << "  \"seed\": " << o.seed << ",\n  \"config\": {\"experts\": " << E << ", \"topk\": " << k
        << ", \"tokens\": " << S << ", \"batches\": " << o.batches << ", \"token_dim\": " << TD
        << ", \"hidden_dim\": " << HD << ", \"mode\": \"" << o.mode << "\", \"capacity_factor\": "
        << num(o.capacity_factor) << ", \"zipf\": " << num(o.zipf) << ", \"persist\": " << num(o.persist)
        << ", \"active_frac\": " << num(o.active_frac) << ", \"cache_size\": " << o.cache_size
        << ", \"routing\": \"" << (o.gate ? "gate" : o.trace.empty() ? "synthetic" : "file:" + o.trace) << "\"},\n  \"outputs\": [";
      for (std::size_t i = 0; i < outputs.size(); ++i) m << (i ? ", " : "") << '"' << outputs[i] << '"';
      m << "]\n}\n";
    }
    for (const auto& [mode, r] : res)
      std::printf("%s: %.3f ms/batch, %.1f tokens/s\n", mode.c_str(), 1e3 * r.total / o.batches,
                  total_tokens / r.total);
    if (verify_err >= 0) std::printf("verify rel_fro %.3e\n", verify_err);
    return 0;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
