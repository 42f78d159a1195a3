// ep_p2p_demo -- expert parallelism from a pure C++ host (no Python, no MPI):
// `world` processes (fork), one per GPU (or all on GPU 0 of a one-GPU box:
// the windows are shared through CUDA IPC either way), each holding E/world
// experts of the LM-style layer, exchange their peer-memory window handles
// through files, run the layer with the exchange over NVLink peer memory
// (moesim::gpu::ExpertParallelLayer -> moe_ep_*), and the parent checks every
// rank's output rows bit for bit against the single-GPU layer (same weights,
// same tokens).  Token residency is round robin: token t on rank t % world
// (proj/src/exchange.cpp:35-37); placement contiguous (balance.cpp:59-67).
//
//   ep_p2p_demo [--world 2] [--devices 1] [--tokens 2048] [--token-dim 1024]
//               [--hidden-dim 4096] [--experts 64] [--topk 2] [--steps 4]
//               [--dir /tmp/ep_demo] [--transport p2p|nccl]
// Exit 0 = bitwise equal on every rank and step.
#include <sys/wait.h>
#include <unistd.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <memory>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "moesim/gpu_layer.hpp"

namespace fs = std::filesystem;
using namespace moesim;

namespace {

struct Options {
  int world = 2, devices = 1, tokens = 2048, token_dim = 1024, hidden_dim = 4096, experts = 64,
      topk = 2, steps = 4;
  std::string dir = "/tmp/ep_p2p_demo";
  std::string transport = "p2p";  // or "nccl" (NCCL refuses two ranks on one GPU: world 1 there)
};

constexpr std::uint64_t kSeed = 2303061820ull;

Options parse(int argc, char** argv) {
  Options o;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) {
        std::cerr << "missing value for " << a << "\n";
        std::exit(2);
      }
      return argv[++i];
    };
    if (a == "--world") o.world = std::stoi(next());
    else if (a == "--devices") o.devices = std::stoi(next());
    else if (a == "--tokens") o.tokens = std::stoi(next());
    else if (a == "--token-dim") o.token_dim = std::stoi(next());
    else if (a == "--hidden-dim") o.hidden_dim = std::stoi(next());
    else if (a == "--experts") o.experts = std::stoi(next());
    else if (a == "--topk") o.topk = std::stoi(next());
    else if (a == "--steps") o.steps = std::stoi(next());
    else if (a == "--dir") o.dir = next();
    else if (a == "--transport") o.transport = next();
    else {
      std::cerr << "unknown option " << a << "\n";
      std::exit(2);
    }
  }
  return o;
}

// Weights and tokens with the counter generator (make_weights / make_tokens).
struct Model {
  gpu::DeviceBuffer wg, w1, w2, x;
  Model(gpu::Context& ctx, const Options& o) {
    const std::int64_t TD = o.token_dim, HD = o.hidden_dim, E = o.experts;
    wg = gpu::DeviceBuffer(ctx, E * TD * 2);
    w1 = gpu::DeviceBuffer(ctx, E * HD * TD * 2);
    w2 = gpu::DeviceBuffer(ctx, E * TD * HD * 2);
    x = gpu::DeviceBuffer(ctx, static_cast<std::size_t>(o.tokens) * TD * 2);
    const float r3 = std::sqrt(3.0f);
    gpu::fill_uniform_bf16(ctx, wg.get(), E * TD, kSeed, 2, r3 / std::sqrt((float)TD));
    gpu::fill_uniform_bf16(ctx, w1.get(), E * HD * TD, kSeed, 3, r3 * std::sqrt(2.0f / TD));
    gpu::fill_uniform_bf16(ctx, w2.get(), E * TD * HD, kSeed, 4, r3 / std::sqrt((float)HD));
    gpu::fill_uniform_bf16(ctx, x.get(), (std::int64_t)o.tokens * TD, kSeed, 1, r3);
  }
};

void write_file(const fs::path& p, const std::string& bytes) {
  const fs::path tmp = p.string() + ".tmp";
  {
    std::ofstream f(tmp, std::ios::binary);
    f.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
  }
  fs::rename(tmp, p);  // atomic: readers never see a partial file
}

std::string read_file(const fs::path& p) {
  std::ifstream f(p, std::ios::binary);
  std::ostringstream s;
  s << f.rdbuf();
  return s.str();
}

// File rendezvous: every rank writes <dir>/<tag><rank>, waits for all ranks.
std::vector<std::string> file_all_gather(const fs::path& dir, const std::string& tag, int rank,
                                         int world, const std::string& mine) {
  write_file(dir / (tag + std::to_string(rank)), mine);
  std::vector<std::string> all(world);
  for (int r = 0; r < world; ++r) {
    const fs::path p = dir / (tag + std::to_string(r));
    const auto t0 = std::chrono::steady_clock::now();
    while (!fs::exists(p)) {
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
        throw std::runtime_error("rendezvous timed out waiting for " + p.string());
      std::this_thread::sleep_for(std::chrono::milliseconds(2));
    }
    all[r] = read_file(p);
  }
  return all;
}

int run_rank(const Options& o, int rank) {
  gpu::Context ctx(rank % o.devices);
  Model m(ctx, o);
  const int D = o.world, E = o.experts, El = E / D, TD = o.token_dim, HD = o.hidden_dim;
  // this rank's tokens: t = i * D + rank
  const int S = (o.tokens - rank + D - 1) / D;
  std::vector<std::int32_t> rows(S);
  for (int i = 0; i < S; ++i) rows[i] = i * D + rank;
  gpu::DeviceBuffer rows_d(ctx, rows.size() * 4), xl(ctx, (std::size_t)S * TD * 2),
      out(ctx, (std::size_t)S * TD * 2);
  gpu::Stream stream(ctx);
  gpu::copy(ctx, rows_d.get(), rows.data(), rows.size() * 4, gpu::CopyKind::kHostToDevice);
  gpu::check(moe_gather_rows(ctx.get(), m.x.get(), static_cast<const std::int32_t*>(rows_d.get()), S,
                             1, TD, xl.get(), nullptr));
  gpu::check(moe_stream_synchronize(ctx.get(), nullptr));  // inputs ready before the EP stream
  std::vector<std::int32_t> device_of(E);
  for (int e = 0; e < E; ++e) device_of[e] = e / El;  // contiguous placement
  const char* w1 = static_cast<const char*>(m.w1.get()) + (std::size_t)rank * El * HD * TD * 2;
  const char* w2 = static_cast<const char*>(m.w2.get()) + (std::size_t)rank * El * TD * HD * 2;
  std::string bits;
  {
    std::unique_ptr<gpu::ExpertParallelLayer> ep_ptr;
    if (o.transport == "nccl") {
      gpu::ExpertParallelLayer::Nccl nccl{[&](const std::string& root_bytes) {
        return file_all_gather(o.dir, "ncclid", rank, D, root_bytes)[0];
      }};
      ep_ptr = std::make_unique<gpu::ExpertParallelLayer>(ctx, gpu::LayerShape{TD, HD, E, o.topk}, rank, D, S,
                                                          device_of, m.wg.get(), w1, w2, nccl);
    } else {
      ep_ptr = std::make_unique<gpu::ExpertParallelLayer>(
          ctx, gpu::LayerShape{TD, HD, E, o.topk}, rank, D, S, device_of, m.wg.get(), w1, w2,
          gpu::ExpertParallelLayer::AllGather([&](const std::string& mine) {
            return file_all_gather(o.dir, "handle", rank, D, mine);
          }));
    }
    gpu::ExpertParallelLayer& ep = *ep_ptr;
    const bool graph_ok = o.transport != "nccl";  // the NCCL transport syncs the host: eager
    for (int step = 0; step < o.steps; ++step) {
      if (step < o.steps / 2 || !graph_ok)
        ep.forward(xl.get(), S, out.get(), stream.get());
      else
        ep.forward_graph(xl.get(), S, out.get(), stream.get());
      ep.check_errors(stream.get());
      std::string host((std::size_t)S * TD * 2, '\0');
      gpu::copy(ctx, host.data(), out.get(), host.size(), gpu::CopyKind::kDeviceToHost);
      if (step == 0) bits = host;
      else if (host != bits) {
        std::cerr << "rank " << rank << ": step " << step << " differs from step 0\n";
        return 1;
      }
    }
    // no peer may still read this rank's window when it is freed
    file_all_gather(o.dir, "done", rank, D, "1");
  }
  write_file(fs::path(o.dir) / ("out" + std::to_string(rank)), bits);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  const Options o = parse(argc, argv);
  if (o.world < 1 || o.world > MOE_EP_MAX_RANKS || o.experts % o.world) {
    std::cerr << "world must be in [1, " << MOE_EP_MAX_RANKS << "] and divide the experts\n";
    return 2;
  }
  fs::remove_all(o.dir);
  fs::create_directories(o.dir);
  // fork before any CUDA call: each child initialises its own context
  std::vector<pid_t> kids;
  for (int r = 0; r < o.world; ++r) {
    const pid_t pid = fork();
    if (pid == 0) {
      int rc = 1;
      try {
        rc = run_rank(o, r);
      } catch (const std::exception& e) {
        std::cerr << "rank " << r << ": " << e.what() << "\n";
      }
      std::_Exit(rc);
    }
    kids.push_back(pid);
  }
  bool ok = true;
  for (pid_t pid : kids) {
    int st = 0;
    waitpid(pid, &st, 0);
    ok = ok && WIFEXITED(st) && WEXITSTATUS(st) == 0;
  }
  if (!ok) {
    std::cerr << "ep_p2p_demo: a rank failed\n";
    return 1;
  }
  // single-GPU reference: the whole layer on one device, same weights/tokens
  gpu::Context ctx(0);
  Model m(ctx, o);
  const int TD = o.token_dim;
  gpu::MoeLayer layer(ctx, {TD, o.hidden_dim, o.experts, o.topk}, o.tokens,
                      GatingConfig{o.experts, o.topk, 0.0, GatingMode::kDynamic}, m.wg.get(),
                      m.w1.get(), m.w2.get());
  gpu::DeviceBuffer out(ctx, (std::size_t)o.tokens * TD * 2);
  layer.forward(m.x.get(), o.tokens, out.get());
  layer.check_errors();
  std::string ref((std::size_t)o.tokens * TD * 2, '\0');
  gpu::copy(ctx, ref.data(), out.get(), ref.size(), gpu::CopyKind::kDeviceToHost);
  const std::size_t row = (std::size_t)TD * 2;
  long mismatched = 0;
  for (int r = 0; r < o.world; ++r) {
    const std::string got = read_file(fs::path(o.dir) / ("out" + std::to_string(r)));
    const int S = (o.tokens - r + o.world - 1) / o.world;
    if (got.size() != (std::size_t)S * row) {
      std::cerr << "rank " << r << ": wrong output size\n";
      return 1;
    }
    for (int i = 0; i < S; ++i)
      if (std::memcmp(got.data() + i * row, ref.data() + (std::size_t)(i * o.world + r) * row, row))
        ++mismatched;
  }
  std::printf("ep_p2p_demo: world=%d tokens=%d E=%d k=%d TD=%d HD=%d steps=%d: %ld rows differ\n",
              o.world, o.tokens, o.experts, o.topk, TD, o.hidden_dim, o.steps, mismatched);
  return mismatched == 0 ? 0 : 1;
}
