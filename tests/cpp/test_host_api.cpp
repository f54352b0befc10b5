// test_host_api.cpp -- the C++ drop-in layer (include/rcomm_b200) driven the
// way the reference's own tests drive rcomm: host std::vector<float> buffers,
// one worker thread per GPU (tests/test_collectives.cpp:14-39 run_workers),
// results compared bit for bit with the CPU oracle (oracle/rcomm_oracle.h).
// Prints one PASS/FAIL line per check (acceptance.cpp style); exit code =
// number of failures.  Multi-worker cases run with min(#GPUs, 4) workers.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../oracle/rcomm_oracle.h"
#include "rcomm_b200/rcomm_b200.hpp"

using namespace rcomm::b200;

static int failures = 0, passes = 0;

static void report(bool ok, const std::string& name) {
  std::printf("%s %s\n", ok ? "PASS" : "FAIL", name.c_str());
  (ok ? passes : failures)++;
}

static bool bitwise(const std::vector<float>& a, const std::vector<float>& b) {
  return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), 4 * a.size()) == 0);
}

static std::vector<float> synth(std::size_t n, std::uint64_t seed) {
  std::vector<float> v(n);
  orc_synth(v.data(), n, seed, 0);
  return v;
}

template <typename F>
static void run_workers(int g, F fn) {  // one thread per GPU, like test_collectives.cpp:23-39
  ThreadGroup group(g);
  std::vector<std::thread> th;
  std::vector<std::string> errs(static_cast<std::size_t>(g));
  for (int r = 0; r < g; ++r)
    th.emplace_back([&, r] {
      try {
        cudaSetDevice(r);
        B200Endpoint ep(r, g, r, group.allgather(r));
        fn(ep, r);
      } catch (const std::exception& e) {
        errs[static_cast<std::size_t>(r)] = e.what();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : errs)
    if (!e.empty()) throw Error(B2_ERR_INVALID, e);
}

static void test_codec_kats() {
  Codec u8{CodecKind::uniform8};
  auto p = u8.encode(std::vector<float>{-1.0f, 1.0f, 0.0f});  // test_codec.cpp:114-123
  float lo, hi;
  std::memcpy(&lo, p.data(), 4);
  std::memcpy(&hi, p.data() + 4, 4);
  report(p.size() == 11 && lo == -1.0f && hi == 1.0f && p[8] == 0 && p[9] == 255 && p[10] == 128,
         "codec wire KAT {-1,1,0}");
  auto y = u8.decode(u8.encode(std::vector<float>{3.25f, 3.25f, 3.25f}), 3);  // test_codec.cpp:96-101
  report(y[0] == 3.25f && y[1] == 3.25f && y[2] == 3.25f, "codec degenerate constant");
  bool threw = false;
  try {
    u8.encode(std::vector<float>{1.0f, INFINITY});
  } catch (const Error&) {
    threw = true;
  }
  report(threw, "codec non-finite throws");
  threw = false;
  try {
    u8.decode(Payload{1, 2, 3}, 10);
  } catch (const Error&) {
    threw = true;
  }
  report(threw, "codec malformed payload throws");
  // random vectors vs the oracle, wire bytes exact
  bool ok = true;
  for (std::size_t n : {1ul, 7ul, 1000ul, 65537ul}) {
    auto x = synth(n, 100 + n);
    auto w = u8.encode(x);
    std::vector<std::uint8_t> ref(8 + n);
    orc_u8_encode_wire(x.data(), n, ref.data());
    ok &= w == ref;
    auto d = u8.decode(w, n);
    std::vector<float> rd(n);
    orc_u8_decode(x.empty() ? 0 : *reinterpret_cast<float*>(ref.data()), *reinterpret_cast<float*>(ref.data() + 4),
                  ref.data() + 8, n, rd.data());
    ok &= bitwise(d, rd);
  }
  report(ok, "codec random vectors bit-exact vs oracle");
  // compensate_encode residual definition (codec.cpp:125-137)
  auto x = synth(33, 9);
  std::vector<float> delta(33, 0.01f), dref = delta, dec;
  compensate_encode(u8, x, delta, nullptr, &dec);
  float l2, h2;
  std::vector<std::uint8_t> c(33);
  std::vector<float> dd(33);
  orc_u8_compensate_encode(x.data(), dref.data(), 33, &l2, &h2, c.data(), dd.data());
  report(bitwise(delta, dref) && bitwise(dec, dd), "compensate_encode bit-exact vs oracle");
}

static void test_onebit() {
  Codec ob{CodecKind::onebit};
  auto p = ob.encode(std::vector<float>{1, -1, 1, 1, -1, 1, 1, 1, -1});  // test_codec.cpp:103-123
  float scale;
  std::memcpy(&scale, p.data(), 4);
  report(p.size() == 6 && scale == 1.0f && p[4] == 0xED && p[5] == 0, "onebit wire KAT");
  bool ok = true;
  for (std::size_t n : {1ul, 9ul, 1000ul, 65537ul}) {
    auto x = synth(n, 300 + n);
    auto w = ob.encode(x);
    std::vector<std::uint8_t> ref(4 + (n + 7) / 8);
    orc_onebit_encode_wire(x.data(), n, ref.data());
    ok &= w == ref;
    auto d = ob.decode(w, n);
    std::vector<float> rd(n);
    orc_onebit_decode_wire(ref.data(), n, rd.data());
    ok &= bitwise(d, rd);
  }
  report(ok, "onebit random vectors bit-exact vs oracle");
  B200Endpoint ep(0, 1, 0);
  std::vector<float> x = {0.3f, -0.1f};  // test_collectives.cpp:209-225
  ErrorState es(2, 2, 0);
  c_lp_s(ep, 0.0, x, ob, &es);
  std::vector<float> d(2), e(2);
  cudaMemcpy(d.data(), es.delta(), 8, cudaMemcpyDefault);
  cudaMemcpy(e.data(), es.epsilon(), 8, cudaMemcpyDefault);
  report(std::fabs(x[0] - 0.2f) < 1e-6f && std::fabs(x[1] + 0.2f) < 1e-6f && std::fabs(d[0] - 0.1f) < 1e-6f &&
             std::fabs(d[1] - 0.1f) < 1e-6f && e[0] == 0.0f && e[1] == 0.0f,
         "c_lp_s onebit+EC single-worker KAT");
  for (std::size_t n : {37ul, 1000003ul}) {
    auto y = synth(n, 4242), want = y;
    float* xs[] = {want.data()};
    orc_c_lp_s(1, n, xs, ORC_CODEC_ONEBIT, nullptr, nullptr);
    c_lp_s(ep, 0.0, y, ob, nullptr);
    report(bitwise(y, want), "c_lp_s onebit g=1 n=" + std::to_string(n));
    auto z = synth(n, 4343);
    const float* nb[] = {z.data()};
    std::vector<float> wz(n);
    orc_d_lp_s_rank(n, nb, 1, ORC_CODEC_ONEBIT, ORC_REDUCE_AVERAGE, wz.data());
    d_lp_s(ep, 0.0, z, Topology{TopologyKind::ring, 1, 0}, 0, ob, ReduceMode::average);
    report(bitwise(z, wz), "d_lp_s onebit g=1 n=" + std::to_string(n));
  }
}

static void test_tensor() {  // test_tensor.cpp:10-60
  FlatTensor t1("t1", {2}, {1.0f, 2.0f}), t2("t2", {1}, {3.0f});
  auto arena = BucketArena::flatten({&t1, &t2});
  std::vector<float> h(3);
  cudaMemcpy(h.data(), arena.data(), 12, cudaMemcpyDeviceToHost);
  report(arena.size() == 3 && h == std::vector<float>{1.0f, 2.0f, 3.0f} && arena.members()[1].offset == 2,
         "flatten order and members");
  float nine = 9.0f;
  cudaMemcpy(arena.data() + 2, &nine, 4, cudaMemcpyHostToDevice);
  report(t2.to_host()[0] == 9.0f, "arena writes alias members");
  bool threw = false;
  FlatTensor a("x", {1}, {1.0f}), b("x", {1}, {2.0f});
  try {
    BucketArena::flatten({&a, &b});
  } catch (const Error&) {
    threw = true;
  }
  report(threw, "flatten rejects duplicate names");
}

static void test_single_rank() {
  B200Endpoint ep(0, 1, 0);
  Codec u8{CodecKind::uniform8};
  for (std::size_t n : {1ul, 37ul, 1000003ul}) {
    auto x = synth(n, 2026), want = x;
    float* xs[] = {want.data()};
    orc_c_lp_s(1, n, xs, ORC_CODEC_UNIFORM8, nullptr, nullptr);
    c_lp_s(ep, 0.0, x, u8, nullptr);  // host vector, staged
    report(bitwise(x, want), "c_lp_s g=1 host buffer n=" + std::to_string(n));
  }
  auto x = synth(10, 1), orig = x;
  c_fp_s(ep, 0.0, x);
  report(bitwise(x, orig), "c_fp_s g=1 leaves x untouched");
  bool threw = false;
  try {
    std::vector<float> v(10, 1.0f);
    ErrorState bad(3, 1);
    c_lp_s(ep, 0.0, v, u8, &bad);  // collectives.cpp:102-107
  } catch (const Error&) {
    threw = true;
  }
  report(threw, "error-state length validation throws");
  threw = false;
  try {
    std::vector<float> v(4, 0.0f);
    d_fp_s(ep, 0.0, v, Topology{TopologyKind::full, 5, 0}, 0, ReduceMode::sum);
  } catch (const Error&) {
    threw = true;
  }
  report(threw, "topology size mismatch throws");
}

static void test_multi(int g) {
  Codec u8{CodecKind::uniform8}, id{CodecKind::identity};
  for (std::size_t n : {5ul, 37ul, 100003ul}) {
    std::vector<std::vector<float>> in(g);
    for (int r = 0; r < g; ++r) in[r] = synth(n, 500 + r);
    // c_fp_s == fp64 ordered sum (test_collectives.cpp:77-93)
    auto want = in;
    std::vector<float*> ptr;
    for (auto& v : want) ptr.push_back(v.data());
    orc_c_fp_s(g, n, ptr.data());
    auto got = in;
    run_workers(g, [&](B200Endpoint& ep, int r) { c_fp_s(ep, 0.0, got[r]); });
    bool ok = true;
    for (int r = 0; r < g; ++r) ok &= bitwise(got[r], want[r]);
    report(ok, "c_fp_s g=" + std::to_string(g) + " n=" + std::to_string(n));
    // c_lp_s uint8 and identity collapse
    for (auto* codec : {&u8, &id}) {
      auto w2 = in;
      ptr.clear();
      for (auto& v : w2) ptr.push_back(v.data());
      orc_c_lp_s(g, n, ptr.data(), codec == &u8 ? ORC_CODEC_UNIFORM8 : ORC_CODEC_IDENTITY, nullptr, nullptr);
      auto g2 = in;
      std::vector<std::uint64_t> msgs(g);
      run_workers(g, [&](B200Endpoint& ep, int r) {
        c_lp_s(ep, 0.0, g2[r], *codec, nullptr);
        msgs[r] = ep.messages_sent();
      });
      ok = true;
      for (int r = 0; r < g; ++r) ok &= bitwise(g2[r], w2[r]) && msgs[r] == std::uint64_t(2 * (g - 1));
      report(ok, std::string("c_lp_s ") + (codec == &u8 ? "uint8" : "identity") + " g=" + std::to_string(g) +
                     " n=" + std::to_string(n));
    }
    // d_lp_s / d_fp_s on a ring
    Topology ring{TopologyKind::ring, g, 0};
    auto gd = in, gl = in;
    run_workers(g, [&](B200Endpoint& ep, int r) {
      d_fp_s(ep, 0.0, gd[r], ring, 3, ReduceMode::average);
      d_lp_s(ep, 0.0, gl[r], ring, 3, u8, ReduceMode::average);
    });
    ok = true;
    for (int r = 0; r < g; ++r) {
      auto nb = ring.neighbors(r, 3);
      std::vector<const float*> src;
      for (int j : nb) src.push_back(in[j].data());
      std::vector<float> wd(n), wl(n);
      orc_d_fp_s_rank(n, src.data(), static_cast<int>(src.size()), ORC_REDUCE_AVERAGE, wd.data());
      orc_d_lp_s_rank(n, src.data(), static_cast<int>(src.size()), ORC_CODEC_UNIFORM8, ORC_REDUCE_AVERAGE, wl.data());
      ok &= bitwise(gd[r], wd) && bitwise(gl[r], wl);
    }
    report(ok, "d_fp_s / d_lp_s ring g=" + std::to_string(g) + " n=" + std::to_string(n));
  }
  // error feedback over rounds (acceptance.cpp c4 shape)
  const std::size_t n = 37;
  std::vector<std::vector<float>> deltas(g, std::vector<float>(n, 0.0f)), eps(g);
  for (int r = 0; r < g; ++r) eps[r].assign(owned_partition_len(n, g, r), 0.0f);
  bool ok = true;
  {
    ThreadGroup group(g);
    std::vector<std::thread> th;
    std::vector<std::vector<std::vector<float>>> outs(g), dl(g);
    for (int r = 0; r < g; ++r)
      th.emplace_back([&, r] {
        cudaSetDevice(r);
        B200Endpoint ep(r, g, r, group.allgather(r));
        ErrorState es(n, owned_partition_len(n, g, r), r);
        for (int t = 0; t < 50; ++t) {
          auto x = synth(n, 7000 + 1000 * r + t);
          c_lp_s(ep, 0.0, x, Codec{CodecKind::uniform8}, &es);
          outs[r].push_back(x);
          dl[r].push_back(es.delta_host());
        }
      });
    for (auto& t : th) t.join();
    std::vector<float*> dp, ep_;
    for (int r = 0; r < g; ++r) {
      dp.push_back(deltas[r].data());
      ep_.push_back(eps[r].data());
    }
    for (int t = 0; t < 50; ++t) {
      std::vector<std::vector<float>> xs(g);
      std::vector<float*> xp;
      for (int r = 0; r < g; ++r) {
        xs[r] = synth(n, 7000 + 1000 * r + t);
        xp.push_back(xs[r].data());
      }
      orc_c_lp_s(g, n, xp.data(), ORC_CODEC_UNIFORM8, dp.data(), ep_.data());
      for (int r = 0; r < g; ++r) ok &= bitwise(outs[r][t], xs[r]) && bitwise(dl[r][t], deltas[r]);
    }
  }
  report(ok, "c_lp_s + error feedback, 50 rounds, g=" + std::to_string(g));
}

// engine: plan KAT (test_engine.cpp:65-93) + bucketed C_LP_S overlapping a
// compute stream, every bucket vs the oracle over that bucket of every rank
void test_engine(int g) {
  if (g == 1) {
    auto b = plan_buckets({32, 8, 8, 1}, 40);
    bool ok = b.size() == 3 && b[0].layers == std::vector<std::size_t>{3, 2} &&
              b[1].layers == std::vector<std::size_t>{1} && b[2].layers == std::vector<std::size_t>{0} &&
              b[0].trigger_layer == 2 && b[0].elements == 9 && b[2].elements == 32;
    ok &= plan_buckets({32, 8, 8, 1}, 40, false).size() == 4;
    report(ok, "engine plan_buckets (reference KATs)");
    return;
  }
  const std::vector<std::size_t> sizes = {3000, 17, 70001, 5, 25000, 1024};
  const auto plan = plan_buckets(sizes, 4 * 30000);
  std::vector<std::vector<std::vector<float>>> got(g);  // [rank][bucket]
  {
    ThreadGroup group(g);
    std::vector<std::thread> th;
    for (int r = 0; r < g; ++r)
      th.emplace_back([&, r] {
        cudaSetDevice(r);
        B200Endpoint ep(r, g, r, group.allgather(r));
        OverlapEngine eng(ep, sizes, 4 * 30000);
        cudaStream_t compute;
        cudaStreamCreateWithFlags(&compute, cudaStreamNonBlocking);
        for (std::size_t i = 0; i < sizes.size(); ++i) {
          const std::size_t l = sizes.size() - 1 - i;
          auto v = synth(sizes[l], 41000 + 10 * l + r);
          cudaMemcpyAsync(eng.grad(l), v.data(), 4 * v.size(), cudaMemcpyHostToDevice, compute);
          cudaStreamSynchronize(compute);  // v dies here
          eng.layer_done(l, compute);
        }
        eng.finish(compute);
        cudaStreamSynchronize(compute);
        for (const auto& b : eng.buckets()) {
          std::vector<float> h(b.elements);
          cudaMemcpy(h.data(), eng.arena(b.id).data(), 4 * h.size(), cudaMemcpyDeviceToHost);
          got[r].push_back(std::move(h));
        }
        cudaStreamDestroy(compute);
      });
    for (auto& t : th) t.join();
  }
  bool ok = true;
  for (const auto& b : plan) {
    std::vector<std::vector<float>> xs(g);
    std::vector<float*> xp;
    for (int r = 0; r < g; ++r) {
      for (std::size_t l : b.layers) {
        auto v = synth(sizes[l], 41000 + 10 * l + r);
        xs[r].insert(xs[r].end(), v.begin(), v.end());
      }
      xp.push_back(xs[r].data());
    }
    orc_c_lp_s(g, b.elements, xp.data(), ORC_CODEC_UNIFORM8, nullptr, nullptr);
    for (int r = 0; r < g; ++r) ok &= bitwise(got[r][b.id], xs[r]);
  }
  report(ok, "engine: bucketed c_lp_s overlapping a compute stream, g=" + std::to_string(g) + ", " +
                 std::to_string(plan.size()) + " buckets");
}

int main() {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    std::printf("SKIP no GPU\n");
    return 0;
  }
  try {
    test_codec_kats();
    test_onebit();
    test_tensor();
    test_single_rank();
    for (int g = 2; g <= std::min(ndev, 4); g *= 2) test_multi(g);
    test_engine(1);
    for (int g = 2; g <= std::min(ndev, 4); g *= 2) test_engine(g);
  } catch (const std::exception& e) {
    report(false, std::string("exception: ") + e.what());
  }
  std::printf("%d passed, %d failed\n", passes, failures);
  return failures;
}
