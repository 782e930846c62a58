// SPDX-License-Identifier: Apache-2.0
// TEST INFRASTRUCTURE: the train-math seams driven by the reference's own data
// plane. TransferQueue, StreamLoader and StalenessGate are the reference's
// (proj/src/{transfer_queue,stream_loader,staleness,common}.cpp, compiled where
// they lie by `make -C oracle bus` into oracle/_ref/libsfbus.a); the seams
// (include/staleflow/train_math_seam.hpp) are the product.
//
//   ./test_bus_seam cpu      CPU: bus delivery in readiness order, group-completion
//                            batching in the Advantages stage (no ConfigError on a
//                            shuffled stream, GRPO over complete groups equal to a
//                            direct computation), the trainer's decode of every
//                            sample, staleness tags vs StalenessGate::staleness_of,
//                            version boundaries at G consumed samples
//   ./test_bus_seam gpu      B200: the same loop with the device seams: Advantages
//                            via AdvantageStageSeam, the Actor loss via
//                            ActorLossSeam::step (bitwise equal to the C-ABI on the
//                            same arrays), version-boundary normalisation equal to
//                            the explicit-N run, the R3 record uploaded token-major
//                            and transposed on device (FNV digest equal to the host
//                            codec)
//   ./test_bus_seam bench    B200: the trainer loop StreamLoader::next_micro_batch ->
//                            ActorLossSeam::step at the config-2 micro-batch shape
//                            (32 x 4096 tokens, V = 151,936 bf16), one JSON line
//
// Reference defects on this path do not arise here: the
// field contract is declared directly (no ScenarioConfig / validate_algorithm)
// and the bus is in-process (no TCP server teardown).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "staleflow/staleness.hpp"
#include "staleflow/stream_loader.hpp"
#include "staleflow/train_math_seam.hpp"
#include "staleflow/transfer_queue.hpp"

#ifdef SF_WITH_CUDA
#include <cuda_runtime.h>
#endif

using staleflow::Bytes;
using staleflow::MicroBatch;
namespace tms = staleflow::train_math;

namespace {

int fails = 0;
size_t max_partial_groups = 0;  // the readiness order really did split groups across fetches
#define CHECK(c)                                                         \
  do {                                                                   \
    if (!(c)) {                                                          \
      std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);   \
      ++fails;                                                           \
    }                                                                    \
  } while (0)

template <class T>
Bytes enc(const T* v, size_t n) {
  Bytes b(n * sizeof(T));
  if (n) std::memcpy(b.data(), v, b.size());
  return b;
}

[[maybe_unused]] uint64_t fnv1a(const void* p, size_t n) {  // FNV-1a 64 (proj/include/staleflow/hash.hpp:14-31)
  uint64_t h = 1469598103934665603ull;
  const uint8_t* b = static_cast<const uint8_t*>(p);
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 1099511628211ull;
  }
  return h;
}

struct Truth {  // what the producers put for one sample
  std::vector<int32_t> response;
  std::vector<float> logp, ref_logp;
  float reward = 0.f;
  float advantage = 0.f;
  std::vector<uint8_t> routed;  // [L, layers, k] token-major
  int64_t version = 0;
};

struct Cfg {
  int G = 8;           // rollouts per prompt (GRPO group size)
  int prompts = 16;    // per version
  int versions = 3;
  int m = 32;          // micro-batch size
  int lmin = 40, lmax = 300;
  int V = 32000;
  int layers = 0, k = 8, experts = 128;  // R3 record (layers = 0: no record)
  uint32_t seed = 7;
};

// Producers: StalenessGate permits assign sample ids (sequential per permit,
// staleness.cpp:102-106) and versions; each sample's fields become ready at a
// random time, so the bus order interleaves groups (transfer_queue.cpp:162-175).
struct World {
  Cfg c;
  double clock = 0.0;
  staleflow::TransferQueue q;
  staleflow::StalenessGate gate;
  std::map<uint64_t, Truth> truth;
  std::mt19937 rng;
  std::vector<std::string> trainer_fields;
  explicit World(const Cfg& cfg)
      : c(cfg), q([this] { return clock; }),
        gate(staleflow::GatePolicy{2, static_cast<uint64_t>(cfg.G * cfg.prompts), static_cast<uint32_t>(cfg.m), 2}),
        rng(cfg.seed) {
    trainer_fields = {"advantage", "logp", "ref_logp", "response", "reward"};
    if (c.layers > 0) trainer_fields.push_back("routed_experts");
    std::sort(trainer_fields.begin(), trainer_fields.end());
  }

  // One version's samples, produced by two replicas (one lagging a version).
  void produce_version(int64_t v_t) {
    const int n = c.G * c.prompts;
    std::vector<std::pair<double, uint64_t>> done;
    int made = 0;
    while (made < n) {
      const std::string rep = (made / c.m) % 2 ? "r1" : "r0";
      auto out = gate.acquire_generation_permit(rep);
      if (!out.ok() || !std::holds_alternative<staleflow::GenerationPermit>(out.value())) {
        std::printf("no permit for %s at v_t=%lld\n", rep.c_str(), static_cast<long long>(v_t));
        ++fails;
        return;
      }
      const auto& p = std::get<staleflow::GenerationPermit>(out.value());
      for (uint32_t i = 0; i < p.sample_count; ++i) {
        const uint64_t id = p.first_sample_id + i;
        Truth& t = truth[id];
        t.version = p.granted_at_version;
        const int L = c.lmin + static_cast<int>(rng() % static_cast<uint32_t>(c.lmax - c.lmin + 1));
        std::uniform_real_distribution<float> u(-6.f, -0.1f);
        t.response.resize(L);
        t.logp.resize(L);
        t.ref_logp.resize(L);
        for (int j = 0; j < L; ++j) {
          t.response[j] = static_cast<int32_t>(rng() % static_cast<uint32_t>(c.V));
          t.logp[j] = u(rng);
          t.ref_logp[j] = t.logp[j] + 0.05f * (u(rng) + 3.f);
        }
        t.reward = (rng() & 1) ? 1.f : 0.f;
        if (c.layers > 0) {
          t.routed.resize(static_cast<size_t>(L) * c.layers * c.k);
          for (auto& b : t.routed) b = static_cast<uint8_t>(rng() % static_cast<uint32_t>(c.experts));
        }
        done.emplace_back(std::uniform_real_distribution<double>(0, 1)(rng), id);
      }
      gate.complete_permit(p.permit_id);
      made += static_cast<int>(p.sample_count);
    }
    std::sort(done.begin(), done.end());
    std::vector<std::string> expected = {"logp", "ref_logp", "response", "reward"};
    if (c.layers > 0) expected.push_back("routed_experts");
    expected.push_back("advantage");
    for (const auto& [tm, id] : done) {
      clock = static_cast<double>(v_t) + tm;
      const Truth& t = truth[id];
      staleflow::SampleMeta meta{id, v_t, t.version, ""};
      const size_t L = t.response.size();
      auto put = [&](const char* f, Bytes b) {
        auto r = q.put_field(meta, staleflow::FieldKey{f, staleflow::Modality::Text}, std::move(b), expected);
        if (!r.ok()) {
          std::printf("put_field %s failed\n", f);
          ++fails;
        }
      };
      put("response", enc(t.response.data(), L));
      put("logp", enc(t.logp.data(), L));
      put("ref_logp", enc(t.ref_logp.data(), L));
      put("reward", enc(&t.reward, 1));
      if (c.layers > 0) put("routed_experts", enc(t.routed.data(), t.routed.size()));
    }
  }
};

// GRPO over one complete group (unbiased std, eps 1e-6; P2/P3), in double.
void grpo_direct(const std::vector<float>& r, std::vector<float>& a) {
  const double n = static_cast<double>(r.size());
  double mean = 0, mn = r[0], mx = r[0];
  for (float x : r) {
    mean += x;
    mn = std::min<double>(mn, x);
    mx = std::max<double>(mx, x);
  }
  mean /= n;
  double ss = 0;
  for (float x : r) ss += (x - mean) * (x - mean);
  a.resize(r.size());
  for (size_t i = 0; i < r.size(); ++i)
    a[i] = mx == mn ? 0.f : static_cast<float>((r[i] - mean) / (std::sqrt(ss / (n - 1)) + 1e-6));
}

// The Advantages stage (controller.cpp:79 reward -> advantage): fetch reward in
// readiness order, assemble complete groups, compute, put `advantage`.
int advantages_stage(World& w, tms::GroupAssembler<MicroBatch>& asmb, bool gpu, void* stream) {
  (void)stream;
  int batches = 0;
  for (;;) {
    auto got = w.q.get_ready_batch("adv", {"reward"}, w.c.m, false, true);
    if (!got.ok()) break;
    std::string err;
    CHECK(asmb.feed(got.value(), &err) == SF_TM_OK);
    max_partial_groups = std::max(max_partial_groups, asmb.pending_groups());
    w.q.mark_consumed("adv", got.value().batch_id);
    MicroBatch mb;
    while (asmb.pop(mb, static_cast<size_t>(w.c.m)) > 0) {
      ++batches;
      tms::PackedBatch pb;
      // every popped batch is whole groups (the trainer-side check passes)
      for (size_t i = 0; i < mb.sample_ids.size(); ++i) pb.group_ids.push_back(static_cast<int32_t>((mb.sample_ids[i] - 1) / w.c.G));
      CHECK(tms::check_complete_groups(pb, w.c.G, &err) == SF_TM_OK);
      std::vector<Bytes> adv;
#ifdef SF_WITH_CUDA
      if (gpu) {
        static tms::AdvantageStageSeam seam(0);
        CHECK(seam.run(mb, w.c.G, 1e-6f, SF_TM_STD_UNBIASED, adv, stream) == SF_TM_OK);
      }
#endif
      // direct GRPO per group (the check of the stage's output)
      for (size_t g0 = 0; g0 < mb.sample_ids.size(); g0 += static_cast<size_t>(w.c.G)) {
        std::vector<float> r, a;
        for (int i = 0; i < w.c.G; ++i) r.push_back(w.truth[mb.sample_ids[g0 + i]].reward);
        grpo_direct(r, a);
        for (int i = 0; i < w.c.G; ++i) {
          const uint64_t id = mb.sample_ids[g0 + i];
          float av = a[static_cast<size_t>(i)];
          if (gpu) {
            float got_a;
            std::memcpy(&got_a, adv[g0 + i].data(), 4);
            CHECK(std::fabs(got_a - av) <= 1e-6f + 1e-6f * std::fabs(av));
            av = got_a;
          }
          w.truth[id].advantage = av;
          const Truth& t = w.truth[id];
          staleflow::SampleMeta meta{id, 0, t.version, ""};
          auto r2 = w.q.put_field(meta, staleflow::FieldKey{"advantage", staleflow::Modality::Scalar}, enc(&av, 1), {});
          CHECK(r2.ok());
        }
      }
    }
  }
  return batches;
}

bool decode_matches(World& w, const MicroBatch& b, const tms::PackedBatch& p) {
  size_t off = 0;
  for (size_t i = 0; i < b.sample_ids.size(); ++i) {
    const Truth& t = w.truth[b.sample_ids[i]];
    const size_t L = t.response.size();
    if (p.seq_lens[i] != static_cast<int32_t>(L)) return false;
    if (std::memcmp(p.targets.data() + off, t.response.data(), L * 4) ||
        std::memcmp(p.logp.data() + off, t.logp.data(), L * 4) ||
        std::memcmp(p.ref_logp.data() + off, t.ref_logp.data(), L * 4) || p.per_sample[i] != t.advantage ||
        p.producer_versions[i] != t.version)
      return false;
    off += L;
  }
  return off == static_cast<size_t>(p.T);
}

#ifdef SF_WITH_CUDA
#define CU(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) {                                                                   \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);          \
      std::exit(2);                                                                            \
    }                                                                                          \
  } while (0)
#endif

// The trainer: StreamLoader over the bus; decode + (GPU) ActorLossSeam::step;
// version boundaries every G consumed samples.
int run_loop(const Cfg& c, bool gpu) {
  World w(c);
  w.q.register_group("adv");
  CHECK(w.gate.register_replica("r0", 0).ok());
  CHECK(w.gate.register_replica("r1", 0).ok());
  staleflow::LoaderConfig lc;
  lc.micro_batch_size = c.m;
  lc.global_batch_size = c.G * c.prompts;
  lc.required_fields = w.trainer_fields;
  staleflow::StreamLoader loader(w.q, "actor", lc, [&w] { return w.clock; });
  CHECK(loader.attach().ok());
  tms::GroupAssembler<MicroBatch> asmb(c.G);
  tms::VersionAccumulator acc(static_cast<uint64_t>(c.G * c.prompts));
  std::map<int64_t, uint64_t> stale_hist;
  int64_t v_t = 0;
  uint64_t delivered = 0;
  int adv_batches = 0;
  void* stream = nullptr;
#ifdef SF_WITH_CUDA
  tms::ActorLossSeam actor(0);
  tms::RoutedExpertsSeam r3(0);
  sf_tm_t h = nullptr;
  CHECK(sf_tm_create(0, &h) == SF_TM_OK);
  void *d_logits = nullptr, *d_dl = nullptr, *d_dl2 = nullptr, *d_tok = nullptr, *d_rec = nullptr;
  const int64_t Tcap = static_cast<int64_t>(c.m) * c.lmax;
  if (gpu) {
    CU(cudaMalloc(&d_logits, static_cast<size_t>(Tcap) * c.V * 2));
    CU(cudaMalloc(&d_dl, static_cast<size_t>(Tcap) * c.V * 2));
    CU(cudaMalloc(&d_dl2, static_cast<size_t>(Tcap) * c.V * 2));
    if (c.layers > 0) {
      CU(cudaMalloc(&d_tok, static_cast<size_t>(Tcap) * c.layers * c.k));
      CU(cudaMalloc(&d_rec, static_cast<size_t>(Tcap) * c.layers * c.k));
    }
  }
  std::vector<std::vector<float>> version_metrics;  // micro metrics (inv_norm = 1) of the open version
  std::vector<MicroBatch> version_batches;
  double r3_dev_ms = 0, r3_host_ms = 0;
#endif
  for (int ver = 0; ver < c.versions; ++ver) {
    if (ver > 0) {  // r1 lags one version behind the trainer: staleness 1 samples
      CHECK(w.gate.set_replica_version("r0", v_t).ok());
      CHECK(w.gate.set_replica_version("r1", v_t - 1).ok());
    }
    w.produce_version(v_t);
    adv_batches += advantages_stage(w, asmb, gpu, stream);
    CHECK(asmb.pending_samples() == 0 && asmb.ready_samples() == 0);
    for (;;) {
      auto got = loader.try_next();
      if (!got.ok()) break;
      const MicroBatch& b = got.value();
      delivered += b.sample_ids.size();
      tms::PackedBatch pb;
      std::string err;
      CHECK(tms::pack_trainer_batch(b, c.G, pb, &err) == SF_TM_OK);
      CHECK(decode_matches(w, b, pb));
      int64_t bs = 0;
      auto hist = tms::staleness_histogram(pb, v_t, &bs);
      CHECK(bs == staleflow::StalenessGate::staleness_of(v_t, b.producer_versions));
      for (const auto& kv : hist) stale_hist[kv.first] += kv.second;
      float met[SF_TM_NUM_METRICS] = {};
#ifdef SF_WITH_CUDA
      if (gpu) {
        // device logits of this micro-batch (the LM-head output in the trainer)
        CHECK(sf_tm_synth_logits(h, d_logits, SF_TM_BF16, pb.T, c.V, c.V, 1000 + b.batch_id, 2.f, nullptr, 5.f, 25.f,
                                 1e-3f, nullptr) == SF_TM_OK);
        sf_tm_loss_params prm;
        sf_tm_default_loss_params(&prm);
        const sf_tm_loss_params mp = tms::VersionAccumulator::micro_params(prm);
        CHECK(actor.step(b, d_logits, SF_TM_BF16, c.V, d_dl, mp, met, stream, c.G) == SF_TM_OK);
        CU(cudaDeviceSynchronize());
        // the same arrays through the C-ABI directly: bitwise equal
        float met2[SF_TM_NUM_METRICS];
        CHECK(sf_tm_pg_step_host(h, d_logits, SF_TM_BF16, pb.T, c.V, c.V, pb.targets.data(), pb.logp.data(),
                                 pb.ref_logp.data(), nullptr, pb.seq_lens.data(), nullptr, pb.per_sample.data(),
                                 pb.group_ids.data(), pb.B, -1.f, SF_TM_STD_UNBIASED, &mp, d_dl2, c.V, met2,
                                 nullptr) == SF_TM_OK);
        CU(cudaDeviceSynchronize());
        CHECK(std::memcmp(met, met2, sizeof(met)) == 0);
        std::vector<uint16_t> a(static_cast<size_t>(pb.T) * c.V), bb(a.size());
        CU(cudaMemcpy(a.data(), d_dl, a.size() * 2, cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(bb.data(), d_dl2, bb.size() * 2, cudaMemcpyDeviceToHost));
        CHECK(a == bb);
        version_metrics.emplace_back(met, met + SF_TM_NUM_METRICS);
        version_batches.push_back(b);
        if (c.layers > 0) {  // R3 record: token-major upload + device transpose == host codec
          int64_t T3 = 0;
          auto t0 = std::chrono::steady_clock::now();
          CHECK(r3.upload(b, c.layers, c.k, d_tok, d_rec, &T3, stream) == SF_TM_OK);
          CU(cudaDeviceSynchronize());
          auto t1 = std::chrono::steady_clock::now();
          std::vector<uint8_t> host;
          int64_t T4 = 0;
          CHECK(tms::pack_routed_experts(b, c.layers, c.k, host, &T4, &err) == SF_TM_OK);
          CU(cudaMemcpy(d_tok, host.data(), host.size(), cudaMemcpyHostToDevice));
          auto t2 = std::chrono::steady_clock::now();
          std::vector<uint8_t> dev(host.size());
          CU(cudaMemcpy(dev.data(), d_rec, dev.size(), cudaMemcpyDeviceToHost));
          CHECK(T3 == T4 && fnv1a(dev.data(), dev.size()) == fnv1a(host.data(), host.size()));
          r3_dev_ms += std::chrono::duration<double, std::milli>(t1 - t0).count();
          r3_host_ms += std::chrono::duration<double, std::milli>(t2 - t1).count();
        }
      } else
#endif
      {
        met[SF_TM_M_ACTIVE] = static_cast<float>(pb.T);
      }
      acc.add(met, b.sample_ids.size());
      CHECK(loader.ack(b).ok());
      if (acc.at_boundary()) {  // version boundary (sim_runtime.cpp:453-454)
        const auto cl = acc.close();
        CHECK(cl.samples == static_cast<uint64_t>(c.G * c.prompts));
#ifdef SF_WITH_CUDA
        if (gpu) {
          // the same version with N known up front: equal metrics (linearity)
          sf_tm_loss_params prm;
          sf_tm_default_loss_params(&prm);
          prm.norm_mode = SF_TM_NORM_EXPLICIT;
          prm.inv_norm = static_cast<float>(1.0 / cl.active_tokens);
          double sum[SF_TM_NUM_METRICS] = {};
          for (size_t j = 0; j < version_batches.size(); ++j) {
            const MicroBatch& vb = version_batches[j];
            tms::PackedBatch vp;
            CHECK(tms::pack_trainer_batch(vb, c.G, vp, &err) == SF_TM_OK);
            CHECK(sf_tm_synth_logits(h, d_logits, SF_TM_BF16, vp.T, c.V, c.V, 1000 + vb.batch_id, 2.f, nullptr, 5.f,
                                     25.f, 1e-3f, nullptr) == SF_TM_OK);
            float m2[SF_TM_NUM_METRICS];
            CHECK(actor.step(vb, d_logits, SF_TM_BF16, c.V, d_dl2, prm, m2, stream, c.G) == SF_TM_OK);
            CU(cudaDeviceSynchronize());
            for (int i = 0; i < SF_TM_NUM_METRICS; ++i) sum[i] += m2[i];
            if (j == 0) {  // gradients: the unnormalised run scaled by 1/N == the normalised run (1 bf16 ulp)
              sf_tm_loss_params mp = tms::VersionAccumulator::micro_params(prm);
              float m1[SF_TM_NUM_METRICS];
              CHECK(actor.step(vb, d_logits, SF_TM_BF16, c.V, d_dl, mp, m1, stream, c.G) == SF_TM_OK);
              CU(cudaDeviceSynchronize());
              std::vector<uint16_t> g1(static_cast<size_t>(vp.T) * c.V), g2(g1.size());
              CU(cudaMemcpy(g1.data(), d_dl, g1.size() * 2, cudaMemcpyDeviceToHost));
              CU(cudaMemcpy(g2.data(), d_dl2, g2.size() * 2, cudaMemcpyDeviceToHost));
              size_t bad = 0;
              for (size_t e = 0; e < g1.size(); ++e) {
                uint32_t u1 = static_cast<uint32_t>(g1[e]) << 16, u2 = static_cast<uint32_t>(g2[e]) << 16;
                float f1, f2;
                std::memcpy(&f1, &u1, 4);
                std::memcpy(&f2, &u2, 4);
                const double x = static_cast<double>(f1) * cl.grad_scale;
                const double ulp = std::ldexp(1.0, std::ilogb(std::fabs(x) > 1e-38 ? x : 1e-38) - 7);
                if (std::fabs(x - f2) > 2 * ulp + 1e-12) ++bad;
              }
              CHECK(bad == 0);
            }
          }
          for (int i = 0; i < SF_TM_NUM_METRICS; ++i) {
            const double tol = (i == SF_TM_M_ACTIVE) ? 0 : 1e-5 * std::fabs(sum[i]) + 1e-6;
            if (!(std::fabs(cl.metrics[i] - sum[i]) <= tol)) {
              std::printf("version metric %d: boundary %.9g vs explicit-N %.9g\n", i, cl.metrics[i], sum[i]);
              ++fails;
            }
          }
          version_metrics.clear();
          version_batches.clear();
        }
#endif
        ++v_t;
        CHECK(w.gate.record_train_version(v_t).ok());
      }
    }
  }
  CHECK(delivered == static_cast<uint64_t>(c.G * c.prompts * c.versions));
  CHECK(max_partial_groups > 0);
  CHECK(stale_hist.size() == 2 && stale_hist[1] > 0);  // staleness tags 0 and 1 pass through
  std::printf("loop: %llu samples, %d versions, %d advantage micro-batches (complete groups; up to %zu partial "
              "groups buffered), staleness",
              static_cast<unsigned long long>(delivered), c.versions, adv_batches, max_partial_groups);
  for (const auto& kv : stale_hist) std::printf(" %lld:%llu", static_cast<long long>(kv.first),
                                                static_cast<unsigned long long>(kv.second));
  std::printf("\n");
#ifdef SF_WITH_CUDA
  if (gpu && c.layers > 0)
    std::printf("r3 record: token-major upload + device transpose %.3f ms vs host transpose + H2D %.3f ms (total)\n",
                r3_dev_ms, r3_host_ms);
  if (gpu) {
    cudaFree(d_logits);
    cudaFree(d_dl);
    cudaFree(d_dl2);
    if (d_tok) cudaFree(d_tok);
    if (d_rec) cudaFree(d_rec);
    sf_tm_destroy(h);
  }
#endif
  return 0;
}

#ifdef SF_WITH_CUDA
// Trainer e2e through the reference's API at the config-2 micro-batch shape:
// StreamLoader::next_micro_batch (bus deep copy of the payloads) ->
// ActorLossSeam::step (decode, pinned staging, H2D, GRPO/weights, fused loss,
// D2H metrics). The logits are device-resident (the LM-head output).
int bench(int micro_batches) {
  Cfg c;
  c.G = 8;
  c.m = 32;
  c.prompts = 4 * micro_batches;  // 32 samples per micro-batch
  c.versions = 1;
  c.lmin = c.lmax = 4096;
  c.V = 151936;
  World w(c);
  CHECK(w.gate.register_replica("r0", 0).ok());
  CHECK(w.gate.register_replica("r1", 0).ok());
  w.produce_version(0);
  // advantages precomputed (this line times the trainer, not the stage)
  for (auto& kv : w.truth) {
    staleflow::SampleMeta meta{kv.first, 0, kv.second.version, ""};
    CHECK(w.q.put_field(meta, staleflow::FieldKey{"advantage", staleflow::Modality::Scalar},
                        enc(&kv.second.reward, 1), {})
              .ok());
  }
  staleflow::LoaderConfig lc;
  lc.micro_batch_size = c.m;
  lc.global_batch_size = c.G * c.prompts;
  lc.required_fields = w.trainer_fields;
  staleflow::StreamLoader loader(w.q, "actor", lc, [] { return 0.0; });
  CHECK(loader.attach().ok());
  tms::ActorLossSeam actor(0);
  sf_tm_t h = nullptr;
  CHECK(sf_tm_create(0, &h) == SF_TM_OK);
  const int64_t T = static_cast<int64_t>(c.m) * c.lmax;
  void *d_logits = nullptr, *d_dl = nullptr;
  CU(cudaMalloc(&d_logits, static_cast<size_t>(T) * c.V * 2));
  CU(cudaMalloc(&d_dl, static_cast<size_t>(T) * c.V * 2));
  CHECK(sf_tm_synth_logits(h, d_logits, SF_TM_BF16, T, c.V, c.V, 42, 2.f, nullptr, 5.f, 25.f, 1e-3f, nullptr) == 0);
  sf_tm_loss_params prm;
  sf_tm_default_loss_params(&prm);
  prm.norm_mode = SF_TM_NORM_EXPLICIT;
  prm.inv_norm = 1.f / static_cast<float>(T);
  std::vector<float> met(static_cast<size_t>(micro_batches) * SF_TM_NUM_METRICS);
  cudaEvent_t e0, e1;
  CU(cudaEventCreate(&e0));
  CU(cudaEventCreate(&e1));
  // warm-up: the first micro-batch (grow-once staging and scratch)
  auto first = loader.next_micro_batch();
  CHECK(first.ok());
  CHECK(actor.step(first.value(), d_logits, SF_TM_BF16, c.V, d_dl, prm, met.data(), nullptr, c.G) == SF_TM_OK);
  CHECK(loader.ack(first.value()).ok());
  CU(cudaDeviceSynchronize());
  const auto h0 = std::chrono::steady_clock::now();
  CU(cudaEventRecord(e0, nullptr));
  int n = 0;
  uint64_t tokens = 0;
  double fetch_ms = 0, step_ms = 0;
  std::vector<MicroBatch> kept;
  for (int i = 1; i < micro_batches; ++i) {
    const auto a0 = std::chrono::steady_clock::now();
    auto got = loader.next_micro_batch();
    if (!got.ok()) break;
    const auto a1 = std::chrono::steady_clock::now();
    CHECK(actor.step(got.value(), d_logits, SF_TM_BF16, c.V, d_dl, prm, met.data() + i * SF_TM_NUM_METRICS,
                     nullptr, c.G) == SF_TM_OK);
    const auto a2 = std::chrono::steady_clock::now();
    CHECK(loader.ack(got.value()).ok());
    fetch_ms += std::chrono::duration<double, std::milli>(a1 - a0).count();
    step_ms += std::chrono::duration<double, std::milli>(a2 - a1).count();
    tokens += static_cast<uint64_t>(actor.packed().T);
    kept.push_back(got.value());
    ++n;
  }
  CU(cudaEventRecord(e1, nullptr));
  CU(cudaEventSynchronize(e1));
  const auto h1 = std::chrono::steady_clock::now();
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, e0, e1));
  const double wall = std::chrono::duration<double, std::milli>(h1 - h0).count();
  // the same steps on the already fetched batches (no bus in the timed region)
  CU(cudaEventRecord(e0, nullptr));
  for (int i = 0; i < n; ++i)
    CHECK(actor.step(kept[i], d_logits, SF_TM_BF16, c.V, d_dl, prm, met.data(), nullptr, c.G) == SF_TM_OK);
  CU(cudaEventRecord(e1, nullptr));
  CU(cudaEventSynchronize(e1));
  float ms_steps = 0;
  CU(cudaEventElapsedTime(&ms_steps, e0, e1));
  // and the fused loss alone on device-resident fields
  CU(cudaEventRecord(e0, nullptr));
  for (int i = 0; i < n; ++i)
    CHECK(sf_tm_pg_step_host(h, d_logits, SF_TM_BF16, actor.packed().T, c.V, c.V, actor.packed().targets.data(),
                             actor.packed().logp.data(), actor.packed().ref_logp.data(), nullptr,
                             actor.packed().seq_lens.data(), nullptr, actor.packed().per_sample.data(),
                             actor.packed().group_ids.data(), actor.packed().B, -1.f, SF_TM_STD_UNBIASED, &prm, d_dl,
                             c.V, met.data(), nullptr) == SF_TM_OK);
  CU(cudaEventRecord(e1, nullptr));
  CU(cudaEventSynchronize(e1));
  float ms_abi = 0;
  CU(cudaEventElapsedTime(&ms_abi, e0, e1));
  std::printf("{\"path\": \"StreamLoader::next_micro_batch -> ActorLossSeam::step (reference bus, in-process)\", "
              "\"micro_batches\": %d, \"tokens\": %llu, \"ms_per_micro_batch\": %.4f, \"tokens_per_s\": %.1f, "
              "\"wall_ms_per_micro_batch\": %.4f, \"host_fetch_ms_per_micro_batch\": %.4f, "
              "\"host_step_call_ms_per_micro_batch\": %.4f, \"seam_steps_only_ms_per_micro_batch\": %.4f, "
              "\"c_abi_host_call_ms_per_micro_batch\": %.4f, \"bus_bytes\": %llu}\n",
              n, static_cast<unsigned long long>(tokens), ms / n, tokens / (ms / 1e3), wall / n, fetch_ms / n,
              step_ms / n, ms_steps / n, ms_abi / n, static_cast<unsigned long long>(loader.wait_stats().bus_bytes));
  cudaFree(d_logits);
  cudaFree(d_dl);
  sf_tm_destroy(h);
  return 0;
}
#endif

}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  if (mode == "cpu") {
    Cfg c;
    run_loop(c, false);
    Cfg c2;  // group size 16, odd micro-batch/group ratio
    c2.G = 16;
    c2.prompts = 6;
    c2.m = 24;
    c2.seed = 11;
    run_loop(c2, false);
    std::printf(fails ? "BUS CPU FAIL %d\n" : "BUS CPU OK\n", fails);
    return fails ? 1 : 0;
  }
#ifdef SF_WITH_CUDA
  if (mode == "gpu") {
    Cfg c;
    c.layers = 48;
    c.prompts = 8;
    run_loop(c, true);
    std::printf(fails ? "BUS GPU FAIL %d\n" : "BUS GPU OK\n", fails);
    return fails ? 1 : 0;
  }
  if (mode == "bench") {
    bench(argc > 2 ? std::atoi(argv[2]) : 16);
    return fails ? 1 : 0;
  }
#endif
  std::printf("unknown mode %s\n", mode.c_str());
  return 2;
}
