// SPDX-License-Identifier: Apache-2.0
// Exercises include/staleflow/train_math_seam.hpp.
//   ./test_seam pack   CPU: MicroBatch payload codec (against the reference's own
//                      staleflow::MicroBatch when built with -DSF_USE_REF_TYPES)
//   ./test_seam gpu    B200: ActorLossSeam::step == sf_tm_pg_step_host on the same
//                      packed arrays (bitwise metrics and dlogits)
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#ifdef SF_USE_REF_TYPES
#include "staleflow/types.hpp"  // /root/reference/proj/include (drop-in check)
using staleflow::Bytes;
using staleflow::MicroBatch;
#else
namespace mirror {  // same member names as proj/include/staleflow/types.hpp:48-59
using Bytes = std::vector<std::uint8_t>;
struct MicroBatch {
  std::uint64_t batch_id = 0;
  std::vector<std::uint64_t> sample_ids;
  std::vector<std::string> field_set;
  std::vector<std::int64_t> producer_versions;
  std::vector<std::int64_t> global_steps;
  std::vector<std::vector<Bytes>> payloads;
};
}  // namespace mirror
using mirror::Bytes;
using mirror::MicroBatch;
#endif

#include "staleflow/train_math_seam.hpp"

#ifdef SF_WITH_CUDA
#include <cuda_runtime.h>
#endif

namespace {
template <class T>
Bytes enc(const std::vector<T>& v) {
  Bytes b(v.size() * sizeof(T));
  if (!v.empty()) std::memcpy(b.data(), v.data(), b.size());
  return b;
}
int fails = 0;
#define CHECK(c)                                                 \
  do {                                                           \
    if (!(c)) {                                                  \
      std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++fails;                                                   \
    }                                                            \
  } while (0)

MicroBatch make_batch(int V, int S, int Lmax, unsigned seed, bool with_adv) {
  MicroBatch b;
  b.field_set = with_adv ? std::vector<std::string>{"advantage", "logp", "ref_logp", "response", "reward"}
                         : std::vector<std::string>{"logp", "ref_logp", "response", "reward"};
  unsigned x = seed;
  auto rnd = [&]() { x = x * 1664525u + 1013904223u; return x >> 8; };
  for (int i = 0; i < S; ++i) {
    const int L = 16 + static_cast<int>(rnd() % Lmax);
    std::vector<int32_t> resp(L);
    std::vector<float> lp(L), rl(L);
    for (int t = 0; t < L; ++t) {
      resp[t] = static_cast<int32_t>(rnd() % V);
      lp[t] = -1.f - (rnd() % 1000) * 1e-3f;
      rl[t] = lp[t] + ((rnd() % 200) - 100) * 1e-3f;
    }
    const float reward = (rnd() % 2) ? 1.f : 0.f, adv = ((rnd() % 200) - 100) * 1e-2f;
    b.sample_ids.push_back(static_cast<std::uint64_t>(i + 1));
    b.producer_versions.push_back(3 + (i % 2));
    b.global_steps.push_back(7);
    if (with_adv)
      b.payloads.push_back({enc(std::vector<float>{adv}), enc(lp), enc(rl), enc(resp), enc(std::vector<float>{reward})});
    else
      b.payloads.push_back({enc(lp), enc(rl), enc(resp), enc(std::vector<float>{reward})});
  }
  return b;
}

void test_pack() {
  MicroBatch b = make_batch(1000, 5, 40, 7, true);
  staleflow::train_math::PackedBatch p;
  std::string err;
  CHECK(staleflow::train_math::pack_trainer_batch(b, 0, p, &err) == SF_TM_OK);
  CHECK(p.B == 5 && p.has_advantage && !p.has_mask);
  int64_t T = 0;
  size_t off = 0;
  for (size_t i = 0; i < b.payloads.size(); ++i) {
    const Bytes& resp = b.payloads[i][3];
    const size_t L = resp.size() / 4;
    CHECK(p.seq_lens[i] == static_cast<int32_t>(L));
    CHECK(std::memcmp(p.targets.data() + off, resp.data(), resp.size()) == 0);
    CHECK(std::memcmp(p.logp.data() + off, b.payloads[i][1].data(), L * 4) == 0);
    CHECK(std::memcmp(&p.per_sample[i], b.payloads[i][0].data(), 4) == 0);
    off += L;
    T += static_cast<int64_t>(L);
  }
  CHECK(p.T == T && p.targets.size() == static_cast<size_t>(T));
  // rewards only: group ids from sample ids
  MicroBatch r = make_batch(1000, 8, 20, 9, false);
  CHECK(staleflow::train_math::pack_trainer_batch(r, 4, p, &err) == SF_TM_OK);
  CHECK(!p.has_advantage && p.group_ids.size() == 8 && p.group_ids[3] == 0 && p.group_ids[4] == 1);
  // ragged payload is rejected with ConfigError
  r.payloads[2][0].pop_back();
  CHECK(staleflow::train_math::pack_trainer_batch(r, 4, p, &err) == SF_TM_CONFIG_ERROR && !err.empty());
  r.field_set = {"logp", "response"};
  CHECK(staleflow::train_math::pack_trainer_batch(r, 4, p, &err) == SF_TM_CONFIG_ERROR);
  // staleness tags pass through: v_t - v_producer per sample, batch = v_t - min
  MicroBatch st = make_batch(1000, 6, 20, 3, true);
  CHECK(staleflow::train_math::pack_trainer_batch(st, 0, p, &err) == SF_TM_OK);
  int64_t bs = -1;
  auto hist = staleflow::train_math::staleness_histogram(p, 5, &bs);
  CHECK(bs == 2 && hist.size() == 2 && hist[2] == 3 && hist[1] == 3);
  // complete groups (H6): 8 samples in groups of 4 pass; dropping one fails
  MicroBatch g = make_batch(1000, 8, 20, 5, false);
  CHECK(staleflow::train_math::pack_trainer_batch(g, 4, p, &err) == SF_TM_OK);
  CHECK(staleflow::train_math::check_complete_groups(p, 4, &err) == SF_TM_OK);
  g.sample_ids.pop_back();
  g.payloads.pop_back();
  g.producer_versions.pop_back();
  g.global_steps.pop_back();
  CHECK(staleflow::train_math::pack_trainer_batch(g, 4, p, &err) == SF_TM_OK);
  CHECK(staleflow::train_math::check_complete_groups(p, 4, &err) == SF_TM_CONFIG_ERROR && !err.empty());
  // routed_experts: token-major (token, layer, slot) payloads -> layer-major [layers, T, k]
  {
    const int layers = 3, k = 2;
    MicroBatch rb;
    rb.field_set = {"response", "routed_experts"};
    const int lens[2] = {4, 5};
    for (int i = 0; i < 2; ++i) {
      rb.sample_ids.push_back(static_cast<std::uint64_t>(i + 1));
      rb.producer_versions.push_back(1);
      rb.global_steps.push_back(1);
      Bytes rec(static_cast<size_t>(lens[i]) * layers * k);
      for (int t = 0; t < lens[i]; ++t)
        for (int l = 0; l < layers; ++l)
          for (int j = 0; j < k; ++j) rec[(t * layers + l) * k + j] = static_cast<std::uint8_t>(100 * i + 10 * t + 3 * l + j);
      rb.payloads.push_back({enc(std::vector<int32_t>(lens[i], 7)), rec});
    }
    std::vector<uint8_t> lm;
    int64_t T = 0;
    CHECK(staleflow::train_math::pack_routed_experts(rb, layers, k, lm, &T, &err) == SF_TM_OK);
    CHECK(T == 9 && lm.size() == static_cast<size_t>(layers * T * k));
    bool ok = true;
    for (int l = 0; l < layers; ++l)
      for (int t = 0; t < 9; ++t)
        for (int j = 0; j < k; ++j) {
          const int i = t < 4 ? 0 : 1, tt = t < 4 ? t : t - 4;
          ok &= lm[(static_cast<size_t>(l) * T + t) * k + j] == static_cast<std::uint8_t>(100 * i + 10 * tt + 3 * l + j);
        }
    CHECK(ok);
    rb.payloads[1][1].pop_back();
    CHECK(staleflow::train_math::pack_routed_experts(rb, layers, k, lm, &T, &err) == SF_TM_CONFIG_ERROR);
  }
  std::printf(fails ? "PACK FAILED\n" : "PACK OK\n");
}

#ifdef SF_WITH_CUDA
void test_gpu() {
  const int V = 32000;
  MicroBatch b = make_batch(V, 16, 200, 11, false);
  staleflow::train_math::ActorLossSeam seam(0);
  CHECK(seam.status() == SF_TM_OK);
  staleflow::train_math::PackedBatch p;
  std::string err;
  staleflow::train_math::pack_trainer_batch(b, 4, p, &err);
  void *logits = nullptr, *dl1 = nullptr, *dl2 = nullptr;
  cudaMalloc(&logits, p.T * V * 2);
  cudaMalloc(&dl1, p.T * V * 2);
  cudaMalloc(&dl2, p.T * V * 2);
  CHECK(sf_tm_synth_logits(seam.handle(), logits, SF_TM_BF16, p.T, V, V, 5, 2.f, nullptr, 0.f, 0.f, 1e-3f, nullptr) == SF_TM_OK);
  sf_tm_loss_params prm;
  sf_tm_default_loss_params(&prm);
  float m1[SF_TM_NUM_METRICS], m2[SF_TM_NUM_METRICS];
  CHECK(seam.step(b, logits, SF_TM_BF16, V, dl1, prm, m1, nullptr, 4) == SF_TM_OK);
  cudaDeviceSynchronize();
  // reference path: the C-ABI seam call on the same packed host arrays
  CHECK(sf_tm_pg_step_host(seam.handle(), logits, SF_TM_BF16, p.T, V, V, p.targets.data(), p.logp.data(),
                           p.ref_logp.data(), nullptr, p.seq_lens.data(), nullptr, p.per_sample.data(),
                           p.group_ids.data(), p.B, 1e-6f, SF_TM_STD_UNBIASED, &prm, dl2, V, m2, nullptr) == SF_TM_OK);
  cudaDeviceSynchronize();
  CHECK(std::memcmp(m1, m2, sizeof(m1)) == 0);
  CHECK(m1[SF_TM_M_ACTIVE] == static_cast<float>(p.T));
  std::vector<unsigned char> h1(p.T * V * 2), h2(p.T * V * 2);
  cudaMemcpy(h1.data(), dl1, h1.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(h2.data(), dl2, h2.size(), cudaMemcpyDeviceToHost);
  CHECK(h1 == h2);
  cudaFree(logits);
  cudaFree(dl1);
  cudaFree(dl2);
  // back-to-back steps (no sync between them: the seam refills its pinned
  // staging only after the previous step's H2D has read it) == synced steps
  {
    const int nb = 4;
    std::vector<MicroBatch> bs;
    std::vector<int64_t> Ts;
    std::vector<void*> lg(nb), da(nb), db(nb);
    std::vector<std::vector<float>> ma(nb, std::vector<float>(SF_TM_NUM_METRICS)),
        mb(nb, std::vector<float>(SF_TM_NUM_METRICS));
    for (int i = 0; i < nb; ++i) {
      bs.push_back(make_batch(V, 8 + 4 * i, 120 + 60 * i, 21 + i, false));
      staleflow::train_math::PackedBatch q;
      staleflow::train_math::pack_trainer_batch(bs[i], 4, q, &err);
      Ts.push_back(q.T);
      cudaMalloc(&lg[i], q.T * V * 2);
      cudaMalloc(&da[i], q.T * V * 2);
      cudaMalloc(&db[i], q.T * V * 2);
      CHECK(sf_tm_synth_logits(seam.handle(), lg[i], SF_TM_BF16, q.T, V, V, 30 + i, 2.f, nullptr, 0.f, 0.f, 1e-3f,
                               nullptr) == SF_TM_OK);
    }
    for (int i = 0; i < nb; ++i) {
      CHECK(seam.step(bs[i], lg[i], SF_TM_BF16, V, da[i], prm, ma[i].data(), nullptr, 4) == SF_TM_OK);
      cudaDeviceSynchronize();
    }
    for (int i = 0; i < nb; ++i)
      CHECK(seam.step(bs[i], lg[i], SF_TM_BF16, V, db[i], prm, mb[i].data(), nullptr, 4) == SF_TM_OK);
    cudaDeviceSynchronize();
    for (int i = 0; i < nb; ++i) {
      CHECK(ma[i] == mb[i]);
      std::vector<unsigned char> ha(Ts[i] * V * 2), hb(Ts[i] * V * 2);
      cudaMemcpy(ha.data(), da[i], ha.size(), cudaMemcpyDeviceToHost);
      cudaMemcpy(hb.data(), db[i], hb.size(), cudaMemcpyDeviceToHost);
      CHECK(ha == hb);
      cudaFree(lg[i]);
      cudaFree(da[i]);
      cudaFree(db[i]);
    }
  }
  // routed_experts codec -> R3 gate: the replayed indices are the decoded record, bit for bit
  {
    const int layers = 4, k = 8, E = 128;
    MicroBatch rb;
    rb.field_set = {"response", "routed_experts"};
    unsigned x = 99;
    auto rnd = [&]() { x = x * 1664525u + 1013904223u; return x >> 8; };
    for (int i = 0; i < 5; ++i) {
      const int L = 20 + static_cast<int>(rnd() % 50);
      rb.sample_ids.push_back(static_cast<std::uint64_t>(i + 1));
      rb.producer_versions.push_back(1);
      rb.global_steps.push_back(1);
      Bytes rec(static_cast<size_t>(L) * layers * k);
      for (auto& v : rec) v = static_cast<std::uint8_t>(rnd() % E);
      rb.payloads.push_back({enc(std::vector<int32_t>(L, 1)), rec});
    }
    std::vector<uint8_t> lm;
    int64_t T = 0;
    CHECK(staleflow::train_math::pack_routed_experts(rb, layers, k, lm, &T, &err) == SF_TM_OK);
    void *z = nullptr, *rec_d = nullptr, *w = nullptr, *idx = nullptr;
    cudaMalloc(&z, static_cast<size_t>(layers) * T * E * 4);
    cudaMalloc(&rec_d, lm.size());
    cudaMalloc(&w, lm.size() * 4);
    cudaMalloc(&idx, lm.size() * 4);
    cudaMemcpy(rec_d, lm.data(), lm.size(), cudaMemcpyHostToDevice);
    CHECK(sf_tm_synth_logits(seam.handle(), z, SF_TM_F32, layers * T, E, E, 3, 2.f, nullptr, 0.f, 0.f, 0.f, nullptr) ==
          SF_TM_OK);
    CHECK(sf_tm_r3_gate_fwd(seam.handle(), z, SF_TM_F32, layers, T, E, k, rec_d, SF_TM_IDX_U8, 1,
                            static_cast<float*>(w), static_cast<int32_t*>(idx), nullptr, nullptr) == SF_TM_OK);
    std::vector<int32_t> got(lm.size());
    cudaMemcpy(got.data(), idx, got.size() * 4, cudaMemcpyDeviceToHost);
    bool same = true;
    for (size_t i = 0; i < lm.size(); ++i) same &= got[i] == static_cast<int32_t>(lm[i]);
    CHECK(same);
    cudaFree(z);
    cudaFree(rec_d);
    cudaFree(w);
    cudaFree(idx);
  }
  // stage producers: ActorFwd/RefLogP logp payloads and the Advantages stage
  {
    MicroBatch sb = make_batch(V, 6, 120, 21, false);  // fields logp, ref_logp, response, reward
    staleflow::train_math::PackedBatch sp;
    staleflow::train_math::pack_trainer_batch(sb, 3, sp, &err);
    void* lg = nullptr;
    cudaMalloc(&lg, sp.T * V * 2);
    staleflow::train_math::LogpStageSeam st(0);
    CHECK(sf_tm_synth_logits(st.handle(), lg, SF_TM_BF16, sp.T, V, V, 8, 2.f, nullptr, 0.f, 0.f, 1e-3f, nullptr) ==
          SF_TM_OK);
    std::vector<Bytes> lp_payloads;
    CHECK(st.run(sb, lg, SF_TM_BF16, V, 1.f, lp_payloads, nullptr) == SF_TM_OK);
    CHECK(lp_payloads.size() == 6);
    // same numbers as the device-buffer C-ABI call
    int32_t* dt = nullptr;
    float* dl = nullptr;
    cudaMalloc(&dt, sp.T * 4);
    cudaMalloc(&dl, sp.T * 4);
    cudaMemcpy(dt, sp.targets.data(), sp.T * 4, cudaMemcpyHostToDevice);
    CHECK(sf_tm_logprob_fwd(st.handle(), lg, SF_TM_BF16, sp.T, V, V, dt, 1.f, dl, nullptr, nullptr, nullptr) == SF_TM_OK);
    std::vector<float> ref(sp.T);
    cudaMemcpy(ref.data(), dl, sp.T * 4, cudaMemcpyDeviceToHost);
    size_t off = 0;
    bool same = true;
    for (size_t i = 0; i < lp_payloads.size(); ++i) {
      same &= lp_payloads[i].size() == static_cast<size_t>(sp.seq_lens[i]) * 4;
      same &= std::memcmp(lp_payloads[i].data(), ref.data() + off, lp_payloads[i].size()) == 0;
      off += sp.seq_lens[i];
    }
    CHECK(same);
    cudaFree(lg);
    cudaFree(dt);
    cudaFree(dl);
    staleflow::train_math::AdvantageStageSeam av(0);
    std::vector<Bytes> adv_payloads;
    CHECK(av.run(sb, 3, 1e-6f, SF_TM_STD_UNBIASED, adv_payloads, nullptr) == SF_TM_OK);
    bool ok = adv_payloads.size() == 6;
    for (int g = 0; g < 2 && ok; ++g) {
      double m = 0, v = 0;
      for (int j = 0; j < 3; ++j) m += sp.per_sample[3 * g + j];
      m /= 3;
      for (int j = 0; j < 3; ++j) v += (sp.per_sample[3 * g + j] - m) * (sp.per_sample[3 * g + j] - m);
      const double sd = std::sqrt(v / 2);
      for (int j = 0; j < 3; ++j) {
        float a;
        std::memcpy(&a, adv_payloads[3 * g + j].data(), 4);
        const double want = sd == 0 ? 0.0 : (sp.per_sample[3 * g + j] - m) / (sd + 1e-6);
        ok &= std::fabs(a - want) <= 1e-5 * (1 + std::fabs(want));
      }
    }
    CHECK(ok);
    CHECK(av.run(sb, 4, 1e-6f, SF_TM_STD_UNBIASED, adv_payloads, nullptr) == SF_TM_CONFIG_ERROR);  // 6 % 4: incomplete
  }
  std::printf(fails ? "GPU FAILED\n" : "GPU OK loss=%g active=%g\n", m1[0], m1[SF_TM_M_ACTIVE]);
}
#endif
}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "pack";
  if (mode == "pack") test_pack();
#ifdef SF_WITH_CUDA
  if (mode == "gpu") test_gpu();
#endif
  return fails ? 1 : 0;
}
