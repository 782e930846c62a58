// SPDX-License-Identifier: Apache-2.0
//
// The fused hot path (SURVEY.md §8 rows a1 + a4 + a2): per token, the vocab-wide
// log-softmax gather (logp, entropy), the DAPO/GRPO surrogate with optional KL
// and entropy bonus, and the dlogits backward — in ONE pass over HBM: each
// logits row is read once and its gradient written once (4V bytes per
// loss-active bf16 token).
//
// sm_100a structure (one CTA per SM, persistent, rows grid-strided; a row is
// split over a C-CTA cluster only when one CTA's slice would not fit the row
// store):
//
//   warp 24        TMA producer: cp.async.bulk 12 KB chunks of the row slice
//                  into an 8-slot smem ring (mbarrier complete_tx), L2
//                  evict-first, running ahead across rows.
//   warps 12..23   FORWARD: read a chunk (2 x LDS.128 per thread), copy it into
//                  the ROW STORE, release the ring slot, and fold it into the
//                  online softmax state (fixed per-thread exponent base, packed
//                  FFMA2/FADD2, MUFU.EX2). Row end: warp merge, per-warp partial
//                  into a flow-controlled smem ring.
//   warps 25..27   CONTROL (rotating rows): merge the 12 partials, exchange
//                  them with the cluster (DSMEM mailboxes) or, in the XP
//                  instantiation, with the other GPUs (peer-memory mailboxes;
//                  then warp 25 sends and warps 26, 27 receive), compute the loss
//                  scalars once, publish them to the backward warps; metrics
//                  accumulate in fp64.
//   warps 0..11    BACKWARD: wait for the row's scalars, re-read the row from
//                  the row store, form dlogits (bf16: |c0| folded into the
//                  exponent, the sign XOR-ed onto packed words), 16-B streaming
//                  stores.
//
// The row store is TMEM (21 slots of 24 columns, tcgen05.st/ld.32x32b.x8)
// followed by 10 smem slots: 31 x 12 KB, a whole Qwen3 bf16 row (25 chunks) and
// part of the next, so forward(r+1) overlaps backward(r) and every row is read
// from HBM exactly once. Each backward warp reads exactly the TMEM lanes/columns
// its partner forward warp (same SM sub-partition) wrote. Every slot is
// released only after the values read from it fed a dependent instruction
// (SASS issues an mbarrier arrive right behind an LDS without waiting for it).
//
// Narrow rows (a vocab-parallel shard) run NS = 2 or 4 ROW STREAMS: the warp
// pairs split into NS groups, consecutive loss-active rows go to the groups in
// turn, and each ring / row-store slot carries one sub-chunk of every group's
// row, so the per-row work is paid NS times less often per SM (see the kernel
// comment; the control warps then hand rows off strictly in row order). Rows
// are found 32 at a time by a ballot over their weights, and the control warps
// hold a 32-row window of per-row inputs, one row per lane.
//
// Reference seam replaced: trainer_compute_batch latency (proj/src/sim_runtime.cpp:441)
// and trainer_thread sleep (proj/src/wall_runtime.cpp:197); math pinned in
// DESIGN.md §2, fp64 twin oracle/sf_oracle.c orc_pg_loss_fwd_bwd.

#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "tm_rowmath.cuh"

namespace sftm {

namespace loss {

#ifndef SFTM_DBG_MODE
#define SFTM_DBG_MODE 0
#endif

#ifndef SFTM_FW
#define SFTM_FW 12
#endif
constexpr int kFW = SFTM_FW;                // forward warps (3 per SM sub-partition)
constexpr int kBW = SFTM_FW;                // backward warps (3 per SM sub-partition)
static_assert(kFW % 4 == 0, "forward / backward warps come in SM sub-partition quads");
constexpr int kFT = kFW * 32;               // 384 forward threads
constexpr int kProd = kFW + kBW;            // producer warp index
constexpr int kCtl = kFW + kBW + 1;         // control warps (2, alternating rows): merge, exchange, scalars
#ifndef SFTM_NCTL
#define SFTM_NCTL 3
#endif
constexpr int kNCtl = SFTM_NCTL;
constexpr int kThreads = (kFW + kBW + 1 + kNCtl) * 32;  // 896
static_assert(kNCtl >= 2, "the peer exchange needs a sender and at least one receiver warp");
constexpr int kCB = kFT * 32;               // chunk bytes: two 16-B vectors per thread = 12 KB
#ifndef SFTM_RING_SLOTS
#define SFTM_RING_SLOTS 8
#endif
constexpr int kSlots = SFTM_RING_SLOTS;     // TMA landing ring slots (96 KB)
constexpr int kSSlots = (216 * 1024) / kCB - kSlots;  // shared-memory row-store slots (120 KB)
constexpr int kRingBytes = (kSlots + kSSlots) * kCB;  // dynamic smem: ring + smem row store
constexpr int kSlotCols = kCB / (128 * 4);  // TMEM columns per chunk slot (24)
constexpr int kTSlots = 512 / kSlotCols;    // 21 TMEM chunk slots (252 KB)
constexpr int kStore = kTSlots + kSSlots;   // row-store slots: TMEM first, then smem (31)
constexpr int kTCols = 512;
#ifndef SFTM_RD
#define SFTM_RD 4
#endif
constexpr int kRD = SFTM_RD;                      // depth of the per-row partial / scalar rings (flow-controlled)
// Mailbox ring depth (rows). Not flow-controlled across the cluster: with the
// red/scal rings bounded, a CTA's control warp is at most 2*kRD+1 rows ahead
// of its partner's mailbox reads, so 16 can never be overrun.
constexpr int kMailD = 16;
// XP sender credit: the sender posts row n only after its receiver finished
// row n - kXpCredit. Then a rank posting row n into a peer's slot n % kXpMailD
// implies that peer's receiver finished row n - 2*kXpCredit >= n - kXpMailD.
#ifndef SFTM_XP_CREDIT
#define SFTM_XP_CREDIT 6
#endif
constexpr int kXpCredit = SFTM_XP_CREDIT;
constexpr int kCredD = kXpCredit + 2;
static_assert(2 * kXpCredit <= kXpMailD && kXpCredit < kCredD, "credit bounds");

// Per-row scalars computed once by the control warp and broadcast in smem.
struct RowScal {
  float lse2, lse2f, c0, c1, gt;
  int tck;         // chunk holding the target column in this CTA's slice, or -1
  uint32_t sgn;    // 0x80008000 when dlogits entries are -p*|c0| (bf16 fast path)
  uint32_t town;   // (thread owning the target << 8) | its element index j
};
constexpr int kMaxChunks = kStore - 2;      // a whole row slice must fit the row store

template <typename T>
struct Geo {
  static constexpr int es = sizeof(T);
  static constexpr int CE = kCB / es;       // elements per chunk
  static constexpr int HALF = CE / 2;       // second 16-B vector of a thread starts here
  static constexpr int EV = 16 / es;        // elements per 16-B vector
  static constexpr int NE = 2 * EV;         // elements per thread per chunk
};

// 8 words (two 16-B vectors) -> NE floats
__device__ __forceinline__ void unpack(const float*, uint4 a, uint4 b, float (&x)[8]) {
  x[0] = __uint_as_float(a.x); x[1] = __uint_as_float(a.y);
  x[2] = __uint_as_float(a.z); x[3] = __uint_as_float(a.w);
  x[4] = __uint_as_float(b.x); x[5] = __uint_as_float(b.y);
  x[6] = __uint_as_float(b.z); x[7] = __uint_as_float(b.w);
}
__device__ __forceinline__ void unpack(const uint16_t*, uint4 a, uint4 b, float (&x)[16]) {
  x[0] = bf16lo(a.x); x[1] = bf16hi(a.x); x[2] = bf16lo(a.y); x[3] = bf16hi(a.y);
  x[4] = bf16lo(a.z); x[5] = bf16hi(a.z); x[6] = bf16lo(a.w); x[7] = bf16hi(a.w);
  x[8] = bf16lo(b.x); x[9] = bf16hi(b.x); x[10] = bf16lo(b.y); x[11] = bf16hi(b.y);
  x[12] = bf16lo(b.z); x[13] = bf16hi(b.z); x[14] = bf16lo(b.w); x[15] = bf16hi(b.w);
}

// Element offset (within a chunk) of a thread's j-th element.
template <typename T>
__device__ __forceinline__ int elem_off(int tid, int j) {
  using G = Geo<T>;
  return (j < G::EV) ? (G::EV * tid + j) : (G::HALF + G::EV * tid + (j - G::EV));
}

// Online update with N elements; no clamp: a -inf logit makes w NaN, which the
// caller repairs on a slow path (logits from an LM head are finite).
template <int N>
__device__ __forceinline__ void accum(Stats& st, const float (&x)[N], float c) {
  float xm = x[0];
#pragma unroll
  for (int j = 1; j < N; ++j) xm = fmaxf(xm, x[j]);
  const float cm = xm * c;
  if (cm > st.m2) {
    if (st.m2 != -INFINITY) {
      const float d = st.m2 - cm;
      const float f = ex2(d);
      st.w = f * fmaf(st.s, d, st.w);
      st.s *= f;
    }
    st.m2 = cm;
  }
  float s[4] = {0.f, 0.f, 0.f, 0.f}, w[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const float a = fmaf(x[j], c, -st.m2);
    const float e = ex2(a);
    s[j & 3] += e;
    w[j & 3] = fmaf(e, a, w[j & 3]);
  }
  st.s += (s[0] + s[1]) + (s[2] + s[3]);
  st.w += (w[0] + w[1]) + (w[2] + w[3]);
}

// Careful (slow) variant: masked elements and -inf logits contribute nothing.
template <int N>
__device__ __forceinline__ void accum_masked(Stats& st, const float (&x)[N], const bool (&ok)[N],
                                             float c) {
  float xm = -INFINITY;
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (ok[j]) xm = fmaxf(xm, x[j]);
  const float cm = xm * c;
  if (cm > st.m2) {
    if (st.m2 != -INFINITY) {
      const float d = st.m2 - cm;
      const float f = ex2(d);
      st.w = f * fmaf(st.s, d, st.w);
      st.s *= f;
    }
    st.m2 = cm;
  }
#pragma unroll
  for (int j = 0; j < N; ++j) {
    if (ok[j] && x[j] != -INFINITY) {
      const float a = fmaf(x[j], c, -st.m2);
      const float e = ex2(a);
      st.s += e;
      st.w = fmaf(e, a, st.w);
    }
  }
}

__device__ __forceinline__ void store_vec(float* p, const float* g) {
  stg128_cs(p, make_uint4(__float_as_uint(g[0]), __float_as_uint(g[1]), __float_as_uint(g[2]),
                          __float_as_uint(g[3])));
}
__device__ __forceinline__ void store_vec(uint16_t* p, const float* g) {
  stg128_cs(p, make_uint4(pack_bf16x2(g[0], g[1]), pack_bf16x2(g[2], g[3]),
                          pack_bf16x2(g[4], g[5]), pack_bf16x2(g[6], g[7])));
}

// Debug wait instrumentation: DBG_WAIT(counter, wait-expression). Compiled in
// only with -DSFTM_WAIT_PROFILE (scripts/wait_profile.py); otherwise free.
#ifndef SFTM_WAIT_PROFILE
#define DBG_WAIT(ctr, expr) expr
#else
#define DBG_WAIT(ctr, expr)                         \
  do {                                              \
    if (dbg) {                                      \
      const long long t0_ = clock64();              \
      expr;                                         \
      ctr += static_cast<unsigned long long>(clock64() - t0_); \
    } else {                                        \
      expr;                                         \
    }                                               \
  } while (0)
#endif

// XP (C == 1 only): vocab-parallel across GPUs. Each rank runs this kernel on
// its vocab shard with the same grid and row schedule; CTA i of every rank
// handles the same rows, and the control warps exchange the per-row partial
// statistics through peer-mapped global-memory mailboxes (NVLink P2P stores,
// system-scope release/acquire) instead of DSMEM. The shard is read once.
// UA (C == 1 only): rows need not start on a 16-B boundary (odd vocabularies,
// odd row strides). Each row is then handled in "sector coordinates": the TMA
// copies start at the row's 16-B-aligned-down address, so the row begins `mis`
// elements into chunk 0; chunk 0 and the tail chunk are masked per element and
// the boundary dlogits vectors are stored per element. Reads extend to whole
// 16-B sectors inside the tensor; the very last row's tail sector is filled by
// the producer with element loads instead, so nothing past the tensor is read.
// NS (C == 1, aligned rows): row streams. The 12 forward / backward warp pairs
// split into NS groups of 12/NS pairs; consecutive loss-active rows of the CTA
// go to the streams in turn, and every ring / row-store slot carries one
// 12/NS-KB sub-chunk of each stream's row (the producer fills it with NS bulk
// copies). A warp then handles only every NS-th row, so the per-row work of
// the compute warps (row-end merge, chunk-0 base, tail chunk, scalar
// hand-off) is spent 1/NS as often per SM — what bounds narrow rows (a
// vocab-parallel shard at P = 4 / 8). Streams advance in lockstep: the NS rows
// of a group have the same width, and a stream with no row in the CTA's last
// group idles through its steps.
// A control warp's per-row inputs, one row per lane of a 32-row window of the
// CTA's rows (rows cid + (32 * win + lane) * ncl); loaded a window ahead, a
// row's inputs are then one shuffle away instead of a dependent load per row.
struct RowIn {
  float w, A, old, ref;
  int32_t y;
};
__device__ __forceinline__ RowIn load_row_in(const RowArgs& a, int64_t cid, int64_t ncl, int64_t win, int lane) {
  RowIn r{0.f, 0.f, 0.f, 0.f, 0};
  const int64_t t = cid + (32 * win + lane) * ncl;
  if (t < a.T) {
    r.w = __ldg(a.w_tok + t);
    r.A = __ldg(a.adv_tok + t);
    r.old = __ldg(a.old_logp + t);
    r.ref = __ldg(a.ref_logp + t);
    r.y = __ldg(a.targets + t);
  }
  return r;
}
// masked rows get logp = entropy = 0 (each lane its own row of the window)
__device__ __forceinline__ void zero_masked_outputs(const RowArgs& a, int64_t t, float w) {
  if (t < a.T && w == 0.f) {
    if (a.out_logp) a.out_logp[t] = 0.f;
    if (a.out_entropy) a.out_entropy[t] = 0.f;
  }
}

// Warp-collective walk over a CTA's rows t = cid + n * ncl (n = 0, 1, ...)
// yielding the loss-active ones (w_tok != 0): 32 rows per ballot over their
// weights, the next window's weights loaded one window ahead, so finding the
// next active row costs no dependent global load. Every lane gets the same rows.
struct RowWalk {
  const float* w;
  int64_t T, cid, ncl, win;
  uint32_t act;  // active rows of the current window not yet returned
  uint32_t msk;  // masked rows (w == 0) of the current window not yet returned (next_all)
  float wnext;   // this lane's row weight in the next window
  int lane;
  __device__ __forceinline__ bool exists(int64_t wi) const { return cid + (32 * wi + lane) * ncl < T; }
  __device__ __forceinline__ float load(int64_t wi) const {
    const int64_t t = cid + (32 * wi + lane) * ncl;
    return t < T ? __ldg(w + t) : 0.f;
  }
  __device__ __forceinline__ void init(const float* w_, int64_t T_, int64_t cid_, int64_t ncl_, int lane_) {
    w = w_;
    T = T_;
    cid = cid_;
    ncl = ncl_;
    lane = lane_;
    win = 0;
    const float w0 = load(0);
    act = __ballot_sync(0xffffffffu, w0 != 0.f);
    msk = __ballot_sync(0xffffffffu, exists(0) && w0 == 0.f);
    wnext = load(1);
  }
  __device__ __forceinline__ bool advance() {
    if (cid + 32 * (win + 1) * ncl >= T) return false;
    ++win;
    act = __ballot_sync(0xffffffffu, wnext != 0.f);
    msk = __ballot_sync(0xffffffffu, exists(win) && wnext == 0.f);
    wnext = load(win + 1);
    return true;
  }
  // every row in order, loss-active or not (the backward zero-fills masked rows)
  __device__ __forceinline__ bool next_all(int64_t& t, bool& active) {
    while ((act | msk) == 0u)
      if (!advance()) return false;
    const int i = __ffs(act | msk) - 1;
    active = (act >> i) & 1u;
    act &= ~(1u << i);
    msk &= ~(1u << i);
    t = cid + (32 * win + i) * ncl;
    return true;
  }
  __device__ __forceinline__ bool next(int64_t& t) {
    while (act == 0u)
      if (!advance()) return false;
    const int i = __ffs(act) - 1;
    act &= act - 1u;
    t = cid + (32 * win + i) * ncl;
    return true;
  }
};

// The loss-active rows of a CTA in order (and, with next_all, the masked
// ones too). Row streams (NS > 1) skip most rows, so they find them with the
// ballot walk; one row at a time (NS == 1), the next row's weight loaded a row
// ahead by each thread is as fast and measured cheaper at wide rows.
template <int NS>
struct RowSeq {
  RowWalk rw;
  const float* w;
  int64_t T, ncl, t;
  float wn;
  __device__ __forceinline__ void init(const float* w_, int64_t T_, int64_t cid, int64_t ncl_, int lane) {
    if constexpr (NS > 1) {
      rw.init(w_, T_, cid, ncl_, lane);
    } else {
      w = w_;
      T = T_;
      ncl = ncl_;
      t = cid - ncl_;
      wn = (cid < T_) ? __ldg(w_ + cid) : 0.f;
    }
  }
  __device__ __forceinline__ bool next_all(int64_t& row, bool& active) {
    if constexpr (NS > 1) {
      return rw.next_all(row, active);
    } else {
      t += ncl;
      if (t >= T) return false;
      active = wn != 0.f;
      if (t + ncl < T) wn = __ldg(w + t + ncl);
      row = t;
      return true;
    }
  }
  __device__ __forceinline__ bool next(int64_t& row) {
    if constexpr (NS > 1) {
      return rw.next(row);
    } else {
      bool active = false;
      while (next_all(row, active))
        if (active) return true;
      return false;
    }
  }
};

#ifdef SFTM_HANG_DEBUG
// Debug build only (EXTRA=-DSFTM_HANG_DEBUG, scripts/hang_debug.py): a wait that
// gives up after 2 s and records where, so a protocol deadlock shows its
// waiting sites instead of hanging the GPU. Records (host-mapped memory, so
// they survive a fault): line | parity << 16 | rank << 20 | row << 24 |
// CTA << 40 | warp << 56; dbg[0] the first give-up, dbg[16 + (rank * 148 +
// CTA) * 32 + warp] each warp's first; dbg[15] the abort flag (later waits give
// up at once). `row` is the warp's active-row counter (dbg_row).
__device__ __forceinline__ void kwait(unsigned long long* dbg, int line, uint32_t bar, uint32_t par, int rank,
                                      uint32_t row) {
  if (mbar_try_wait(bar, par)) return;
  volatile unsigned long long* vd = dbg;  // host-mapped (pinned) memory: readable after a fault
  const uint64_t t0 = globaltimer_ns();
  while (!mbar_try_wait(bar, par)) {
    if (vd[15] != 0ull || globaltimer_ns() - t0 > 2000000000ull) {
      const unsigned long long rec = static_cast<unsigned long long>(line) | (static_cast<unsigned long long>(par) << 16) |
                                     (static_cast<unsigned long long>(rank & 15) << 20) |
                                     (static_cast<unsigned long long>(row & 0xffffu) << 24) |
                                     (static_cast<unsigned long long>(blockIdx.x & 0xffu) << 40) |
                                     (static_cast<unsigned long long>(threadIdx.x >> 5) << 56);
      const size_t i = 16 + (static_cast<size_t>(rank & 7) * 148 + blockIdx.x) * 32 + (threadIdx.x >> 5);
      if (vd[i] == 0ull) vd[i] = rec;
      if (vd[15] == 0ull) vd[0] = rec;
      vd[15] = 1ull;
      __threadfence_system();
      return;
    }
  }
}
#define KWAIT(bar, par) kwait(a.dbg, __LINE__, bar, par, a.xp_rank, dbg_row)
#define DBG_ROW(n) (dbg_row = (n))
#else
#define KWAIT(bar, par) mbar_wait(bar, par)
#define DBG_ROW(n) ((void)0)
#endif

template <typename T, int C, bool XP = false, bool UA = false, int NS = 1>
__global__ void __launch_bounds__(kThreads, 1)
    loss_tmem_kernel(const RowArgs a, int64_t slice_elems) {
  // pipeline-ceiling experiments only (build with EXTRA=-DSFTM_DBG_MODE=n): 1 = no
  // forward math, 2 = backward stores the raw words, 4 = ... and no dlogits
  // stores, 8 = no TMEM traffic. Compile-time, so the product build carries none of it.
  constexpr int dbg_mode = SFTM_DBG_MODE;
  static_assert(!XP || C == 1, "peer exchange runs one CTA per row per rank");
  static_assert(!UA || C == 1, "unaligned rows run one CTA per row");
  static_assert(NS == 1 || C == 1, "row streams: one CTA per row slice");
  static_assert(NS == 1 || NS == 2 || NS == 4, "row streams");
  using G = Geo<T>;
  constexpr int CE = G::CE;
  constexpr int NE = G::NE;
  constexpr int EV = G::EV;
  constexpr int SW = kFW / NS;       // warp pairs per row stream
  constexpr int SCE = CE / NS;       // elements of one stream's sub-chunk of a slot
  constexpr int SCB = kCB / NS;      // ... and its bytes
  constexpr int SHALF = SCE / 2;     // a thread's second vector starts here (sub-chunk coordinates)
  constexpr int RD = (2 * NS > kRD) ? 2 * NS : kRD;  // per-row rings hold two groups of rows

  extern __shared__ __align__(1024) uint8_t ring[];
  __shared__ __align__(8) uint64_t full_bar[kSlots];
  __shared__ __align__(8) uint64_t empty_bar[kSlots];
  __shared__ __align__(8) uint64_t tfull_bar[kStore];
  __shared__ __align__(8) uint64_t tempty_bar[kStore];
  constexpr int kMB = (C > 1) ? kMailD : 1;  // cluster mailboxes (C == 1 exchanges nothing in smem)
  __shared__ __align__(8) uint64_t mail_bar[kMB];
  __shared__ __align__(16) float4 mail[kMB][8];
  __shared__ __align__(16) float4 red[RD][SW];       // per forward warp of the row's stream: (m2, s, w, -)
  __shared__ __align__(8) uint64_t red_bar[RD], red_free[RD];
  __shared__ __align__(16) RowScal scal[RD];
  __shared__ __align__(8) uint64_t scal_bar[RD], scal_free[RD];
  __shared__ __align__(8) uint64_t rcv_done[kCredD];  // XP: receiver progress (sender credit)
  __shared__ uint32_t tmem_base_sh;
  __shared__ uint32_t sink_sh[kBW];

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
#ifdef SFTM_HANG_DEBUG
  uint32_t dbg_row = 0;
#endif
  const uint32_t crank = (C > 1) ? cluster_ctarank() : 0u;
  const int64_t cid = (C > 1) ? static_cast<int64_t>(cluster_id_x()) : blockIdx.x;
  const int64_t ncl = (C > 1) ? static_cast<int64_t>(nclusters_x()) : gridDim.x;
  const int64_t slice_start = static_cast<int64_t>(crank) * slice_elems;
  int64_t sl64 = a.V - slice_start;
  if (sl64 > slice_elems) sl64 = slice_elems;
  if (sl64 < 0) sl64 = 0;
  const int slice_len = static_cast<int>(sl64);
  const int nck = (slice_len + SCE - 1) / SCE;
  const int nfull = slice_len / SCE;
  // slot steps per group of rows: unaligned rows start up to EV - 1 elements
  // into their first sub-chunk, so a group takes the most any row can need and
  // a row with fewer chunks idles the rest
  const int nstep = UA ? (slice_len + EV - 1 + SCE - 1) / SCE : nck;
  const uint32_t ring_base = smem_u32(ring);
  const uint32_t stash_base = ring_base + kSlots * kCB;  // smem row-store slot i = store slot kTSlots + i

  if (tid == 0) {
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(smem_u32(&full_bar[i]), 1);
      mbar_init(smem_u32(&empty_bar[i]), kFT);  // every forward thread arrives
    }
    for (int i = 0; i < kStore; ++i) {
      mbar_init(smem_u32(&tfull_bar[i]), kFT);
      mbar_init(smem_u32(&tempty_bar[i]), kFT);  // backward threads (same count)
    }
    for (int i = 0; i < kMB; ++i) mbar_init(smem_u32(&mail_bar[i]), C);
    for (int i = 0; i < RD; ++i) {
      mbar_init(smem_u32(&red_bar[i]), SW);   // lane 0 of each forward warp of the row's stream
      mbar_init(smem_u32(&red_free[i]), 1);   // lane 0 of the control warp that read it
      mbar_init(smem_u32(&scal_bar[i]), 1);   // lane 0 of the control warp that wrote it
      mbar_init(smem_u32(&scal_free[i]), SW);  // lane 0 of each backward warp of the row's stream
    }
    for (int i = 0; i < kCredD; ++i) mbar_init(smem_u32(&rcv_done[i]), 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(smem_u32(&tmem_base_sh), kTCols);
  tc_fence_before();
  if (C > 1) {
    cluster_sync_all();
  } else {
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tbase = tmem_base_sh;
  const T* logits = static_cast<const T*>(a.logits);
#ifdef SFTM_WAIT_PROFILE
  unsigned long long* const dbg = a.dbg;
#else
  unsigned long long* const dbg = nullptr;
#endif
  unsigned long long w_a = 0, w_b = 0;  // per-role wait cycles (debug)
  const long long t_role0 = dbg ? clock64() : 0;
  // elements between a row slice's start and its 16-B sector start (UA only)
  auto row_mis = [&](int64_t t) -> int {
    if constexpr (UA) {
      return static_cast<int>((reinterpret_cast<uintptr_t>(logits + t * a.ld + slice_start) & 15u) / G::es);
    } else {
      (void)t;
      return 0;
    }
  };
  // A partial chunk (the front / tail of a row slice) may hold no element of a
  // whole warp's share (a narrow vocab-parallel shard row ends a few vectors
  // into its last chunk). Such a warp keeps the barrier protocol (waits and
  // arrives, so every phase count stays exact) but skips the loads, the row
  // store and the math. The test is warp-uniform and the forward warp and its
  // backward partner (same element mapping) take the same decision.
  auto warp_idle = [&](int k, bool partial, int mis, int span, int wbase) -> bool {
    if (!partial) return false;
    const int rem = span - k * SCE, lo = (UA && k == 0) ? mis : 0;
    const int a0 = EV * wbase, a1 = EV * (wbase + 32);  // the warp's first-vector block
    const int b0 = SHALF + a0, b1 = SHALF + a1;         // ... and second-vector block
    return !(a0 < rem && a1 > lo) && !(b0 < rem && b1 > lo);
  };
  // where the backward finds the target column (computed once per row by the
  // control warp): chunk, owning thread and its element index
  auto target_slot = [&](int64_t yl64, int mis, int& tck, uint32_t& town) {
    tck = -1;
    town = 0;
    if (yl64 >= 0 && yl64 < slice_len) {
      const int yp = static_cast<int>(yl64) + mis;  // sector coordinates
      const int r = yp % SCE;
      const int v = r >= SHALF ? 1 : 0;
      const int rr = r - v * SHALF;
      tck = yp / SCE;
      town = (static_cast<uint32_t>(rr / EV) << 8) | static_cast<uint32_t>(v * EV + rr % EV);
    }
  };

  if (warp == kProd) {
    // ================================================================ producer
    if (NS > 1) {
      // Row streams: a group of up to NS loss-active rows, one per stream;
      // slot step k carries sub-chunk k of every row of the group, copied by
      // lane g for stream g. The whole warp runs the loop: loss-active rows
      // are found 32 at a time by a ballot over their weights (loaded one
      // window ahead), and the NS copies of a step share one call site. With
      // a lane-0 loop and one row weight per iteration (one dependent load per
      // row) and a 64-bit address setup per copy, the producer needed ~120
      // instructions per step at ~0.1 IPC and starved 4 streams.
      const uint64_t pol = l2_evict_first_policy();
      uint32_t slot = 0, ph = 0;
      RowWalk rw;
      rw.init(a.w_tok, a.T, cid, ncl, lane);
      const T* my_row = nullptr;  // lane g < NS: stream g's row of the current group (sector start if UA)
      int my_span = 0;            // ... its extent in sector coordinates
      int64_t my_t = -1;
      int ng = 0;
      auto issue_group = [&]() {
        for (int k = 0; k < nstep; ++k) {
          const int rem = my_span - k * SCE;
          uint32_t bytes = (lane < ng && rem > 0) ? static_cast<uint32_t>(rem < SCE ? rem : SCE) * G::es : 0u;
          int tail = 0;  // UA: elements of the tensor's final partial sector, loaded by this lane
          if constexpr (UA) {
            if ((bytes & 15u) && my_t == a.T - 1 && rem <= SCE) {
              tail = static_cast<int>((bytes & 15u) / G::es);  // never read past the tensor
              bytes &= ~15u;
            } else {
              bytes = (bytes + 15u) & ~15u;  // whole sectors (inside the tensor)
            }
          }
          const uint32_t total = __reduce_add_sync(0xffffffffu, bytes);  // the step's TMA bytes
          DBG_WAIT(w_a, KWAIT(smem_u32(&empty_bar[slot]), ph ^ 1u));
          if constexpr (UA) {
            if (tail) {
              const T* tp = my_row + static_cast<int64_t>(k) * SCE + bytes / G::es;
              T* ts_ = reinterpret_cast<T*>(ring + slot * kCB + lane * SCB + bytes);
              for (int j = 0; j < tail; ++j) ts_[j] = tp[j];
              __threadfence_block();  // ordered before lane 0's release arrive (after the warp sync)
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive_expect_tx(smem_u32(&full_bar[slot]), total);
          __syncwarp();
          if (bytes)
            bulk_g2s(ring_base + slot * kCB + lane * SCB, my_row + static_cast<int64_t>(k) * SCE, bytes,
                     smem_u32(&full_bar[slot]), pol);
          if (++slot == kSlots) {
            slot = 0;
            ph ^= 1u;
          }
        }
      };
      int64_t t;
      while (rw.next(t)) {
        if (lane == ng) {
          const int mis = row_mis(t);
          my_row = logits + t * a.ld + slice_start - mis;
          my_span = slice_len + mis;
          my_t = t;
        }
        if (++ng == NS) {
          issue_group();
          ng = 0;
        }
      }
      if (ng > 0) {
        if (lane >= ng) my_span = 0;  // streams with no row in the last group
        issue_group();
      }
    } else if (lane == 0) {
      // one row at a time (one copy per step): lane 0 alone, the next row's
      // weight loaded a row ahead (measured faster than the warp-wide walk here)
      const uint64_t pol = l2_evict_first_policy();
      uint32_t slot = 0, ph = 0;
      float wn = (cid < a.T) ? __ldg(a.w_tok + cid) : 0.f;
      for (int64_t t = cid; t < a.T; t += ncl) {
        const float wcur = wn;
        if (t + ncl < a.T) wn = __ldg(a.w_tok + t + ncl);
        if (wcur == 0.f) continue;
        const int mis = row_mis(t);
        const int span = slice_len + mis;
        const int nck_r = UA ? (span + SCE - 1) / SCE : nck;
        const T* row = logits + t * a.ld + slice_start - mis;
        for (int k = 0; k < nck_r; ++k) {
          const int rem = span - k * SCE;
          uint32_t bytes = static_cast<uint32_t>(rem < CE ? rem : CE) * G::es;
          int tail = 0;  // UA: elements of a final partial sector loaded by this lane
          if constexpr (UA) {
            if ((bytes & 15u) && t == a.T - 1 && k == nck_r - 1) {
              tail = static_cast<int>((bytes & 15u) / G::es);  // never read past the tensor
              bytes &= ~15u;
            } else {
              bytes = (bytes + 15u) & ~15u;  // whole sectors (inside the tensor)
            }
          }
          DBG_WAIT(w_a, KWAIT(smem_u32(&empty_bar[slot]), ph ^ 1u));
          if constexpr (UA) {
            const T* tp = row + static_cast<int64_t>(k) * CE + bytes / G::es;
            uint8_t* ts_ = ring + slot * kCB + bytes;
            for (int j = 0; j < tail; ++j) reinterpret_cast<T*>(ts_)[j] = tp[j];
          }
          mbar_arrive_expect_tx(smem_u32(&full_bar[slot]), bytes);  // release: orders the tail stores
          if (bytes)
            bulk_g2s(ring_base + slot * kCB, row + static_cast<int64_t>(k) * CE, bytes,
                     smem_u32(&full_bar[slot]), pol);
          if (++slot == kSlots) {
            slot = 0;
            ph ^= 1u;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp >= kBW && warp < kBW + kFW) {
    // ================================================================ forward
    // Forward warps take the higher warp ids: the SM sub-partition arbiter
    // issues the highest eligible warp id first, and the forward is the
    // critical path (its row statistics gate the backward).
    const int fw = warp - kBW;                 // 0..kFW-1
    const int ftid = tid - kBW * 32;           // 0..kFT-1
    const int sg = fw / SW;                    // row stream
    const int sid = ftid - sg * (SW * 32);     // thread index within the stream
    const uint32_t tlane = static_cast<uint32_t>(32 * (fw & 3)) << 16;
    const uint32_t tcol = 8u * static_cast<uint32_t>(fw >> 2);  // 8 columns per warp of a sub-partition
    const float c = a.inv_tau * kLog2e;
    const uint32_t full0 = smem_u32(&full_bar[0]), empty0 = smem_u32(&empty_bar[0]);
    const uint32_t tfull0 = smem_u32(&tfull_bar[0]), tempty0 = smem_u32(&tempty_bar[0]);
    const uint32_t ring_t = ring_base + static_cast<uint32_t>(sg * SCB) + 16u * sid;
    const uint32_t stash_t = stash_base + 16u * ftid;
    const uint32_t tm_t = tbase + tlane + tcol;
    // row-store read-back (repair path)
    auto load_store = [&](uint32_t q, uint4& v0r, uint4& v1r) {
      if (q < static_cast<uint32_t>(kTSlots)) {
        tmem_ld8(tm_t + q * static_cast<uint32_t>(kSlotCols), v0r, v1r);
        tmem_wait_ld(v0r, v1r);
      } else {
        v0r = lds128(stash_t + (q - kTSlots) * kCB);
        v1r = lds128(stash_t + (q - kTSlots) * kCB + kCB / 2);
      }
    };
    uint32_t slot = 0, ph = 0, ts = 0, tph = 0, nrow = 0;
    // a thread's j-th element within its stream's sub-chunk
    auto eoff = [&](int j) { return (j < EV) ? (EV * sid + j) : (SHALF + EV * sid + (j - EV)); };
    // one slot step with nothing of this warp in it: keep the barrier protocol
    auto fidle = [&]() {
      DBG_WAIT(w_a, KWAIT(full0 + 8u * slot, ph));
      mbar_arrive(empty0 + 8u * slot);  // nothing read from the slot
      if (++slot == kSlots) {
        slot = 0;
        ph ^= 1u;
      }
      DBG_WAIT(w_b, KWAIT(tempty0 + 8u * ts, tph ^ 1u));
      mbar_arrive(tfull0 + 8u * ts);  // nothing written to the row-store slot
      if (++ts == kStore) {
        ts = 0;
        tph ^= 1u;
      }
    };
    RowSeq<NS> rows;
    rows.init(a.w_tok, a.T, cid, ncl, lane);
    int64_t t;
    while (rows.next(t)) {
      if (NS > 1 && static_cast<int>(nrow % NS) != sg) {  // another stream's row
        ++nrow;
        DBG_ROW(nrow);
        continue;
      }
      const int mis = row_mis(t);
      const int span = slice_len + mis;  // row extent in sector coordinates
      const int nck_r = UA ? (span + SCE - 1) / SCE : nck;
      float m2 = 0.f;
      // two float2 partial sums = 4 independent chains, updated with FADD2/FFMA2
      float2 s2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      float2 w2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      const uint32_t ts0 = ts;
      // One chunk: smem -> registers (slot released at once) -> TMEM stash ->
      // online softmax. `first` sets the exponent base from this thread's max of
      // chunk 0; `partial` masks elements past the slice end. Both are constants
      // at every call site, so the hot loop carries no per-chunk branches.
      auto chunk = [&](int k, bool first, bool partial) {
        if (warp_idle(k, partial, mis, span, 32 * (fw % SW))) {
          if (first) m2 = 0.f;  // no element of this warp in the row's only chunk
          fidle();
          return;
        }
        DBG_WAIT(w_a, KWAIT(full0 + 8u * slot, ph));
        const uint32_t sa = ring_t + slot * kCB;
        uint4 v0 = lds128(sa);
        uint4 v1 = lds128(sa + SCB / 2);
        DBG_WAIT(w_b, KWAIT(tempty0 + 8u * ts, tph ^ 1u));
        const bool in_tmem = ts < kTSlots;
        if (in_tmem) {
          tc_fence_after();
          if (!(dbg_mode & 8)) tmem_st8(tm_t + ts * static_cast<uint32_t>(kSlotCols), v0, v1);
        } else {
          const uint32_t sa2 = stash_t + (ts - kTSlots) * kCB;
          sts128(sa2, v0);
          sts128(sa2 + kCB / 2, v1);
        }
        // Release the ring slot only now: the row-store write above consumed
        // v0/v1, so both LDS have returned. An arrive issued straight after the
        // LDS can overtake them (SASS issues SYNCS.ARRIVE without a scoreboard
        // wait) and the next TMA fill of the slot then races the reads.
        mbar_arrive(empty0 + 8u * slot);
        if (++slot == kSlots) {
          slot = 0;
          ph ^= 1u;
        }
        float x[NE];
        unpack(logits, v0, v1, x);
        const int rem = span - k * SCE;             // valid elements end here (chunk coordinates)
        const int lo = (UA && k == 0) ? mis : 0;   // ... and start here
        if (first) {
          // Later elements may exceed this base (arguments > 0 are fine); only a
          // jump of > 126 in log2 units overflows, which the row-end repair handles.
          float xm = -INFINITY;
#pragma unroll
          for (int j = 0; j < NE; ++j) {
            const int pj = eoff(j);
            if (!partial || (pj >= lo && pj < rem)) xm = fmaxf(xm, x[j]);
          }
          m2 = xm * c;
          if (!(m2 > -INFINITY)) m2 = 0.f;  // nothing finite: any finite base works
        }
        if (!partial && (dbg_mode & 1)) {
          s2[0].x += __uint_as_float(v0.x & 0x3fffffffu);  // debug: no math (pipeline ceiling)
        } else if (!partial) {
          const float2 c2 = make_float2(c, c), nm2 = make_float2(-m2, -m2);
#pragma unroll
          for (int p = 0; p < NE / 2; ++p) {
            const float2 av = __ffma2_rn(make_float2(x[2 * p], x[2 * p + 1]), c2, nm2);
            const float2 e = make_float2(ex2(av.x), ex2(av.y));
            s2[p & 1] = __fadd2_rn(s2[p & 1], e);
            w2[p & 1] = __ffma2_rn(e, av, w2[p & 1]);
          }
        } else if (UA) {
          // unaligned row, front or tail chunk: packed math on vectors wholly
          // inside the row, element masks only on the (at most two) boundary
          // vectors of the chunk
          const float2 c2 = make_float2(c, c), nm2 = make_float2(-m2, -m2);
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int p0 = v * SHALF + EV * sid;
            if (p0 >= lo && p0 + EV <= rem) {
#pragma unroll
              for (int q = 0; q < EV / 2; ++q) {
                const int p = v * (EV / 2) + q;
                const float2 av = __ffma2_rn(make_float2(x[2 * p], x[2 * p + 1]), c2, nm2);
                const float2 e = make_float2(ex2(av.x), ex2(av.y));
                s2[p & 1] = __fadd2_rn(s2[p & 1], e);
                w2[p & 1] = __ffma2_rn(e, av, w2[p & 1]);
              }
            } else if (p0 + EV > lo && p0 < rem) {
#pragma unroll
              for (int j = 0; j < EV; ++j) {
                const int pj = p0 + j;
                if (pj >= lo && pj < rem && x[v * EV + j] != -INFINITY) {
                  const float av = fmaf(x[v * EV + j], c, -m2);
                  const float e = ex2(av);
                  s2[0].x += e;
                  w2[0].x = fmaf(e, av, w2[0].x);
                }
              }
            }
          }
        } else {
          // Partial chunk. Aligned slice lengths are multiples of the 16-B
          // vector, so each of this thread's two vectors lies wholly inside or
          // outside the slice: the packed path, per vector.
          // A -inf logit makes w NaN here as on full chunks -> row-end repair.
          const bool ok0 = EV * sid < rem, ok1 = SHALF + EV * sid < rem;
          const float2 c2 = make_float2(c, c), nm2 = make_float2(-m2, -m2);
#pragma unroll
          for (int p = 0; p < NE / 2; ++p) {
            if ((2 * p < EV) ? ok0 : ok1) {
              const float2 av = __ffma2_rn(make_float2(x[2 * p], x[2 * p + 1]), c2, nm2);
              const float2 e = make_float2(ex2(av.x), ex2(av.y));
              s2[p & 1] = __fadd2_rn(s2[p & 1], e);
              w2[p & 1] = __ffma2_rn(e, av, w2[p & 1]);
            }
          }
        }
        if (in_tmem) {
          if (!(dbg_mode & 8)) tmem_wait_st(v0, v1);
          tc_fence_before();
        }
        mbar_arrive(tfull0 + 8u * ts);  // release: orders the smem-store writes too
        if (++ts == kStore) {
          ts = 0;
          tph ^= 1u;
        }
      };
      if constexpr (UA) {
        // peeled like the aligned schedule: only the front and tail chunks are
        // masked (one masked copy for every chunk measured 25-30% slower)
        const int nfull_r = span / SCE;
        if (nck_r > 0) {
          if (mis > 0 || span < SCE) {
            chunk(0, true, true);
          } else {
            chunk(0, true, false);
          }
          for (int k = 1; k < nfull_r; ++k) chunk(k, false, false);
          if (nck_r > nfull_r && nck_r > 1) chunk(nck_r - 1, false, true);
        }
        if (NS > 1)
          for (int k = nck_r; k < nstep; ++k) fidle();  // the group's longer rows still stream
      } else if (nck == 0) {
        // empty slice (a cluster wider than the vocab): contributes nothing
      } else if (nfull == 0) {
        chunk(0, true, true);
      } else {
        chunk(0, true, false);
        for (int k = 1; k < nfull; ++k) chunk(k, false, false);
        if (nck > nfull) chunk(nfull, false, true);
      }
      Stats my{m2, (s2[0].x + s2[1].x) + (s2[0].y + s2[1].y), (w2[0].x + w2[1].x) + (w2[0].y + w2[1].y)};
      // Repair (rare): a -inf logit (0 * -inf in w) or an exponent overflow
      // (a logit > 126/log2e above the chunk-0 base) made s or w non-finite:
      // recompute this thread's partials exactly from its TMEM words.
      const bool bad = !(fabsf(my.s) <= 3.0e38f) || !(fabsf(my.w) <= 3.0e38f);
      if (__any_sync(0xffffffffu, bad)) {
        float mx = -INFINITY;
        uint32_t q = ts0;
        for (int k = 0; k < nck_r; ++k) {
          uint4 v0r, v1r;
          load_store(q, v0r, v1r);
          float x[NE];
          unpack(logits, v0r, v1r, x);
          const int rem = span - k * SCE, lo = (UA && k == 0) ? mis : 0;
#pragma unroll
          for (int j = 0; j < NE; ++j) {
            const int pj = eoff(j);
            if (pj >= lo && pj < rem) mx = fmaxf(mx, x[j]);
          }
          if (++q == kStore) q = 0;
        }
        const float mb2 = (mx == -INFINITY) ? -INFINITY : mx * c;
        float sr = 0.f, wr = 0.f;
        q = ts0;
        for (int k = 0; k < nck_r; ++k) {
          uint4 v0r, v1r;
          load_store(q, v0r, v1r);
          float x[NE];
          unpack(logits, v0r, v1r, x);
          const int rem = span - k * SCE, lo = (UA && k == 0) ? mis : 0;
#pragma unroll
          for (int j = 0; j < NE; ++j) {
            const int pj = eoff(j);
            if (pj >= lo && pj < rem && x[j] != -INFINITY) {
              const float av = fmaf(x[j], c, -mb2);
              const float e = ex2(av);
              sr += e;
              wr = fmaf(e, av, wr);
            }
          }
          if (++q == kStore) q = 0;
        }
        if (bad) my = Stats{mb2, sr, wr};
      }
      if (my.s == 0.f) my = stats_empty();  // nothing finite in this thread's share
      // Per-warp partial -> smem ring; no CTA barrier: the control warp
      // merges the 12 partials, so forward warps go straight to the next row.
      my = warp_merge(my);
      if (lane == 0) {
        KWAIT(smem_u32(&red_free[nrow % RD]), ((nrow / RD) & 1u) ^ 1u);
        red[nrow % RD][fw % SW] = make_float4(my.m2, my.s, my.w, 0.f);
        mbar_arrive(smem_u32(&red_bar[nrow % RD]));
      }
      ++nrow;
      DBG_ROW(nrow);
    }
    // the CTA's last group of rows has no row for this stream: idle through its steps
    if (NS > 1 && static_cast<int>(nrow % NS) != 0 && sg >= static_cast<int>(nrow % NS))
      for (int k = 0; k < nstep; ++k) fidle();
  } else if (warp >= kCtl) {
    // ================================================================ control
    // Per row: merge the 12 forward partials, exchange with the cluster through
    // DSMEM mailboxes, compute the loss scalars once and publish them to the
    // backward warps. Never touches the row data, so it runs as far ahead as
    // the forward warps allow. The control warps take rotating active rows
    // so the per-row latency chain (merge -> DSMEM round trip -> scalars) of
    // one row overlaps the next.
    const int ci = warp - kCtl;
    const LossParamsDev P{a.eps_lo, a.eps_hi, a.dual_c, a.beta, a.ent_coef, a.kl_mode};
    const bool leader = (crank == 0 && lane == 0);
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (XP) {
      // Peer exchange: the latency of a cross-GPU round trip is several rows
      // long, so sending and receiving are split. Warp 0 (sender) merges the
      // forward partials and posts them to every rank's mailbox as soon as the
      // row's forward is done; the receivers (the other control warps, rows
      // alternating) merge the P partials in rank order and publish the scalars. The
      // sender stays at most kXpCredit rows ahead of the receiver, which with
      // the same bound on every rank keeps any rank from overrunning a peer's
      // kMailD-deep mailbox ring.
      uint32_t nrow = 0;
      RowIn nx = load_row_in(a, cid, ncl, 0, lane);
      for (int64_t win = 0; cid + 32 * win * ncl < a.T; ++win) {
        const RowIn cur = nx;
        nx = load_row_in(a, cid, ncl, win + 1, lane);  // one window ahead
        const int64_t tl = cid + (32 * win + lane) * ncl;  // this lane's row of the window
        if (ci == 0) zero_masked_outputs(a, tl, cur.w);
        uint32_t bits = __ballot_sync(0xffffffffu, tl < a.T && cur.w != 0.f);
        while (bits != 0u) {
        const int i = __ffs(bits) - 1;
        bits &= bits - 1u;
        const int64_t t = cid + (32 * win + i) * ncl;
        const float w = __shfl_sync(0xffffffffu, cur.w, i), A = __shfl_sync(0xffffffffu, cur.A, i);
        const float old = __shfl_sync(0xffffffffu, cur.old, i), ref = __shfl_sync(0xffffffffu, cur.ref, i);
        const int32_t ycur = __shfl_sync(0xffffffffu, cur.y, i);
        const uint32_t mb = nrow % kXpMailD;
        const uint64_t tag = static_cast<uint64_t>(static_cast<uint32_t>(a.xp_epoch << 20) + nrow + 1u) << 32;
        const int64_t yg = static_cast<int64_t>(ycur) - a.vocab_start;
        if (ci == 0) {
          // ------------------------------------------------ sender
          const uint32_t rs = nrow % RD;
          float zy = __int_as_float(0x7fc00000);
          if (yg >= 0 && yg < a.V) zy = ldg_elem(logits, t * a.ld + yg) * a.inv_tau;
          if (nrow >= static_cast<uint32_t>(kXpCredit)) {
            const uint32_t m = nrow - kXpCredit;
            KWAIT(smem_u32(&rcv_done[m % kCredD]), (m / kCredD) & 1u);
          }
          DBG_WAIT(w_a, KWAIT(smem_u32(&red_bar[rs]), (nrow / RD) & 1u));
          Stats v = stats_empty();
          if (lane < SW) {
            const float4 r = red[rs][lane];
            v = Stats{r.x, r.y, r.z};
          }
          v = warp_merge(v);
          if (lane == 0) mbar_arrive(smem_u32(&red_free[rs]));
          if (lane < a.xp_P) {
            XpMsg* dst = static_cast<XpMsg*>(a.xp_mail[lane]) + xp_index(a.xp_epoch, static_cast<int>(cid), mb, a.xp_rank);
            st_sys_v2u64(&dst->w[0], tag | __float_as_uint(v.m2), tag | __float_as_uint(v.s));
            st_sys_v2u64(&dst->w[2], tag | __float_as_uint(v.w), tag | __float_as_uint(zy));
#ifdef SFTM_HANG_DEBUG
            if (lane == 0)  // the sender's progress: rows posted, epoch, and the address for peer 0 (hang_debug)
              reinterpret_cast<volatile unsigned long long*>(a.dbg)[16 + 2 * 8 * 148 * 32 + (a.xp_rank & 7) * 148 +
                                                                    blockIdx.x] =
                  (nrow + 1) | (static_cast<unsigned long long>(a.xp_epoch & 0xff) << 8) |
                  (static_cast<unsigned long long>(reinterpret_cast<uintptr_t>(
                       static_cast<XpMsg*>(a.xp_mail[0]) + xp_index(a.xp_epoch, static_cast<int>(cid), mb, a.xp_rank)) &
                                                   0xffffffffull)
                   << 16);
            if (lane == 0 && nrow < 4)
              reinterpret_cast<volatile unsigned long long*>(a.dbg)[16 + 2 * 8 * 148 * 32 + 8 * 148 +
                                                                    ((a.xp_rank & 7) * 148 + blockIdx.x) * 4 + nrow] =
                  globaltimer_ns();
#endif
          }
        } else if (static_cast<int>(nrow % (kNCtl - 1)) == ci - 1) {
          // ------------------------------------------------ receivers (rows alternate)
          const uint32_t rs = nrow % RD;
          const uint32_t rpar = (nrow / RD) & 1u;
          const int64_t yl64 = yg - slice_start;
          float4 mv = make_float4(-INFINITY, 0.f, 0.f, __int_as_float(0x7fc00000));
          if (lane < a.xp_P) {
            const XpMsg* src = static_cast<const XpMsg*>(a.xp_mail[a.xp_rank]) +
                               xp_index(a.xp_epoch, static_cast<int>(cid), mb, lane);
            constexpr uint64_t kHi = 0xffffffff00000000ull;
            uint64_t q0, q1, q2, q3;
            ld_sys_v2u64(&src->w[0], q0, q1);
            ld_sys_v2u64(&src->w[2], q2, q3);
            if (((q0 & kHi) != tag) | ((q1 & kHi) != tag) | ((q2 & kHi) != tag) | ((q3 & kHi) != tag)) {
              const uint64_t t0 = globaltimer_ns();
              do {
                __nanosleep(64);
                // A peer that never launches (or died) must not hang the
                // context: past the timeout (or once another CTA of this launch
                // gave up) stop waiting, flag the launch as failed (host-mapped
                // word, surfaced by the next API call as Internal) and let the
                // kernel run to completion on the stale mailbox values.
                const uint64_t el = globaltimer_ns() - t0;
#ifdef SFTM_HANG_DEBUG
                if (el > 1000000000ull) {  // which peer's message of which row is late (hang_debug)
                  volatile unsigned long long* vd = a.dbg + 16 + 8 * 148 * 32;
                  const size_t i = (static_cast<size_t>(a.xp_rank & 7) * 148 + blockIdx.x) * 32 + lane;
                  if (vd[i] == 0ull)
                    vd[i] = (static_cast<unsigned long long>(nrow & 0xff) << 56) | (a.xp_epoch & 0xff) << 48 |
                            (reinterpret_cast<uintptr_t>(src) & 0xffffffffull) << 8 | 1ull;
                  vd[8 * 148 * 32 + 8 * 148 + 8 * 148 * 4 + i] = t0;  // when this receiver started waiting
                }
#endif
                if (el > 1000000ull &&
                    (el > a.xp_timeout_ns || *reinterpret_cast<volatile int*>(a.xp_abort) != 0)) {
                  atomicExch(a.xp_abort, 1);
                  *reinterpret_cast<volatile int*>(a.xp_err) = 1;
                  __threadfence_system();
                  break;
                }
                ld_sys_v2u64(&src->w[0], q0, q1);
                ld_sys_v2u64(&src->w[2], q2, q3);
              } while (((q0 & kHi) != tag) | ((q1 & kHi) != tag) | ((q2 & kHi) != tag) | ((q3 & kHi) != tag));
            }
            mv = make_float4(__uint_as_float(static_cast<uint32_t>(q0)), __uint_as_float(static_cast<uint32_t>(q1)),
                             __uint_as_float(static_cast<uint32_t>(q2)), __uint_as_float(static_cast<uint32_t>(q3)));
          }
          // merge in rank order (identical scalars on every rank); the owner's z_target
          Stats st = stats_empty();
          float zy = __int_as_float(0x7fc00000);
          for (int q = 0; q < a.xp_P; ++q) {
            const float zq = __shfl_sync(0xffffffffu, mv.w, q);
            st = stats_merge(st, Stats{__shfl_sync(0xffffffffu, mv.x, q), __shfl_sync(0xffffffffu, mv.y, q),
                                       __shfl_sync(0xffffffffu, mv.z, q)});
            if (zq == zq) zy = zq;
          }
          float lse2, lse, H, logp;
          row_scalars(st, zy, lse2, lse, H, logp);
          float g, gH, m[8];
          loss_terms(logp, H, w, A, old, ref, P, g, gH, m);
          if (leader) {
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] += static_cast<double>(m[i]);
            if (a.out_logp) a.out_logp[t] = logp;
            if (a.out_entropy) a.out_entropy[t] = H;
          }
          if (lane == 0) {
            RowScal r;
            r.lse2 = lse2;
            r.gt = a.inv_tau * g;
            r.c0 = a.inv_tau * (g + gH * H);
            r.c1 = a.inv_tau * gH * kLn2;
            r.lse2f = lse2 - log2f(fabsf(r.c0));
            r.sgn = r.c0 > 0.f ? 0x80008000u : 0u;
            target_slot(yl64, row_mis(t), r.tck, r.town);
            if (NS > 1 && nrow > 0) {  // publish in row order (see the plain control path)
              const uint32_t p = nrow - 1;
              KWAIT(smem_u32(&scal_bar[p % RD]), (p / RD) & 1u);
            }
            KWAIT(smem_u32(&scal_free[rs]), rpar ^ 1u);
            scal[rs] = r;
            mbar_arrive(smem_u32(&scal_bar[rs]));
            mbar_arrive(smem_u32(&rcv_done[nrow % kCredD]));  // the shuffles consumed the messages
          }
        }
        ++nrow;
        DBG_ROW(nrow);
        }
      }
    } else {
    uint32_t nrow = 0;
    RowIn nx = load_row_in(a, cid, ncl, 0, lane);
    for (int64_t win = 0; cid + 32 * win * ncl < a.T; ++win) {
      const RowIn cur = nx;
      nx = load_row_in(a, cid, ncl, win + 1, lane);  // one window ahead
      const int64_t tl = cid + (32 * win + lane) * ncl;  // this lane's row of the window
      if (ci == 0 && crank == 0) zero_masked_outputs(a, tl, cur.w);
      uint32_t bits = __ballot_sync(0xffffffffu, tl < a.T && cur.w != 0.f);
      // rows of the other control warps
      while (bits != 0u && static_cast<int>(nrow % kNCtl) != ci) {
        bits &= bits - 1u;
        ++nrow;
        DBG_ROW(nrow);
      }
      while (bits != 0u) {
      const int i = __ffs(bits) - 1;
      bits &= bits - 1u;
      const int64_t t = cid + (32 * win + i) * ncl;
      const float w = __shfl_sync(0xffffffffu, cur.w, i), A = __shfl_sync(0xffffffffu, cur.A, i);
      const float old = __shfl_sync(0xffffffffu, cur.old, i), ref = __shfl_sync(0xffffffffu, cur.ref, i);
      const int32_t ycur = __shfl_sync(0xffffffffu, cur.y, i);
      const uint32_t rs = nrow % RD;
      const uint32_t rpar = (nrow / RD) & 1u;
      const int64_t yg = static_cast<int64_t>(ycur) - a.vocab_start;
      const int64_t yl64 = yg - slice_start;
      // z_target straight from HBM, issued before the partials wait; the
      // published scalars depend on it, so the read completes before their
      // release arrive and thus before any dlogits write of the row (in-place
      // dlogits stays safe)
      float zy = __int_as_float(0x7fc00000);
      if (yg >= 0 && yg < a.V) zy = ldg_elem(logits, t * a.ld + yg) * a.inv_tau;
      if (NS > 1 && nrow > 0) {
        // Row streams finish the rows of a group out of order, so a control
        // warp could reach this slot's wait before row nrow - RD was even
        // written and take that phase for its own (parity aliasing). Consuming
        // the partials strictly in row order (row nrow - 1 first) rules it out.
        const uint32_t p = nrow - 1;
        KWAIT(smem_u32(&red_free[p % RD]), (p / RD) & 1u);
      }
      DBG_WAIT(w_a, KWAIT(smem_u32(&red_bar[rs]), rpar));
      Stats v = stats_empty();
      if (lane < SW) {
        const float4 r = red[rs][lane];
        v = Stats{r.x, r.y, r.z};
      }
      v = warp_merge(v);
      if (lane == 0) mbar_arrive(smem_u32(&red_free[rs]));  // the shuffles consumed every lane's read
      Stats st = stats_empty();
      if constexpr (C == 1) {
        st = stats_merge(st, v);  // one CTA per row: no exchange
      } else {
        const float z = 0.f;
        const uint32_t mb = nrow % kXpMailD;
        if (lane == 0) {
          const uint32_t my_slot = smem_u32(&mail[mb][crank]);
          const uint32_t my_bar = smem_u32(&mail_bar[mb]);
#pragma unroll
          for (int q = 0; q < C; ++q) {
            st_cluster_v4(mapa(my_slot, q), v.m2, v.s, v.w, z);
            mbar_arrive_remote(mapa(my_bar, q));
          }
        }
        DBG_WAIT(w_b, mbar_wait_cluster_lite(smem_u32(&mail_bar[mb]), (nrow / kMailD) & 1u));
#pragma unroll
        for (int q = 0; q < C; ++q) {
          const float4 mv = mail[mb][q];
          st = stats_merge(st, Stats{mv.x, mv.y, mv.z});
        }
      }
      float lse2, lse, H, logp;
      row_scalars(st, zy, lse2, lse, H, logp);
      float g, gH, m[8];
      loss_terms(logp, H, w, A, old, ref, P, g, gH, m);
      if (leader) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += static_cast<double>(m[i]);
        if (a.out_logp) a.out_logp[t] = logp;
        if (a.out_entropy) a.out_entropy[t] = H;
      }
      if (lane == 0) {
        // dlogits_v = gt*[v==y] - p_v*(c0 + c1*a_v), a_v = (z_v - lse)*log2e, p_v = 2^a_v;
        // fast form (c1 == 0): p_v*c0 = sign(c0) * 2^(a_v + log2|c0|).
        RowScal r;
        r.lse2 = lse2;
        r.gt = a.inv_tau * g;
        r.c0 = a.inv_tau * (g + gH * H);
        r.c1 = a.inv_tau * gH * kLn2;
        r.lse2f = lse2 - log2f(fabsf(r.c0));
        r.sgn = r.c0 > 0.f ? 0x80008000u : 0u;
        target_slot(yl64, row_mis(t), r.tck, r.town);
        if (NS > 1 && nrow > 0) {
          // publish in row order (row nrow - 1 first): then row nrow - RD was
          // published, its backward waited, and this slot's free phase below
          // cannot alias an older one
          const uint32_t p = nrow - 1;
          KWAIT(smem_u32(&scal_bar[p % RD]), (p / RD) & 1u);
        }
        KWAIT(smem_u32(&scal_free[rs]), rpar ^ 1u);
        scal[rs] = r;
        mbar_arrive(smem_u32(&scal_bar[rs]));
      }
    
      ++nrow;
      DBG_ROW(nrow);
      // skip to this warp's next row (kNCtl - 1 rows of the other control warps)
      for (int q = 1; q < kNCtl && bits != 0u; ++q) {
        bits &= bits - 1u;
        ++nrow;
        DBG_ROW(nrow);
      }
      }
      // rows of this window past our last one belong to the others: nrow already
      // counts every row handed out above
    }
    }  // XP / alternating
    // fixed-order combine of the two control warps' fp64 partials, then the
    // deterministic cross-block finish
    __shared__ double acc_sh[kNCtl - 1][8];
    if (ci >= 1 && lane == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) acc_sh[ci - 1][i] = acc[i];
    }
    named_bar_sync(2, kNCtl * 32);
    if (ci == 0 && leader) {
      for (int q = 0; q < kNCtl - 1; ++q)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += acc_sh[q][i];
      finish_metrics(a, cid, ncl, acc);
    }
  } else {
    // ================================================================ backward
    const int btid = tid;                     // same element mapping as forward warp warp+kBW
    const int bw = warp;
    const int sg = bw / SW;                   // row stream (as its partner forward warp)
    const int sid = btid - sg * (SW * 32);    // thread index within the stream
    const uint32_t tlane = static_cast<uint32_t>(32 * (bw & 3)) << 16;
    const uint32_t tcol = 8u * static_cast<uint32_t>(bw >> 2);
    const float c = a.inv_tau * kLog2e;
    const uint32_t tfull0 = smem_u32(&tfull_bar[0]), tempty0 = smem_u32(&tempty_bar[0]);
    const uint32_t tm_t = tbase + tlane + tcol;
    const uint32_t stash_t = stash_base + 16u * btid;
    const uint32_t sink_a = smem_u32(&sink_sh[warp]);  // dummy-store target (never read)
    uint32_t ts = 0, tph = 0, nrow = 0;
    RowSeq<NS> rows;
    rows.init(a.w_tok, a.T, cid, ncl, lane);
    int64_t t;
    bool active;
    while (rows.next_all(t, active)) {
      if (!active) {
        if (!a.masked_skip) {
          T* drow0 = static_cast<T*>(a.dlogits) + t * a.ld_d + slice_start;
          if constexpr (UA) {
            // element stores up to the first 16-B sector, vectors, element tail
            const int head = static_cast<int>(((16u - (reinterpret_cast<uintptr_t>(drow0) & 15u)) & 15u) / G::es);
            const int h = head < slice_len ? head : slice_len;
            if (btid < h) st1(drow0 + btid, 0.f);
            uint8_t* mid = reinterpret_cast<uint8_t*>(drow0 + h);
            const int nv = (slice_len - h) / EV;
            for (int i = btid; i < nv; i += kFT) stg128_cs(mid + 16 * i, make_uint4(0, 0, 0, 0));
            const int tl = h + nv * EV;
            if (btid < slice_len - tl) st1(drow0 + tl + btid, 0.f);
          } else {
            uint8_t* drow = reinterpret_cast<uint8_t*>(drow0);
            const int nb = slice_len * G::es;
            for (int off = btid * 16; off < nb; off += kFT * 16) stg128_cs(drow + off, make_uint4(0, 0, 0, 0));
          }
        }
        continue;
      }
      if (NS > 1 && static_cast<int>(nrow % NS) != sg) {  // another stream's row
        ++nrow;
        DBG_ROW(nrow);
        continue;
      }
      const int mis = row_mis(t);
      const int span = slice_len + mis;  // row extent in sector coordinates
      const int nck_r = UA ? (span + SCE - 1) / SCE : nck;
      const uint32_t rs = nrow % RD;
      const uint32_t rpar = (nrow / RD) & 1u;
      DBG_WAIT(w_a, KWAIT(smem_u32(&scal_bar[rs]), rpar));
      const RowScal rsc = scal[rs];
      const float lse2 = rsc.lse2, lse2f = rsc.lse2f, c0 = rsc.c0, c1 = rsc.c1, gt = rsc.gt;
      const bool neg = rsc.sgn != 0u;
      const int ck = (static_cast<int>(rsc.town >> 8) == sid) ? rsc.tck : -1;
      const int jt = static_cast<int>(rsc.town & 0xffu);
      // dlogits rows share the logits rows' sector phase (checked at dispatch)
      T* drow = static_cast<T*>(a.dlogits) + t * a.ld_d + slice_start - mis;
      T* const dlane = drow + EV * sid;  // this thread's first vector of chunk 0 (full chunks add k * SCE)
      const uint32_t sgn = neg ? 0x80008000u : 0u;
      const float gts = neg ? -gt : gt;  // target term before the sign flip
      // One chunk of dlogits. MODE (row-uniform): 0 = bf16 with |c0| folded
      // into the exponent and the sign applied to the packed words, 1 = no
      // entropy term, 2 = entropy term. `partial` masks past the slice end.
      auto bchunk = [&](int k, bool partial, int mode) {
        if (warp_idle(k, partial, mis, span, 32 * (bw % SW))) {
          DBG_WAIT(w_b, KWAIT(tfull0 + 8u * ts, tph));
          mbar_arrive(tempty0 + 8u * ts);  // nothing read from the row-store slot
          if (++ts == kStore) {
            ts = 0;
            tph ^= 1u;
          }
          return;
        }
        DBG_WAIT(w_b, KWAIT(tfull0 + 8u * ts, tph));
        tc_fence_after();
        uint4 w0 = make_uint4(0, 0, 0, 0), w1 = make_uint4(0, 0, 0, 0);
        // TMEM slots are released once tcgen05.wait::ld returned; smem-store
        // slots only after the dlogits stores below consumed the LDS results
        // (see the forward's ring release)
        const uint32_t rel = tempty0 + 8u * ts;
        const bool late = ts >= kTSlots;
        if (!late) {
          if (!(dbg_mode & 8)) {
            tmem_ld8(tm_t + ts * static_cast<uint32_t>(kSlotCols), w0, w1);
            tmem_wait_ld(w0, w1);
          }
          tc_fence_before();
          mbar_arrive(rel);
        } else {
          w0 = lds128(stash_t + (ts - kTSlots) * kCB);
          w1 = lds128(stash_t + (ts - kTSlots) * kCB + kCB / 2);
        }
        if (++ts == kStore) {
          ts = 0;
          tph ^= 1u;
        }
        T* dst = drow + k * SCE;
        const int rem = span - k * SCE;
        if (!partial && (dbg_mode & 2)) {  // debug: store the words back (pipeline ceiling)
          if (!(dbg_mode & 4)) {
            stg128_cs(dst + EV * sid, w0);
            stg128_cs(dst + SHALF + EV * sid, w1);
          }
          if (late) {
            __threadfence_block();  // debug path: order the LDS before the release
            mbar_arrive(rel);
          }
          return;
        }
        float x[NE], gr[NE];
        unpack(logits, w0, w1, x);
        // partial chunk: skip the math of vectors wholly outside the row (their
        // stores are skipped too); `dep` ties a thread that stores nothing to
        // its loads and scalars for the release ordering (dummy smem store)
        bool vok0 = true, vok1 = true;
        if (partial) {
          const int lo = (UA && k == 0) ? mis : 0;
          vok0 = (EV * sid + EV > lo) && (EV * sid < rem);
          vok1 = (SHALF + EV * sid + EV > lo) && (SHALF + EV * sid < rem);
        }
        const uint32_t dep = w0.x ^ w1.w ^ __float_as_uint(lse2f) ^ rsc.sgn;
        if (mode == 0) {
          const float2 c2 = make_float2(c, c), nl2 = make_float2(-lse2f, -lse2f);
#pragma unroll
          for (int p = 0; p < NE / 2; ++p) {
            if ((2 * p < EV) ? vok0 : vok1) {
              const float2 av = __ffma2_rn(make_float2(x[2 * p], x[2 * p + 1]), c2, nl2);
              gr[2 * p] = ex2(av.x);
              gr[2 * p + 1] = ex2(av.y);
            } else {
              gr[2 * p] = gr[2 * p + 1] = 0.f;
            }
          }
          if (k == ck) {
#pragma unroll
            for (int j = 0; j < NE; ++j)
              gr[j] += (j == jt) ? gts : 0.f;  // select, not an indexed store (keeps gr in registers)
          }
          if (UA && partial) {
#pragma unroll
            for (int j = 0; j < NE; ++j) gr[j] = neg ? -gr[j] : gr[j];
            goto general_store;
          }
          uint4 p0, p1;
          p0.x = pack_bf16x2(gr[0], gr[1]) ^ sgn;
          p0.y = pack_bf16x2(gr[2], gr[3]) ^ sgn;
          p0.z = pack_bf16x2(gr[4], gr[5]) ^ sgn;
          p0.w = pack_bf16x2(gr[6], gr[7]) ^ sgn;
          p1.x = pack_bf16x2(gr[8], gr[9]) ^ sgn;
          p1.y = pack_bf16x2(gr[10], gr[11]) ^ sgn;
          p1.z = pack_bf16x2(gr[12], gr[13]) ^ sgn;
          p1.w = pack_bf16x2(gr[14], gr[15]) ^ sgn;
          if (!partial) {
            T* const dv = dlane + k * SCE;
            stg128_cs(dv, p0);
            stg128_cs(dv + SHALF, p1);
          } else {
            // vector-granular tail (see the forward's partial chunk)
            const bool s0 = EV * sid < rem, s1 = SHALF + EV * sid < rem;
            if (s0) stg128_cs(dst + EV * sid, p0);
            if (s1) stg128_cs(dst + SHALF + EV * sid, p1);
            // a thread storing nothing still orders its loads before the
            // releases below through a dependent (dummy) smem store
            if (!s0) sink_u32(sink_a, p0.x ^ p1.y ^ dep);
          }
          if (late) mbar_arrive(rel);
          return;
        } else if (mode == 1) {
          const float2 c2 = make_float2(c, c), nl2 = make_float2(-lse2, -lse2);
          const float2 mc0 = make_float2(-c0, -c0);
#pragma unroll
          for (int p = 0; p < NE / 2; ++p) {
            if ((2 * p < EV) ? vok0 : vok1) {
              const float2 av = __ffma2_rn(make_float2(x[2 * p], x[2 * p + 1]), c2, nl2);
              const float2 g2 = __fmul2_rn(make_float2(ex2(av.x), ex2(av.y)), mc0);
              gr[2 * p] = g2.x;
              gr[2 * p + 1] = g2.y;
            } else {
              gr[2 * p] = gr[2 * p + 1] = 0.f;
            }
          }
          if (k == ck) {
#pragma unroll
            for (int j = 0; j < NE; ++j)
              gr[j] += (j == jt) ? gt : 0.f;
          }
        } else {
          // entropy term: -p_v (c0 + c1 a_v); the clamp keeps a -inf logit at 0 (not NaN)
          const float2 c2 = make_float2(c, c), nl2 = make_float2(-lse2, -lse2);
          const float2 mc1 = make_float2(-c1, -c1), mc0 = make_float2(-c0, -c0);
#pragma unroll
          for (int p = 0; p < NE / 2; ++p) {
            if ((2 * p < EV) ? vok0 : vok1) {
              float2 av = __ffma2_rn(make_float2(x[2 * p], x[2 * p + 1]), c2, nl2);
              av.x = fmaxf(av.x, -127.f);
              av.y = fmaxf(av.y, -127.f);
              const float2 t2 = __ffma2_rn(mc1, av, mc0);
              const float2 g2 = __fmul2_rn(make_float2(ex2(av.x), ex2(av.y)), t2);
              gr[2 * p] = g2.x;
              gr[2 * p + 1] = g2.y;
            } else {
              gr[2 * p] = gr[2 * p + 1] = 0.f;
            }
          }
          if (k == ck) {
#pragma unroll
            for (int j = 0; j < NE; ++j)
              gr[j] += (j == jt) ? gt : 0.f;
          }
        }
      general_store:
        if (!partial) {
          T* const dv = dlane + k * SCE;
          store_vec(dv, gr);
          store_vec(dv + SHALF, gr + EV);
        } else if (UA) {
          // front/tail chunk of an unaligned row: whole vectors where they are
          // entirely inside the row, element stores on the boundary vectors
          const int lo = (k == 0) ? mis : 0;
          bool any = false;
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int p0 = v * SHALF + EV * sid;
            if (p0 >= lo && p0 + EV <= rem) {
              store_vec(dst + p0, gr + v * EV);
              any = true;
            } else {
#pragma unroll
              for (int j = 0; j < EV; ++j)
                if (p0 + j >= lo && p0 + j < rem) {
                  st1(dst + p0 + j, gr[v * EV + j]);
                  any = true;
                }
            }
          }
          if (!any) sink_u32(sink_a, __float_as_uint(gr[0]) ^ __float_as_uint(gr[NE - 1]) ^ dep);
        } else {
          const bool s0 = EV * sid < rem;
          if (s0) store_vec(dst + EV * sid, gr);
          if (SHALF + EV * sid < rem) store_vec(dst + SHALF + EV * sid, gr + EV);
          if (!s0) sink_u32(sink_a, __float_as_uint(gr[0]) ^ __float_as_uint(gr[NE - 1]) ^ dep);
        }
        if (late) mbar_arrive(rel);
      };
      const int mode = (G::es == 2 && c1 == 0.f) ? 0 : (c1 == 0.f ? 1 : 2);
      if constexpr (UA) {
        // bf16 rows take mode 0 or 2, fp32 rows 1 or 2: only those schedules are
        // instantiated, and a full chunk 0 runs as the loop's first step. The
        // unaligned kernel's code size is what its narrow rows pay for in
        // instruction-cache misses (ncu at 12,569-wide rows: no_instruction
        // stalls 2.8 per issue vs 0.5 aligned); this trim: +12% there.
        auto sched = [&](auto md) {
          constexpr int M = decltype(md)::value;
          const int nfull_r = span / SCE;
          const bool front = mis > 0 || span < SCE;
          if (nck_r == 0) return;
          if (front) bchunk(0, true, M);
          for (int k = front ? 1 : 0; k < nfull_r; ++k) bchunk(k, false, M);
          if (nck_r > nfull_r && nck_r > 1) bchunk(nck_r - 1, true, M);
        };
        if constexpr (G::es == 2) {
          if (mode == 0) {
            sched(std::integral_constant<int, 0>{});
          } else {
            sched(std::integral_constant<int, 2>{});
          }
        } else {
          if (mode == 1) {
            sched(std::integral_constant<int, 1>{});
          } else {
            sched(std::integral_constant<int, 2>{});
          }
        }
      } else if (mode == 0) {
        for (int k = 0; k < nfull; ++k) bchunk(k, false, 0);
        if (nck > nfull) bchunk(nfull, true, 0);
      } else if (mode == 1) {
        for (int k = 0; k < nfull; ++k) bchunk(k, false, 1);
        if (nck > nfull) bchunk(nfull, true, 1);
      } else {
        for (int k = 0; k < nfull; ++k) bchunk(k, false, 2);
        if (nck > nfull) bchunk(nfull, true, 2);
      }
      if (UA && NS > 1) {
        for (int k = nck_r; k < nstep; ++k) {  // the group's longer rows still stream
          DBG_WAIT(w_b, KWAIT(tfull0 + 8u * ts, tph));
          mbar_arrive(tempty0 + 8u * ts);
          if (++ts == kStore) {
            ts = 0;
            tph ^= 1u;
          }
        }
      }
      // the row's stores consumed every lane's scalars (a row with no chunk
      // here consumes them through a dependent dummy smem store): free the slot
      if (nck_r == 0) sink_u32(sink_a, __float_as_uint(lse2f) ^ __float_as_uint(c0) ^ rsc.sgn ^ rsc.town);
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&scal_free[rs]));
      ++nrow;
      DBG_ROW(nrow);
    }
    // the CTA's last group of rows has no row for this stream: idle through its steps
    if (NS > 1 && static_cast<int>(nrow % NS) != 0 && sg >= static_cast<int>(nrow % NS)) {
      for (int k = 0; k < nstep; ++k) {
        DBG_WAIT(w_b, KWAIT(tfull0 + 8u * ts, tph));
        mbar_arrive(tempty0 + 8u * ts);  // nothing read from the row-store slot
        if (++ts == kStore) {
          ts = 0;
          tph ^= 1u;
        }
      }
    }
  }

  if (dbg && lane == 0) {
    const int role = (warp == kProd) ? 0 : (warp >= kCtl) ? 2 : (warp >= kBW) ? 1 : 3;
    atomicAdd(dbg + 3 * role + 0, static_cast<unsigned long long>(clock64() - t_role0));
    atomicAdd(dbg + 3 * role + 1, w_a);
    atomicAdd(dbg + 3 * role + 2, w_b);
    atomicAdd(dbg + 12 + role, 1ull);
  }
  // teardown: every TMEM access is complete before warp 0 frees it
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, kTCols);
  if (C > 1) cluster_sync_all();
}

std::mutex g_mu;

// One-time setup of an instantiation on the current device (dynamic smem
// opt-in, occupancy): returns the co-resident CTA (cluster) count, or < 0 with
// *err. cudaFuncSetAttribute can wait for kernels already running, so the
// peer-exchange instantiations are prepared when the mailboxes are wired
// (prepare_loss_xp), never while a peer's kernel spins waiting for this one.
template <typename T, int C, bool XP = false, bool UA = false, int NS = 1>
int init_c(cudaError_t* err) {
  auto kern = loss_tmem_kernel<T, C, XP, UA, NS>;
  static PerDevice cache;  // per instantiation and device
  int& max_active = cache();
  *err = cudaSuccess;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (max_active < 0) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingBytes);
      if (e != cudaSuccess) {
          *err = e;
          return -1;
        }
      if (C > 1) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(C * 256);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = kRingBytes;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
        if (e != cudaSuccess) {
          *err = e;
          return -1;
        }
        max_active = n;
      } else {
        int per_sm = 0, dev = 0, sms = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, kRingBytes);
        if (e != cudaSuccess) {
          *err = e;
          return -1;
        }
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        max_active = per_sm * sms;
      }
      if (max_active <= 0) {
        *err = cudaErrorInvalidConfiguration;
        return -1;
      }
    }
  }
  return max_active;
}

template <typename T, int C, bool XP = false, bool UA = false, int NS = 1>
int launch_c(const RowArgs& a, int64_t slice, cudaStream_t s, LaunchInfo* info) {
  auto kern = loss_tmem_kernel<T, C, XP, UA, NS>;
  cudaError_t ie;
  const int max_active = init_c<T, C, XP, UA, NS>(&ie);
  if (max_active < 0) return ie;
  int64_t ncl = a.T < max_active ? a.T : max_active;
  if (XP) {  // same grid on every rank, whatever T
    ncl = max_active < kXpMaxCtas ? max_active : kXpMaxCtas;
    if (a.xp_grid > 0 && a.xp_grid < ncl) ncl = a.xp_grid;  // co-resident emulated ranks (tests)
  }
  RowArgs ad = a;
  ad.dbg = debug_counters();
  if (ncl > a.max_partial_blocks) ncl = a.max_partial_blocks;
  if (ncl < 1) ncl = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(ncl * C));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kRingBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (C > 1) ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ad, slice);
  if (info) {
    info->kernel = XP ? 4 : 2;
    info->cluster = C;
    info->grid = static_cast<int>(ncl * C);
    info->launches = 1;
    info->streams = NS;
  }
  return e;
}

// Row streams for a one-CTA row slice of `slice` elements (for unaligned rows
// the widest span, V + EV - 1). Measured on B200 (scripts/ns_ab.sh, bf16): the
// most streams whose per-stream row takes <= 15 sub-chunks, i.e. leaves the
// row store room for two groups of rows (18,992 wide -> 4, 24,576 / 27,648 /
// 37,984 -> 2); at 16-18 sub-chunks the store holds < 2 groups and the
// pipeline stalls (24,576 at 4 streams, 55,296 at 2: 3-8% slower), unless one
// row at a time wastes a large part of its last chunk or handles unaligned
// rows (50,256: +2.5%, 50,257: +14% at 17 sub-chunks and 2 streams).
// SFTM_LOSS_NS=1|2|4 forces a count (tuning, tests).
template <typename T>
int pick_streams(int64_t slice, bool ua) {
  using G = Geo<T>;
  static const int forced = [] {
    const char* v = getenv("SFTM_LOSS_NS");
    return v ? atoi(v) : 0;
  }();
  auto subs = [&](int ns) { return (slice + G::CE / ns - 1) / (G::CE / ns); };
  if ((forced == 1 || forced == 2 || forced == 4) && subs(forced) <= kMaxChunks) return forced;
  if (subs(4) <= 15) return 4;
  if (subs(2) <= 15) return 2;
  const double fill1 = static_cast<double>(slice) / static_cast<double>(subs(1) * G::CE);
  if (subs(2) <= 17 && (ua || fill1 < 0.95)) return 2;
  return 1;
}

template <typename T, bool XP>
int launch_streams(const RowArgs& a, int64_t slice, cudaStream_t s, LaunchInfo* info) {
  switch (pick_streams<T>(slice, false)) {
    case 4: return launch_c<T, 1, XP, false, 4>(a, slice, s, info);
    case 2: return launch_c<T, 1, XP, false, 2>(a, slice, s, info);
  }
  return launch_c<T, 1, XP, false, 1>(a, slice, s, info);
}

template <typename T>
int launch_with(const RowArgs& a, int C, cudaStream_t s, LaunchInfo* info) {
  using G = Geo<T>;
  int64_t slice = (a.V + C - 1) / C;
  slice = (slice + G::EV - 1) / G::EV * G::EV;  // 16-B aligned slice starts
  switch (C) {
    case 1: return launch_streams<T, false>(a, slice, s, info);
    case 2: return launch_c<T, 2>(a, slice, s, info);
    case 3: return launch_c<T, 3>(a, slice, s, info);
    case 4: return launch_c<T, 4>(a, slice, s, info);
    case 8: return launch_c<T, 8>(a, slice, s, info);
  }
  return -2;
}

template <typename T>
int launch_t(const RowArgs& a, cudaStream_t s, LaunchInfo* info) {
  using G = Geo<T>;
  auto nck_of = [&](int C) {
    int64_t slice = (a.V + C - 1) / C;
    slice = (slice + G::EV - 1) / G::EV * G::EV;
    return (slice + G::CE - 1) / G::CE;
  };
  // Rows not on 16-B boundaries (odd vocabulary or stride): one CTA per row in
  // sector coordinates; the row may straddle one extra chunk.
  const bool ua = (reinterpret_cast<uintptr_t>(a.logits) % 16) || ((a.ld * G::es) % 16) || ((a.V * G::es) % 16);
  if (ua) {
    if ((a.V + G::EV - 1 + G::CE - 1) / G::CE > kMaxChunks) return -2;
    switch (pick_streams<T>(a.V + G::EV - 1, true)) {  // a row spans up to EV - 1 more elements
      case 4: return launch_c<T, 1, false, true, 4>(a, a.V, s, info);
      case 2: return launch_c<T, 1, false, true, 2>(a, a.V, s, info);
    }
    return launch_c<T, 1, false, true, 1>(a, a.V, s, info);
  }
  static const int forced = [] {  // tuning knob: SFTM_LOSS_C=1|2|3|4|8
    const char* v = getenv("SFTM_LOSS_C");
    return v ? atoi(v) : 0;
  }();
  if (forced && nck_of(forced) <= kMaxChunks) return launch_with<T>(a, forced, s, info);
  // Smallest cluster whose slice fits the row store: measured on B200, the
  // cluster exchange costs more than the extra run-ahead a narrower slice buys
  // (Qwen3 bf16: C=1 88% vs C=2 84% of HBM copy bandwidth, same box).
  for (int C : {1, 2, 3, 4, 8}) {
    if (nck_of(C) <= kMaxChunks) return launch_with<T>(a, C, s, info);
  }
  return -2;  // not eligible: caller falls back
}

}  // namespace loss

int launch_loss_tmem(const RowArgs& a, cudaStream_t s, LaunchInfo* info) {
  if (a.dtype == 1) return loss::launch_t<uint16_t>(a, s, info);
  return loss::launch_t<float>(a, s, info);
}

bool loss_xp_eligible(int dtype, int64_t Vp, bool ua) {
  // one CTA per row per rank: the whole shard row (in sector coordinates if
  // unaligned) must fit the row store
  auto fits = [&](auto tag) {
    using G = loss::Geo<decltype(tag)>;
    const int64_t span = ua ? Vp + G::EV - 1 : (Vp + G::EV - 1) / G::EV * G::EV;
    return (span + G::CE - 1) / G::CE <= loss::kMaxChunks;
  };
  return dtype == 1 ? fits(uint16_t{}) : fits(float{});
}

int prepare_loss_xp() {
  cudaError_t e = cudaSuccess, ie = cudaSuccess;
  auto one = [&](int r) {
    if (r < 0 && e == cudaSuccess) e = ie;
  };
  one(loss::init_c<uint16_t, 1, true, false, 1>(&ie));
  one(loss::init_c<uint16_t, 1, true, false, 2>(&ie));
  one(loss::init_c<uint16_t, 1, true, false, 4>(&ie));
  one(loss::init_c<uint16_t, 1, true, true, 1>(&ie));
  one(loss::init_c<uint16_t, 1, true, true, 2>(&ie));
  one(loss::init_c<uint16_t, 1, true, true, 4>(&ie));
  one(loss::init_c<float, 1, true, false, 1>(&ie));
  one(loss::init_c<float, 1, true, false, 2>(&ie));
  one(loss::init_c<float, 1, true, false, 4>(&ie));
  one(loss::init_c<float, 1, true, true, 1>(&ie));
  one(loss::init_c<float, 1, true, true, 2>(&ie));
  one(loss::init_c<float, 1, true, true, 4>(&ie));
  return e;
}

int launch_loss_xp(const RowArgs& a, cudaStream_t s, LaunchInfo* info) {
  auto go = [&](auto tag) -> int {
    using T = decltype(tag);
    using G = loss::Geo<T>;
    const bool ua = (reinterpret_cast<uintptr_t>(a.logits) % 16) || ((a.ld * G::es) % 16) || ((a.V * G::es) % 16);
    if (!loss_xp_eligible(a.dtype, a.V, ua)) return -2;
    if (ua) {  // an odd shard width or stride: sector coordinates (the caller checked the dlogits phase)
      switch (loss::pick_streams<T>(a.V + G::EV - 1, true)) {
        case 4: return loss::launch_c<T, 1, true, true, 4>(a, a.V, s, info);
        case 2: return loss::launch_c<T, 1, true, true, 2>(a, a.V, s, info);
      }
      return loss::launch_c<T, 1, true, true, 1>(a, a.V, s, info);
    }
    const int64_t slice = (a.V + G::EV - 1) / G::EV * G::EV;
    return loss::launch_streams<T, true>(a, slice, s, info);
  };
  if (a.dtype == 1) return go(uint16_t{});
  return go(float{});
}

}  // namespace sftm
