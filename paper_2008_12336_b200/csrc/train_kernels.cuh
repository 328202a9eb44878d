// VERSE/NCE training kernels (templates; instantiated per row layout in
// train_v*.cu): the in-memory vertex pass (trainer.py:184-207)
// and the partitioned pool side (bigtrain.py:215-238), sm_100a.
//
// Work decomposition: a "group" of G lanes of one warp owns one source vertex
// at a time.  The source row lives in the group's registers for all of its
// 1+n_neg (resp. B*(1+n_neg)) chained updates and is written back once; the
// sample rows of a chunk of CH samples are gathered up front (their ids are a
// pure function of the counter-based key, so only the positive waits on the
// xadj->adj chain), updated in registers in the reference's order, and
// written back right after their update (Hogwild).  Repeated samples inside a
// chunk are forwarded in registers; a sample equal to the source uses the
// register copy of the source with the reference's aliasing rule.
//
// Arithmetic is the reference's: fp64 dot of fp32 values (products are exact
// in fp64, so only the summation order can differ -- serial in EXACT mode),
// fp64 clamp/sigmoid, score rounded to fp32, unfused fp32 row updates.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>

#include "common.cuh"

namespace gb {
namespace tk {

constexpr int kChunk = 4;  // sample rows gathered per step
constexpr int kBlock = 256;
constexpr double kClamp = 10.0;  // SIGMOID_CLAMP, trainer.py:35

// ---------------------------------------------------------------------------
// Row fragments.  Row::load/store move one embedding row between global
// memory and the registers of the G lanes of a group.
// ---------------------------------------------------------------------------

// dim == 4*G*NV: lane l holds float4 number k*G + l (k < NV); fully coalesced
// 16-byte accesses, one 128-byte line per 8 lanes.
// kMinBlocks: resident 256-thread blocks per SM the register budget targets.
#ifndef GB_MINB_E16
#define GB_MINB_E16 2  // -DGB_MINB_E16=3: 80 registers, ~1 KB spills, C2 2.91 vs 5.22 G upd/s
#endif
constexpr int min_blocks_for(int elems) {
  return elems >= 16 ? GB_MINB_E16 : (elems >= 8 ? 3 : 4);
}

template <int G_, int NV>
struct VecRow {
  static constexpr int G = G_;
  static constexpr int E = 4 * NV;
  static constexpr int kMinBlocks = min_blocks_for(E);
  float x[E];
  __device__ __forceinline__ static bool valid(int, int, int) { return true; }
  __device__ __forceinline__ void load(const float *row, int gl, int) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      // L2-only (.cg): L1-cached rows (.ca) measured 5.10 vs 5.18 G upd/s on C2
      float4 v = __ldcg(reinterpret_cast<const float4 *>(row) + k * G + gl);
      x[4 * k + 0] = v.x;
      x[4 * k + 1] = v.y;
      x[4 * k + 2] = v.z;
      x[4 * k + 3] = v.w;
    }
  }
  __device__ __forceinline__ void store(float *row, int gl, int) const {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      float4 v = make_float4(x[4 * k + 0], x[4 * k + 1], x[4 * k + 2], x[4 * k + 3]);
      __stcg(reinterpret_cast<float4 *>(row) + k * G + gl, v);
    }
  }
  // shared-memory staging (KIND 3): lane gl's 16-byte pieces of a row go to
  // the same positions of a dim-float shared slot by cp.async (no registers
  // held while in flight) and come back to registers when the row trains
  static constexpr bool kStageable = true;
  __device__ __forceinline__ static void stage(float *slot, const float *row, int gl) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const unsigned dst = (unsigned)__cvta_generic_to_shared(slot + 4 * (k * G + gl));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                   "l"(row + 4 * (k * G + gl))
                   : "memory");
    }
  }
  __device__ __forceinline__ void lds(const float *slot, int gl) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const float4 v = reinterpret_cast<const float4 *>(slot)[k * G + gl];
      x[4 * k + 0] = v.x;
      x[4 * k + 1] = v.y;
      x[4 * k + 2] = v.z;
      x[4 * k + 3] = v.w;
    }
  }
  __device__ __forceinline__ void sts(float *slot, int gl) const {
#pragma unroll
    for (int k = 0; k < NV; ++k)
      reinterpret_cast<float4 *>(slot)[k * G + gl] =
          make_float4(x[4 * k + 0], x[4 * k + 1], x[4 * k + 2], x[4 * k + 3]);
  }
  // Hogwild write-back of increments: elements 4k0/4..+3 (one float4) by a
  // 16-byte vector reduction (red.global.add.v4.f32, performed at L2), so
  // concurrent updates of the same row are all applied instead of the last
  // store winning.  Like every f32 global reduction it flushes subnormals.
  static constexpr int kRedWidth = 4;
  __device__ __forceinline__ static void red_part(float *row, int gl, int, int k0,
                                                  const float (&d)[4]) {
    float *p = row + 4 * ((k0 / 4) * G + gl);
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(d[0]),
                 "f"(d[1]), "f"(d[2]), "f"(d[3])
                 : "memory");
  }
  // source-row write-back against the initial copy kept in a shared slot
  // (see SrcKeep): the increments x - s0 are added by vector reductions
  __device__ __forceinline__ void red_delta_slot(float *row, const float *s0, int gl) const {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const float4 o = reinterpret_cast<const float4 *>(s0)[k * G + gl];
      float *p = row + 4 * (k * G + gl);
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p),
                   "f"(__fsub_rn(x[4 * k + 0], o.x)), "f"(__fsub_rn(x[4 * k + 1], o.y)),
                   "f"(__fsub_rn(x[4 * k + 2], o.z)), "f"(__fsub_rn(x[4 * k + 3], o.w))
                   : "memory");
    }
  }
  // Serial dot in ascending element order (the reference's loop order,
  // trainer.py:122-123): element t = 4*(k*G + l) + c.
  __device__ __forceinline__ static double serial_dot(const VecRow &a, const VecRow &b,
                                                      unsigned gmask, int, int) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double p[4];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        p[c] = __dmul_rn((double)a.x[4 * k + c], (double)b.x[4 * k + c]);
#pragma unroll 1
      for (int src = 0; src < G; ++src) {
#pragma unroll
        for (int c = 0; c < 4; ++c) acc = __dadd_rn(acc, __shfl_sync(gmask, p[c], src, G));
      }
    }
    return acc;
  }
};

// Any dim <= 32*NS: G = 32, lane l holds elements k*32 + l (k < NS).
template <int NS>
struct ScalarRow {
  static constexpr int G = 32;
  static constexpr int E = NS;
  static constexpr int kMinBlocks = min_blocks_for(NS);
  float x[E];
  __device__ __forceinline__ static bool valid(int k, int gl, int dim) { return k * 32 + gl < dim; }
  __device__ __forceinline__ void load(const float *row, int gl, int dim) {
#pragma unroll
    for (int k = 0; k < NS; ++k) x[k] = valid(k, gl, dim) ? __ldcg(row + k * 32 + gl) : 0.0f;
  }
  __device__ __forceinline__ void store(float *row, int gl, int dim) const {
#pragma unroll
    for (int k = 0; k < NS; ++k)
      if (valid(k, gl, dim)) __stcg(row + k * 32 + gl, x[k]);
  }
  static constexpr bool kStageable = false;
  static constexpr int kRedWidth = 1;
  __device__ __forceinline__ static void red_part(float *row, int gl, int dim, int k,
                                                  const float (&d)[1]) {
    if (valid(k, gl, dim)) atomicAdd(row + k * 32 + gl, d[0]);
  }
  __device__ __forceinline__ static double serial_dot(const ScalarRow &a, const ScalarRow &b,
                                                      unsigned gmask, int gl, int dim) {
    // The add chain is inherently serial; the shuffles feeding it are not,
    // so they are issued in batches of 8 ahead of the adds that consume
    // them (a shuffle per add on the critical path costs ~4x).
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const double p = __dmul_rn((double)a.x[k], (double)b.x[k]);
      // not unrolled: the chain is add-latency bound either way, and the
      // fully unrolled form made this file the build's long pole
#pragma unroll 1
      for (int s0 = 0; s0 < 32; s0 += 8) {
        double q[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) q[j] = __shfl_sync(gmask, p, s0 + j, 32);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (k * 32 + s0 + j < dim) acc = __dadd_rn(acc, q[j]);
      }
    }
    return acc;
  }
};

// fp64 dot of two fp32 fragments.  Tree mode: per-lane partial sums of exact
// products then an xor butterfly (identical result on every lane).
template <class Row, bool EXACT>
__device__ __forceinline__ double row_dot(const Row &a, const Row &b, unsigned gmask, int gl,
                                          int dim) {
  if (EXACT) return Row::serial_dot(a, b, gmask, gl, dim);
  double p0 = 0.0, p1 = 0.0;  // two chains: halves the dependent DFMA latency
#pragma unroll
  for (int k = 0; k < Row::E; ++k)
    if (Row::valid(k, gl, dim)) {
      if (k & 1)
        p1 = __fma_rn((double)a.x[k], (double)b.x[k], p1);
      else
        p0 = __fma_rn((double)a.x[k], (double)b.x[k], p0);
    }
  double part = __dadd_rn(p0, p1);
#pragma unroll
  for (int off = Row::G / 2; off > 0; off >>= 1)
    part = __dadd_rn(part, __shfl_xor_sync(gmask, part, off, Row::G));
  return part;
}

// score = f32((b - sigmoid(clamp(acc))) * lr)   (trainer.py:124-130).
// fast (non-exact kernels only): the same quantity in fp32 without the
// cancellation of b - sigmoid: lr*sigmoid(-x) for b=1, -lr*sigmoid(x) for
// b=0 (relative error ~1e-7; the fp64 dot is kept).  Cuts the per-update
// dependency chain by the fp64 exp + divide.
__device__ __forceinline__ float nce_score(double acc, double b, double lr, bool &bad,
                                           bool fast = false) {
  bad |= !isfinite(acc);
  if (acc > kClamp)
    acc = kClamp;
  else if (acc < -kClamp)
    acc = -kClamp;
  if (fast) {
    const float x = __double2float_rn(acc);
    const bool positive = b != 0.0;
    const float s = __fdividef(1.0f, 1.0f + expf(positive ? x : -x));
    const float l = __double2float_rn(lr);
    return positive ? s * l : -s * l;
  }
  double sig = __ddiv_rn(1.0, __dadd_rn(1.0, exp(-acc)));
  return __double2float_rn(__dmul_rn(__dsub_rn(b, sig), lr));
}

// Update of a distinct sample row (trainer.py:131-140).
template <class Row>
__device__ __forceinline__ void update_pair(Row &S, Row &R, float sc, bool reuse) {
  if (reuse) {
#pragma unroll
    for (int k = 0; k < Row::E; ++k) S.x[k] = __fadd_rn(S.x[k], __fmul_rn(R.x[k], sc));
#pragma unroll
    for (int k = 0; k < Row::E; ++k) R.x[k] = __fadd_rn(R.x[k], __fmul_rn(S.x[k], sc));
  } else {
#pragma unroll
    for (int k = 0; k < Row::E; ++k) {
      float vo = S.x[k];
      S.x[k] = __fadd_rn(vo, __fmul_rn(R.x[k], sc));
      R.x[k] = __fadd_rn(R.x[k], __fmul_rn(vo, sc));
    }
  }
}

// Update of a distinct sample row followed by its write-back.  atomic:
// the row's increments fl(vo*sc) (fl(S'*sc) with reuse) are added with
// vector reductions instead of storing the updated row -- identical values
// when nobody else touched the row, and no lost updates when somebody did
// (the reference's per-element read-modify-write, trainer.py:131-140, has a
// window of one element; a stored GPU row has one of a whole chunk).
template <class Row>
__device__ __forceinline__ void update_pair_writeback(Row &S, Row &R, float sc, bool reuse,
                                                      bool atomic, float *row, int gl,
                                                      int dim) {
  if (!atomic) {
    update_pair(S, R, sc, reuse);
    R.store(row, gl, dim);
    return;
  }
  constexpr int W = Row::kRedWidth;
  if (reuse) {
#pragma unroll
    for (int k = 0; k < Row::E; ++k) S.x[k] = __fadd_rn(S.x[k], __fmul_rn(R.x[k], sc));
  }
#pragma unroll
  for (int k0 = 0; k0 < Row::E; k0 += W) {
    float d[W];
#pragma unroll
    for (int c = 0; c < W; ++c) {
      const int k = k0 + c;
      const float vo = S.x[k];
      if (!reuse) S.x[k] = __fadd_rn(vo, __fmul_rn(R.x[k], sc));
      d[c] = __fmul_rn(vo, sc);  // with reuse vo is already the updated S
      R.x[k] = __fadd_rn(R.x[k], d[c]);
    }
    Row::red_part(row, gl, dim, k0, d);
  }
}

// Source-row write-back.  Plain store (EXACT kernels, atomic off): the row
// trained in registers replaces the stored one.  atomic: the source's own
// increments S - S0 (S0 = the row as loaded) are added with vector
// reductions instead, so increments other groups reduced into this row while
// it trained (the source is also their sample -- hub rows are everybody's
// positive) are kept rather than overwritten by the store; the reference's
// per-element read-modify-write (trainer.py:131-140) loses at most one
// element's worth.  Uncontended this gives fl(S0 + fl(S - S0)), which is S
// whenever S0 and S are within a factor 2 (Sterbenz) and within an ulp of
// max(|S|,|S0|) otherwise.
#ifndef GB_SRC_DELTA
#define GB_SRC_DELTA 1  // 0: plain source-row stores also with atomic write-back (A/B builds)
#endif
template <class Row>
__device__ __forceinline__ void writeback_source(const Row &S, const Row &S0, float *row, int gl,
                                                 int dim, bool atomic) {
  if (!atomic || !GB_SRC_DELTA) {
    S.store(row, gl, dim);
    return;
  }
  constexpr int W = Row::kRedWidth;
#pragma unroll
  for (int k0 = 0; k0 < Row::E; k0 += W) {
    float d[W];
#pragma unroll
    for (int c = 0; c < W; ++c) d[c] = __fsub_rn(S.x[k0 + c], S0.x[k0 + c]);
    Row::red_part(row, gl, dim, k0, d);
  }
}

// Where a source row's initial copy S0 lives while the group trains it.
// Registers (any layout): 4*NV more live registers per lane -- at d=128 that
// pushed the 2-3 blocks/SM kernels into 80-120 bytes of spills and cost the
// C2 pass 19% (4.33 vs 5.32 G upd/s).  Shared slot (vector layouts): the
// group's lanes store their own float4 pieces of S0 (no cross-lane traffic,
// so no barrier) and read them back for the write-back.
template <class Row, bool SMEM>
struct SrcKeep;

template <class Row>
struct SrcKeep<Row, false> {
  Row S0;
  __device__ __forceinline__ explicit SrcKeep(float *) {}
  __device__ __forceinline__ void save(const Row &S, int) { S0 = S; }
  __device__ __forceinline__ void writeback(const Row &S, float *row, int gl, int dim,
                                            bool atomic) const {
    writeback_source(S, S0, row, gl, dim, atomic);
  }
};

template <class Row>
struct SrcKeep<Row, true> {
  float *slot;
  __device__ __forceinline__ explicit SrcKeep(float *s) : slot(s) {}
  __device__ __forceinline__ void save(const Row &S, int gl) {
    if (GB_SRC_DELTA) S.sts(slot, gl);
  }
  __device__ __forceinline__ void writeback(const Row &S, float *row, int gl, int dim,
                                            bool atomic) const {
    if (atomic && GB_SRC_DELTA)
      S.red_delta_slot(row, slot, gl);
    else
      S.store(row, gl, dim);
  }
};

// The calling group's base in the kernel's dynamic shared memory, `per`
// floats per group.
template <class Row>
__device__ __forceinline__ float *group_smem(int per) {
  extern __shared__ float4 gb_dyn_smem[];
  return reinterpret_cast<float *>(gb_dyn_smem) +
         (size_t)((threadIdx.x >> 5) * (32 / Row::G) + (threadIdx.x & 31) / Row::G) * per;
}

// Self-sample (s == v).  In-place rule of the single-array kernel
// (_train_pass passes M twice): M[v] = fl(fl(vo + vo*sc) + vo*sc).  Load-once
// rule of the two-array pool kernel on a diagonal pair (numba marks the two
// array arguments noalias, bigtrain.py:234): M[i] = fl(vo + vo*sc).  With
// reuse both paths run the two whole-row loops in sequence.
template <class Row>
__device__ __forceinline__ void update_self(Row &S, float sc, bool reuse, bool load_once) {
  if (reuse) {
#pragma unroll
    for (int k = 0; k < Row::E; ++k) {
      float n1 = __fadd_rn(S.x[k], __fmul_rn(S.x[k], sc));
      S.x[k] = __fadd_rn(n1, __fmul_rn(n1, sc));
    }
  } else if (load_once) {
#pragma unroll
    for (int k = 0; k < Row::E; ++k) S.x[k] = __fadd_rn(S.x[k], __fmul_rn(S.x[k], sc));
  } else {
#pragma unroll
    for (int k = 0; k < Row::E; ++k) {
      float vo = S.x[k];
      float d = __fmul_rn(vo, sc);
      S.x[k] = __fadd_rn(__fadd_rn(vo, d), d);
    }
  }
}

struct GroupCtx {
  int gl;          // lane inside the group
  unsigned gmask;  // lanes of this group
};

template <class Row>
__device__ __forceinline__ GroupCtx group_ctx() {
  GroupCtx c;
  const int lane = threadIdx.x & 31;
  c.gl = lane % Row::G;
  c.gmask = Row::G == 32 ? 0xffffffffu : (((1u << Row::G) - 1u) << (lane / Row::G * Row::G));
  return c;
}

// Runs one chunk of up to kChunk samples against the register-resident
// source S.  ids[j] < 0 marks an unused slot; bit j of pos_mask marks a
// positive (b = 1).  Sample rows are gathered first, then updated in order
// with forwarding of repeated ids, and stored right after their update.
template <class Row>
__device__ __forceinline__ void load_chunk(Row (&R)[kChunk], int64_t src_row,
                                           const int32_t (&ids)[kChunk],
                                           const float *__restrict__ Mtgt, int dim,
                                           bool self_possible, const GroupCtx &g) {
#pragma unroll
  for (int j = 0; j < kChunk; ++j)
    if (ids[j] >= 0 && !(self_possible && ids[j] == src_row))
      R[j].load(Mtgt + (int64_t)ids[j] * dim, g.gl, dim);
}

// The update half of run_chunk on rows already gathered by load_chunk.
template <class Row, bool EXACT>
__device__ __forceinline__ void compute_chunk(Row &S, Row (&R)[kChunk], int64_t src_row,
                                              const int32_t (&ids)[kChunk], unsigned pos_mask,
                                              float *__restrict__ Mtgt, int dim, double lr,
                                              bool reuse, bool self_possible, bool load_once,
                                              const GroupCtx &g, bool &bad, bool fast,
                                              bool atomic) {
  // Repeated ids are rare (~C(4,2)/n per chunk): the row forwarding runs
  // behind one branch per chunk instead of as predicated copies on every
  // update (those cost ~10% of the pair kernel's instructions).
  bool dup = false;
#pragma unroll
  for (int j = 0; j < kChunk; ++j)
#pragma unroll
    for (int jj = j + 1; jj < kChunk; ++jj)
      if (ids[j] >= 0 && ids[j] == ids[jj]) dup = true;
#pragma unroll
  for (int j = 0; j < kChunk; ++j) {
    const int32_t s = ids[j];
    if (s < 0) continue;
    const double b = (pos_mask >> j) & 1u ? 1.0 : 0.0;
    if (self_possible && s == src_row) {
      double acc = row_dot<Row, EXACT>(S, S, g.gmask, g.gl, dim);
      float sc = nce_score(acc, b, lr, bad, fast && !EXACT);
      update_self(S, sc, reuse, load_once);
      continue;
    }
    double acc = row_dot<Row, EXACT>(S, R[j], g.gmask, g.gl, dim);
    float sc = nce_score(acc, b, lr, bad, fast && !EXACT);
    update_pair_writeback(S, R[j], sc, reuse, atomic && !EXACT, Mtgt + (int64_t)s * dim, g.gl,
                          dim);
    if (dup) {
#pragma unroll
      for (int jj = j + 1; jj < kChunk; ++jj)
        if (ids[jj] == s) R[jj] = R[j];
    }
  }
}

template <class Row, bool EXACT>
__device__ __forceinline__ void run_chunk(Row &S, int64_t src_row, const int32_t (&ids)[kChunk],
                                          unsigned pos_mask, float *__restrict__ Mtgt, int dim,
                                          double lr, bool reuse, bool self_possible,
                                          bool load_once, const GroupCtx &g, bool &bad,
                                          bool fast = false, bool atomic = false) {
  Row R[kChunk];
  load_chunk<Row>(R, src_row, ids, Mtgt, dim, self_possible, g);
  compute_chunk<Row, EXACT>(S, R, src_row, ids, pos_mask, Mtgt, dim, lr, reuse, self_possible,
                            load_once, g, bad, fast, atomic);
}

// run_chunk with the sample rows staged in the group's shared slots (KIND 3,
// vector layouts only): slot 0 holds the source's initial copy (SrcKeep),
// samples 1..3 of the chunk are cp.async-staged into slots 1..3 (no
// registers held while in flight) and come to registers one at a time when
// they train; sample 0 (the positive, whose address arrives last through the
// xadj -> adj chain) is loaded straight into registers.
// Walk (PPR passes): ids[0] is resolved by the given walk after rows 1..3
// are in flight, so the walk's dependent xadj/adj loads overlap their copies.
struct NoWalk {
  __device__ __forceinline__ int32_t operator()() const { return -1; }
};

template <class Row, class Walk = NoWalk>
__device__ __forceinline__ void run_chunk_staged(Row &S, int64_t src_row,
                                                 int32_t (&ids)[kChunk], unsigned pos_mask,
                                                 float *__restrict__ Mtgt, int dim, double lr,
                                                 float *slots, const GroupCtx &g, bool &bad,
                                                 bool fast, bool atomic, bool self_possible = true,
                                                 bool load_once = false, Walk walk = Walk(),
                                                 bool do_walk = false) {
#pragma unroll
  for (int j = 1; j < kChunk; ++j)
    if (ids[j] >= 0 && !(self_possible && ids[j] == src_row))
      Row::stage(slots + j * dim, Mtgt + (int64_t)ids[j] * dim, g.gl);
  asm volatile("cp.async.commit_group;" ::: "memory");
  if (do_walk) ids[0] = walk();
  Row R;
  if (ids[0] >= 0 && !(self_possible && ids[0] == src_row))
    R.load(Mtgt + (int64_t)ids[0] * dim, g.gl, dim);
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  bool dup = false;
#pragma unroll
  for (int j = 0; j < kChunk; ++j)
#pragma unroll
    for (int jj = j + 1; jj < kChunk; ++jj)
      if (ids[j] >= 0 && ids[j] == ids[jj]) dup = true;
#pragma unroll
  for (int j = 0; j < kChunk; ++j) {
    const int32_t s = ids[j];
    if (s < 0) continue;
    const double b = (pos_mask >> j) & 1u ? 1.0 : 0.0;
    if (self_possible && s == src_row) {
      double acc = row_dot<Row, false>(S, S, g.gmask, g.gl, dim);
      float sc = nce_score(acc, b, lr, bad, fast);
      update_self(S, sc, false, load_once);
      continue;
    }
    if (j > 0) R.lds(slots + j * dim, g.gl);
    double acc = row_dot<Row, false>(S, R, g.gmask, g.gl, dim);
    float sc = nce_score(acc, b, lr, bad, fast);
    update_pair_writeback(S, R, sc, false, atomic, Mtgt + (int64_t)s * dim, g.gl, dim);
    if (dup) {
#pragma unroll
      for (int jj = j + 1; jj < kChunk; ++jj)
        if (ids[jj] == s) R.sts(slots + jj * dim, g.gl);
    }
  }
}

// Batched-dot chunk (non-exact, latency variant).  With distinct sample ids
// that all differ from the source, S before update k is
// S + sum_{j<k} sc_j R_j, so the k-th dot is
//   d_k = S.R_k + sum_{j<k} sc_j (R_j.R_k)
// -- all 4 + 6 fp64 dot products are independent and reduce together (one
// butterfly, full ILP); only a short scalar chain of sigmoids remains.  The
// row updates are then applied element by element in the reference's order
// (identical fp32 operations).  d_k differs from the dot of the fp32-rounded
// updated row by rounding only (~1e-7 relative), within the 1e-5 bar.
// Returns false (nothing done) when ids repeat or hit the source; the caller
// then takes the sequential path.
template <class Row>
__device__ __forceinline__ bool batched_chunk(Row &S, int64_t src_row, const int32_t (&ids)[kChunk],
                                              unsigned pos_mask, float *__restrict__ Mtgt,
                                              int dim, double lr, bool reuse, const GroupCtx &g,
                                              bool &bad, bool fast, bool atomic = false) {
  static_assert(kChunk == 4, "batched_chunk assumes 4 samples");
  bool simple = true;
#pragma unroll
  for (int j = 0; j < kChunk; ++j) {
    if (ids[j] >= 0 && ids[j] == src_row) simple = false;
#pragma unroll
    for (int k = j + 1; k < kChunk; ++k)
      if (ids[j] >= 0 && ids[j] == ids[k]) simple = false;
  }
  if (!simple) return false;
  Row R[kChunk];
#pragma unroll
  for (int j = 0; j < kChunk; ++j)
    if (ids[j] >= 0) R[j].load(Mtgt + (int64_t)ids[j] * dim, g.gl, dim);
  // 10 partial dots: q[j] = S.R_j, q[4 + pair(j,k)] = R_j.R_k (j < k)
  double q[10];
#pragma unroll
  for (int t = 0; t < 10; ++t) q[t] = 0.0;
#pragma unroll
  for (int e = 0; e < Row::E; ++e) {
    if (!Row::valid(e, g.gl, dim)) continue;
    const double s = (double)S.x[e];
    const double r0 = (double)R[0].x[e], r1 = (double)R[1].x[e];
    const double r2 = (double)R[2].x[e], r3 = (double)R[3].x[e];
    q[0] = __fma_rn(s, r0, q[0]);
    q[1] = __fma_rn(s, r1, q[1]);
    q[2] = __fma_rn(s, r2, q[2]);
    q[3] = __fma_rn(s, r3, q[3]);
    q[4] = __fma_rn(r0, r1, q[4]);
    q[5] = __fma_rn(r0, r2, q[5]);
    q[6] = __fma_rn(r0, r3, q[6]);
    q[7] = __fma_rn(r1, r2, q[7]);
    q[8] = __fma_rn(r1, r3, q[8]);
    q[9] = __fma_rn(r2, r3, q[9]);
  }
#pragma unroll
  for (int off = Row::G / 2; off > 0; off >>= 1) {
#pragma unroll
    for (int t = 0; t < 10; ++t) q[t] = __dadd_rn(q[t], __shfl_xor_sync(g.gmask, q[t], off, Row::G));
  }
  float sc[kChunk];
  const int gram[kChunk][kChunk] = {{-1, 4, 5, 6}, {4, -1, 7, 8}, {5, 7, -1, 9}, {6, 8, 9, -1}};
#pragma unroll
  for (int k = 0; k < kChunk; ++k) {
    sc[k] = 0.0f;
    if (ids[k] < 0) continue;
    double d = q[k];
#pragma unroll
    for (int j = 0; j < k; ++j)
      if (ids[j] >= 0) d = __fma_rn((double)sc[j], q[gram[j][k]], d);
    sc[k] = nce_score(d, (pos_mask >> k) & 1u ? 1.0 : 0.0, lr, bad, fast);
  }
#pragma unroll
  for (int j = 0; j < kChunk; ++j) {
    if (ids[j] < 0) continue;
    update_pair_writeback(S, R[j], sc[j], reuse, atomic, Mtgt + (int64_t)ids[j] * dim, g.gl,
                          dim);
  }
  return true;
}

// Work slots.  Group `gid` (slot g of warp w; gpw = 32/G groups per warp) of
// the `eff` enabled groups handles items gid, gid + eff, ...  The loop bound
// `base` is the same for every group of a warp, so the groups of a warp walk
// their items in lockstep and stay converged.
template <class Row>
struct Slots {
  int64_t warp_base;  // gid of the warp's first group
  int64_t gid;
  int64_t eff;
  bool enabled;
  __device__ __forceinline__ Slots(int64_t max_groups) {
    constexpr int gpw = 32 / Row::G;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t total = ((int64_t)gridDim.x * blockDim.x >> 5) * gpw;
    eff = max_groups > 0 ? min(total, max_groups) : total;
    warp_base = warp * gpw;
    gid = warp_base + (threadIdx.x & 31) / Row::G;
    enabled = gid < eff;
  }
  __device__ __forceinline__ bool warp_idle() const { return warp_base >= eff; }
};

// ---------------------------------------------------------------------------
// In-memory passes (trainer.py:184-207).
// ---------------------------------------------------------------------------
struct PassArgs {
  int64_t V;
  const int64_t *__restrict__ xadj;
  const int32_t *__restrict__ adj;
  const int32_t *__restrict__ sources;  // non-isolated vertices, ascending (may be null)
  int64_t n_sources;
  float *M;
  int dim;
  int n_neg;
  uint64_t seed;
  uint64_t stream;
  int64_t pass_begin;
  int64_t n_passes;
  int64_t ppe;
  const float *__restrict__ lr;
  bool reuse;
  bool fast;
  bool atomic;
  // > 0: positives from VERSE's personalized-PageRank similarity with this
  // continue probability instead of the adjacency similarity (run-time-flag
  // kernels only; see ppr_positive).  float, in the bools' padding: growing
  // the struct changed ptxas's allocation of the HOT KIND 3 pass (stack 24
  // -> 40 bytes, -5% on C2)
  float ppr_alpha;
  int64_t max_groups;
  int64_t *status;
};

// Positive sample of source v (deg > 0).  Adjacency similarity (the
// reference, trainer.py:203): a uniform neighbour.  PPR similarity (VERSE's
// sample_rw, the measure GOSH's paper names beside adjacency):
// start at v; while a uniform draw is below alpha, step to a uniform
// neighbour of the current vertex (stop early at a sink); the sample is the
// vertex reached -- v itself with probability 1 - alpha (a self-sample,
// trained with the self rule).  Walk draws use counters from kPprCtr up, far
// from the negatives' 1..n_neg; walks are capped at kPprMaxSteps.
constexpr uint64_t kPprCtr = 1ull << 40;
constexpr int kPprMaxSteps = 64;

__device__ __forceinline__ int32_t ppr_positive(const int64_t *__restrict__ xadj,
                                                const int32_t *__restrict__ adj, int64_t v,
                                                double alpha, uint64_t key) {
  int64_t u = v;
  for (int t = 0; t < kPprMaxSteps; ++t) {
    if (!(draw_unit(key, kPprCtr + 2 * (uint64_t)t) < alpha)) break;
    const int64_t x0 = __ldg(xadj + u);
    const int64_t d = __ldg(xadj + u + 1) - x0;
    if (d == 0) break;
    u = __ldg(adj + x0 + draw_below(key, kPprCtr + 2 * (uint64_t)t + 1, d));
  }
  return (int32_t)u;
}

template <bool HOT>
__device__ __forceinline__ int32_t positive_sample(const PassArgs &a, int64_t v, int64_t x0,
                                                   int64_t deg, uint64_t key) {
  if constexpr (!HOT) {
    if (a.ppr_alpha > 0.0f) return ppr_positive(a.xadj, a.adj, v, (double)a.ppr_alpha, key);
  }
  return __ldg(a.adj + x0 + draw_below(key, 0, deg));  // trainer.py:203
}

// Index half of a source: v, the positive (xadj -> adj), the first chunk of
// negatives, the RNG key and the pass's lr.  Read-only inputs, so computing
// it early never changes results.
struct SourceIdx {
  int32_t v;
  int32_t ids[kChunk];  // positive + up to kChunk-1 negatives
  uint64_t key;
  float lr;
  int32_t epoch;
  bool active;
};

__device__ __forceinline__ void fetch_source(const PassArgs &a, int64_t p, int64_t i, bool ok,
                                             SourceIdx &d) {
  d.active = ok;
  d.v = 0;
  d.key = 0;
  d.lr = 0.0f;
  d.epoch = 0;
#pragma unroll
  for (int j = 0; j < kChunk; ++j) d.ids[j] = -1;
  if (!ok) return;
  const int64_t v = a.sources ? (int64_t)__ldg(a.sources + i) : i;
  const int64_t x0 = __ldg(a.xadj + v);
  const int64_t deg = __ldg(a.xadj + v + 1) - x0;
  if (deg == 0) {  // isolated sources are skipped (trainer.py:198-200)
    d.active = false;
    return;
  }
  d.v = (int32_t)v;
  d.key = stream_key(a.seed, a.stream, (uint64_t)p, (uint64_t)v);
  d.epoch = (int32_t)(p / a.ppe);
  d.lr = __ldg(a.lr + d.epoch);
  const int nsamp = 1 + a.n_neg;
#pragma unroll
  for (int j = 0; j < kChunk; ++j) {
    if (j >= nsamp)
      d.ids[j] = -1;
    else if (j == 0)  // positive (trainer.py:203, or a PPR walk)
      d.ids[j] = positive_sample<false>(a, v, x0, deg, d.key);
    else  // negatives: uniform over V (trainer.py:205-206)
      d.ids[j] = (int32_t)draw_below(d.key, (uint64_t)j, a.V);
  }
}

// Lane k's SourceIdx, broadcast to its whole group.
__device__ __forceinline__ SourceIdx shfl_source(const SourceIdx &d, int k, unsigned gmask,
                                                 int G) {
  SourceIdx o;
  o.active = __shfl_sync(gmask, (int)d.active, k, G) != 0;
  o.v = __shfl_sync(gmask, d.v, k, G);
#pragma unroll
  for (int j = 0; j < kChunk; ++j) o.ids[j] = __shfl_sync(gmask, d.ids[j], k, G);
  o.key = __shfl_sync(gmask, d.key, k, G);
  o.lr = __shfl_sync(gmask, d.lr, k, G);
  o.epoch = __shfl_sync(gmask, d.epoch, k, G);
  return o;
}

// Row half of a source: gather, chained updates, write-back.
template <class Row, bool EXACT, bool BATCH, bool HOT, bool F64S = false>
__device__ __forceinline__ void train_source(const PassArgs &a, const GroupCtx &g,
                                             const SourceIdx &d, bool &bad, int &first_bad) {
  const int nsamp = 1 + a.n_neg;
  const bool fast = HOT ? !F64S : a.fast, atomic = HOT || a.atomic, reuse = !HOT && a.reuse;
  const double lr = (double)d.lr;
  Row S;
  S.load(a.M + (int64_t)d.v * a.dim, g.gl, a.dim);
  const Row S0 = S;
  bool bad_src = false;
  if constexpr (BATCH) {
    if (EXACT ||
        !batched_chunk<Row>(S, d.v, d.ids, 1u, a.M, a.dim, lr, reuse, g, bad_src, fast, atomic))
      run_chunk<Row, EXACT>(S, d.v, d.ids, 1u, a.M, a.dim, lr, reuse, true, false, g, bad_src,
                            fast, atomic);
  }
  // one run_chunk call site for the non-batched form (code size / registers)
  for (int c0 = BATCH ? kChunk : 0; c0 < nsamp; c0 += kChunk) {
    int32_t ids[kChunk];
#pragma unroll
    for (int j = 0; j < kChunk; ++j)
      ids[j] = c0 == 0 ? d.ids[j]
                       : (c0 + j < nsamp ? (int32_t)draw_below(d.key, (uint64_t)(c0 + j), a.V)
                                         : -1);
    run_chunk<Row, EXACT>(S, d.v, ids, c0 == 0 ? 1u : 0u, a.M, a.dim, lr, reuse, true, false, g,
                          bad_src, fast, atomic);
  }
  writeback_source(S, S0, a.M + (int64_t)d.v * a.dim, g.gl, a.dim, atomic && !EXACT);
  if (bad_src) {
    bad = true;
    first_bad = min(first_bad, d.epoch);
  }
}

// Each group walks a sequence of steps s = 0, 1, ...: step s is pass
// pass_begin + s / spp, item warp_base + (s % spp)*eff + (its slot), with spp
// (steps per pass) uniform across the warp so its groups stay in lockstep.
// Indices come in batches: lane l of a group fetches step s0 + l, then the
// group trains the G sources one by one from shuffled indices -- the
// sources -> xadj -> key -> adj chain and the RNG run once per G sources,
// G-way parallel, instead of redundantly on every lane for every source.
// KIND 0: throughput variant (index chain inline per source); 1: latency
// variant (capped launches): batched index fetch, batched-dot chunks and one
// block per SM worth of registers.  (The batched index fetch with sequential
// dots at full occupancy measured 4.77 vs 5.15 G upd/s on C2 and was
// dropped.)  HOT = true: the default flags (fast
// sigmoid, vector-reduction write-back, no reuse) fixed at compile time --
// the runtime-flag branches otherwise triple the unrolled code, and the
// i-cache misses that cost show up as the top ncu stall (no_instructions).
// F64S (with HOT): the same compile-time flags but the reference's fp64
// sigmoid and divide (trainer.py:118) instead of the fp32 one.  PPRW (KIND 3
// only): positives from the PPR walk (ppr_positive) instead of a uniform
// neighbour.
template <class Row, bool EXACT, int KIND, bool HOT, bool F64S = false, bool PPRW = false>
__global__ void __launch_bounds__(kBlock, (KIND == 1 || EXACT) ? 1 : (KIND == 3 ? 3 : Row::kMinBlocks))
    train_passes_kernel(PassArgs a) {
  constexpr int G = Row::G;
  constexpr bool BATCH = KIND == 1;
  // KIND 0 / 2 keep the source's initial copy in a shared slot per group
  // (launched with kBlock / G * dim floats of dynamic shared memory)
  constexpr bool kS0Smem = Row::kStageable && !EXACT;
  const bool fast = HOT ? !F64S : a.fast, atomic = HOT || a.atomic, reuse = !HOT && a.reuse;
  const GroupCtx g = group_ctx<Row>();
  const Slots<Row> sl(a.max_groups);
  if (sl.warp_idle()) return;
  bool bad = false;
  int first_bad = INT_MAX;
  const int64_t n = a.sources ? a.n_sources : a.V;
  if (sl.warp_base >= n) return;
  const int64_t lane_off = sl.gid - sl.warp_base;
  if constexpr (KIND == 3) {
    // HOT throughput pass with the sample rows staged in shared memory
    // (dynamic: kBlock / G groups x kChunk slots x dim floats): ~80 registers
    // instead of 128, so 3 blocks per SM hold 1.5x the sources in flight
    float *slots = group_smem<Row>(kChunk * a.dim);
    SrcKeep<Row, true> keep(slots);  // slot 0
    const int nsamp = 1 + a.n_neg;
    for (int64_t p = a.pass_begin; p < a.pass_begin + a.n_passes; ++p) {
      const int epoch = (int)(p / a.ppe);
      const double lr = (double)__ldg(a.lr + epoch);
      for (int64_t base = sl.warp_base; base < n; base += sl.eff) {
        const int64_t i = base + lane_off;
        if (!sl.enabled || i >= n) continue;
        const int64_t v = a.sources ? (int64_t)__ldg(a.sources + i) : i;
        const int64_t x0 = __ldg(a.xadj + v);
        const int64_t deg = __ldg(a.xadj + v + 1) - x0;
        if (deg == 0) continue;
        const uint64_t key = stream_key(a.seed, a.stream, (uint64_t)p, (uint64_t)v);
        Row S;
        S.load(a.M + v * (int64_t)a.dim, g.gl, a.dim);
        keep.save(S, g.gl);
        bool bad_src = false;
        for (int c0 = 0; c0 < nsamp; c0 += kChunk) {
          int32_t ids[kChunk];
#pragma unroll
          for (int j = 0; j < kChunk; ++j) {
            const int idx = c0 + j;
            if (idx >= nsamp)
              ids[j] = -1;
            else if (idx == 0)  // PPRW: resolved by the walk inside the chunk
              ids[j] = PPRW ? 0 : __ldg(a.adj + x0 + draw_below(key, 0, deg));
            else
              ids[j] = (int32_t)draw_below(key, (uint64_t)idx, a.V);
          }
          if constexpr (PPRW) {
            const auto walk = [&]() {
              return ppr_positive(a.xadj, a.adj, v, (double)a.ppr_alpha, key);
            };
            run_chunk_staged<Row>(S, v, ids, c0 == 0 ? 1u : 0u, a.M, a.dim, lr, slots, g,
                                  bad_src, fast, atomic, true, false, walk, c0 == 0);
          } else {
            run_chunk_staged<Row>(S, v, ids, c0 == 0 ? 1u : 0u, a.M, a.dim, lr, slots, g,
                                  bad_src, fast, atomic);
          }
        }
        keep.writeback(S, a.M + v * (int64_t)a.dim, g.gl, a.dim, atomic && !EXACT);
        if (bad_src) {
          bad = true;
          first_bad = min(first_bad, epoch);
        }
      }
    }
  } else if constexpr (KIND == 0) {
    // throughput variant (full occupancy, HBM-bound): the index chain is
    // computed inline per source -- its latency hides behind other warps and
    // this keeps the kernel within 128 registers (2 blocks per SM)
    const int nsamp = 1 + a.n_neg;
    SrcKeep<Row, kS0Smem> keep(kS0Smem ? group_smem<Row>(a.dim) : nullptr);
    for (int64_t p = a.pass_begin; p < a.pass_begin + a.n_passes; ++p) {
      const int epoch = (int)(p / a.ppe);
      const double lr = (double)__ldg(a.lr + epoch);
      for (int64_t base = sl.warp_base; base < n; base += sl.eff) {
        const int64_t i = base + lane_off;
        if (!sl.enabled || i >= n) continue;
        const int64_t v = a.sources ? (int64_t)__ldg(a.sources + i) : i;
        const int64_t x0 = __ldg(a.xadj + v);
        const int64_t deg = __ldg(a.xadj + v + 1) - x0;
        if (deg == 0) continue;  // isolated sources are skipped (trainer.py:198-200)
        const uint64_t key = stream_key(a.seed, a.stream, (uint64_t)p, (uint64_t)v);
        Row S;
        S.load(a.M + v * (int64_t)a.dim, g.gl, a.dim);
        keep.save(S, g.gl);
        bool bad_src = false;
        for (int c0 = 0; c0 < nsamp; c0 += kChunk) {
          int32_t ids[kChunk];
#pragma unroll
          for (int j = 0; j < kChunk; ++j) {
            const int idx = c0 + j;
            if (idx >= nsamp)
              ids[j] = -1;
            else if (idx == 0)  // positive: uniform neighbour (trainer.py:203) or PPR
              ids[j] = positive_sample<HOT>(a, v, x0, deg, key);
            else  // negatives: uniform over V (trainer.py:205-206)
              ids[j] = (int32_t)draw_below(key, (uint64_t)idx, a.V);
          }
          run_chunk<Row, EXACT>(S, v, ids, c0 == 0 ? 1u : 0u, a.M, a.dim, lr, reuse, true, false,
                                g, bad_src, fast, atomic);
        }
        keep.writeback(S, a.M + v * (int64_t)a.dim, g.gl, a.dim, atomic && !EXACT);
        if (bad_src) {
          bad = true;
          first_bad = min(first_bad, epoch);
        }
      }
    }
  } else if constexpr (KIND == 2) {
    // throughput variant with the index chain one source ahead: the
    // sources -> xadj -> adj loads of the next source are issued right after
    // this source's row gathers, so their latency overlaps the gathers'
    // instead of following the updates (+1.3% on C2: 5.21 vs 5.14 G upd/s,
    // but 5.17 vs 5.64 and 3.84 vs 4.28 on C3's levels 1 and 2, so opt-in:
    // GB_PASS_AHEAD=1; deeper index pipelines spill at 128 registers, and
    // lane-batched source id loads measured 4.95)
    const int nsamp = 1 + a.n_neg;
    SrcKeep<Row, kS0Smem> keep(kS0Smem ? group_smem<Row>(a.dim) : nullptr);
    const int64_t spp = (n - sl.warp_base + sl.eff - 1) / sl.eff;  // steps per pass
    const int64_t total = spp * a.n_passes;
    // step cursor (uniform across the warp): pass p, item base
    int64_t cp = a.pass_begin, cbase = sl.warp_base;
    int cepoch = (int)(cp / a.ppe);
    float clr = __ldg(a.lr + cepoch);
    struct Idx {
      int32_t v, pos;
      uint64_t key;
      float lr;
      int epoch;
      bool ok;
    };
    auto fetch = [&](int64_t t) {
      Idx d;
      d.ok = false;
      d.v = 0;
      d.pos = -1;
      d.key = 0;
      d.lr = clr;
      d.epoch = cepoch;
      if (t < total) {
        const int64_t i = cbase + lane_off;
        if (sl.enabled && i < n) {
          const int64_t v = a.sources ? (int64_t)__ldg(a.sources + i) : i;
          const int64_t x0 = __ldg(a.xadj + v);
          const int64_t deg = __ldg(a.xadj + v + 1) - x0;
          if (deg > 0) {  // isolated sources are skipped (trainer.py:198-200)
            d.ok = true;
            d.v = (int32_t)v;
            d.key = stream_key(a.seed, a.stream, (uint64_t)cp, (uint64_t)v);
            d.pos = __ldg(a.adj + x0 + draw_below(d.key, 0, deg));  // trainer.py:203
          }
        }
        cbase += sl.eff;  // advance the cursor
        if (cbase >= sl.warp_base + spp * sl.eff) {
          cbase = sl.warp_base;
          ++cp;
          cepoch = (int)(cp / a.ppe);
          clr = cp < a.pass_begin + a.n_passes ? __ldg(a.lr + cepoch) : 0.0f;
        }
      }
      return d;
    };
    Idx cur = fetch(0);
    for (int64_t t = 0; t < total; ++t) {
      if (!cur.ok) {
        cur = fetch(t + 1);
        continue;
      }
      const double lr = (double)cur.lr;
      const int64_t v = cur.v;
      Row S;
      S.load(a.M + v * (int64_t)a.dim, g.gl, a.dim);
      keep.save(S, g.gl);
      int32_t ids[kChunk];
#pragma unroll
      for (int j = 0; j < kChunk; ++j)  // negatives: uniform over V (trainer.py:205-206)
        ids[j] = j == 0 ? cur.pos : (j < nsamp ? (int32_t)draw_below(cur.key, (uint64_t)j, a.V) : -1);
      Row R[kChunk];
      load_chunk<Row>(R, v, ids, a.M, a.dim, true, g);
      const Idx nxt = fetch(t + 1);
      bool bad_src = false;
      // one compute_chunk call site (a second one for the n_neg >= kChunk
      // chunks doubled the code and spilled 1 KB per thread)
      for (int c0 = 0; c0 < nsamp; c0 += kChunk) {
        if (c0 > 0) {
#pragma unroll
          for (int j = 0; j < kChunk; ++j)
            ids[j] = c0 + j < nsamp ? (int32_t)draw_below(cur.key, (uint64_t)(c0 + j), a.V) : -1;
          load_chunk<Row>(R, v, ids, a.M, a.dim, true, g);
        }
        compute_chunk<Row, EXACT>(S, R, v, ids, c0 == 0 ? 1u : 0u, a.M, a.dim, lr, reuse, true,
                                  false, g, bad_src, fast, atomic);
      }
      keep.writeback(S, a.M + v * (int64_t)a.dim, g.gl, a.dim, atomic && !EXACT);
      if (bad_src) {
        bad = true;
        first_bad = min(first_bad, cur.epoch);
      }
      cur = nxt;
    }
  } else {
    const int64_t spp = (n - sl.warp_base + sl.eff - 1) / sl.eff;
    const int64_t total = spp * a.n_passes;
    for (int64_t s0 = 0; s0 < total; s0 += G) {
      SourceIdx mine;
      {
        const int64_t s = s0 + g.gl;
        const int64_t q = s / spp;
        const int64_t i = sl.warp_base + (s - q * spp) * sl.eff + lane_off;
        fetch_source(a, a.pass_begin + q, i, s < total && sl.enabled && i < n, mine);
      }
      const int kmax = (int)(total - s0 < G ? total - s0 : G);
#pragma unroll 1
      for (int k = 0; k < kmax; ++k) {
        const SourceIdx d = shfl_source(mine, k, g.gmask, G);
        if (d.active) train_source<Row, EXACT, BATCH, HOT, F64S>(a, g, d, bad, first_bad);
      }
    }
  }
  if (bad && g.gl == 0) {
    atomicOr(reinterpret_cast<unsigned long long *>(a.status), 1ull);
    atomicMin(reinterpret_cast<long long *>(a.status + 1), (long long)first_bad);
  }
}

// ---------------------------------------------------------------------------
// Pool side (bigtrain.py:215-238), optionally drawing the pool on the fly
// (bigtrain.py:164-196) from the device CSR.
// ---------------------------------------------------------------------------
struct PairParam {
  uint64_t seed;
  double lr;
};

struct PoolArgs {
  float *Msrc;
  float *Mtgt;
  int dim;
  const int32_t *__restrict__ targets;
  int64_t n_src;
  int B;
  int64_t lo_t;
  int64_t n_t;
  int n_neg;
  double lr;
  uint64_t seed;
  uint64_t side;
  const int64_t *__restrict__ xadj;
  const int32_t *__restrict__ adj;
  int64_t lo_s;
  uint64_t pool_side;
  // compacted sources (gb_fill_pool_compact): source k of the launch is
  // src_list[k] (local id), its pool row is targets[k*B ..], and only the
  // first min(n_src, *n_list) entries are live.  Null: source k is k.
  const int32_t *__restrict__ src_list;
  const int64_t *__restrict__ n_list;
  // balanced pools (gb_fill_pool_balanced): entry k draws bal_npos[k]
  // positives from adj[bal_first[k] .. + bal_cnt[k]) on the fly; null: off
  const int64_t *__restrict__ bal_first;
  const int32_t *__restrict__ bal_cnt;
  const int32_t *__restrict__ bal_npos;
  bool reuse;
  bool fast;
  bool atomic;
  int64_t max_groups;
  int64_t *status;
  // device-resident {seed, lr} overriding the two arguments above when set
  // (*_dp entry points: a captured rotation's launches read this rotation's
  // values from a table the host rewrites before each graph replay)
  const PairParam *__restrict__ param;
};

// lower_bound over adj[lo, hi) (rows are sorted ascending).
__device__ __forceinline__ int64_t lower_bound_adj(const int32_t *__restrict__ adj, int64_t lo,
                                                   int64_t hi, int64_t x) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if ((int64_t)__ldg(adj + mid) < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// MODE 0: flags at run time; 1 / 2: HOT flags (see train_passes_kernel) on
// an off-diagonal / diagonal pair, so the self-sample branch is compiled out
// of the off-diagonal kernel.  (Batched-dot chunks as in the latency pass
// variant need 242 registers here: at one block per SM they measured 4.95
// vs 6.03 G upd/s, so the pair kernel keeps the sequential dots.  Rolling
// gathers -- each row slot refilled with the next chunk's sample right after
// its update, stale duplicates re-read -- measured 5.40 vs 6.32: the refill
// loads wait on the write-back reductions still reading the slot's
// registers; with the refill delayed by one sample, 5.14 vs 6.26.  Rows
// staged in shared memory as in the KIND 3 pass: 6.36-6.39 vs 6.24-6.26 at
// d=128 but 2.99 vs 3.27 at d=256; the next chunk cp.async-staged while the
// current one trains from registers: 6.12-6.14 vs 6.27 and 3.13-3.16 vs
// 3.25 -- neither adopted.)
//
// Sample ids come in windows of kWin = 2 chunks: lane l of the group draws
// flat samples l, l + G, ... of the window (the positive from the pool or the
// CSR, a negative from the counter-based key), and the chunks take them by
// shuffle -- the RNG runs once per sample instead of once per lane.
template <class Row, bool EXACT, int MODE, bool F64S = false>
__global__ void __launch_bounds__(kBlock, EXACT ? 1 : Row::kMinBlocks) train_pool_kernel(PoolArgs a) {
  constexpr int G = Row::G;
  constexpr int kWin = 2 * kChunk;
  // the source's initial copy in a shared slot per group (kBlock / G * dim
  // floats of dynamic shared memory), as in train_passes_kernel
  constexpr bool kS0Smem = Row::kStageable && !EXACT;
  constexpr int PL = (kWin + G - 1) / G;  // window samples per lane
  const GroupCtx g = group_ctx<Row>();
  const Slots<Row> sl(a.max_groups);
  if (sl.warp_idle()) return;
  constexpr bool HOT = MODE != 0;
  constexpr bool BALC = MODE >= 3;  // HOT on balanced pools
  const bool fast = HOT ? !F64S : a.fast, atomic = HOT || a.atomic, reuse = !HOT && a.reuse;
  const bool diagonal = HOT ? (MODE == 2 || MODE == 4) : a.Msrc == a.Mtgt;
  const bool bal = BALC || (!HOT && a.bal_npos != nullptr);
  const int per_t = 1 + a.n_neg;
  const int total = a.B * per_t;
  const int gbase = (int)(threadIdx.x & 31) - g.gl;
  const int64_t n = a.src_list ? min(a.n_src, *a.n_list) : a.n_src;
  const uint64_t seed = a.param ? a.param->seed : a.seed;
  const double lr = a.param ? a.param->lr : a.lr;
  bool bad = false;
  unsigned long long pos_count = 0, neg_count = 0;

  for (int64_t base = sl.warp_base; base < n; base += sl.eff) {
    const int64_t k = base + (sl.gid - sl.warp_base);
    if (!sl.enabled || k >= n) continue;
    const int64_t i = a.src_list ? (int64_t)__ldg(a.src_list + k) : k;
    // HOT kernels run on materialized pools only (the fused draw stays in
    // the MODE 0 kernel), so their code carries no binary searches
    const bool mat = !bal && (HOT || a.targets != nullptr);
    const int32_t *trow = mat ? a.targets + k * a.B : nullptr;
    // pool side of this source: the materialized row, the balanced entry
    // or the fused draw
    int64_t first = 0, cnt = 0;
    uint64_t pkey = 0;
    int npos = 0, tot = total;
    if (bal) {
      first = __ldg(a.bal_first + k);
      cnt = __ldg(a.bal_cnt + k);
      npos = __ldg(a.bal_npos + k);
      pkey = stream_key(seed, a.pool_side, 0, (uint64_t)(a.lo_s + i));
      tot = total + max(0, npos - a.B);
    } else if (!HOT && trow == nullptr) {
      const int64_t v = a.lo_s + i;
      const int64_t e0 = __ldg(a.xadj + v), e1 = __ldg(a.xadj + v + 1);
      first = lower_bound_adj(a.adj, e0, e1, a.lo_t);
      cnt = lower_bound_adj(a.adj, first, e1, a.lo_t + a.n_t) - first;
      if (cnt == 0) continue;  // every slot is -1
      pkey = stream_key(seed, a.pool_side, 0, (uint64_t)v);
    }
    const uint64_t key = stream_key(seed, a.side, 1, (uint64_t)i);
    Row S;
    SrcKeep<Row, kS0Smem> keep(kS0Smem ? group_smem<Row>(a.dim) : nullptr);
    bool loaded = false;
    // lane's samples of window c0 (ids, -1 = none) and the window's positive
    // bits.  (An L2 prefetch of the next window's rows was measured and
    // bought nothing: 6.21 vs 6.23 G upd/s.)
    int32_t mine[PL];
    unsigned wpos = 0;
    auto draw_window = [&](int c0) {
      wpos = 0;
#pragma unroll
      for (int p = 0; p < PL; ++p) {
        const int w = g.gl + p * G;
        const int f = c0 + w;
        int32_t id = -1;
        bool pos = false;
        if (w < kWin && f < tot) {
          const int t = f / per_t, q = f - t * per_t;
          if (bal) {
            // slots t < B: positive iff t < npos, then n_neg negatives; the
            // positives beyond B follow one per sample (gb_fill_pool_balanced)
            if (f >= total) {
              id = (int32_t)(__ldg(a.adj + first + draw_below(pkey, (uint64_t)(a.B + f - total), cnt)) - a.lo_t);
              pos = true;
            } else if (q == 0) {
              if (t < npos) {
                id = (int32_t)(__ldg(a.adj + first + draw_below(pkey, (uint64_t)t, cnt)) - a.lo_t);
                pos = true;
              }
            } else {
              id = (int32_t)draw_below(key, (uint64_t)(t * a.n_neg + (q - 1)), a.n_t);
            }
          } else if (mat) {
            const int32_t tgt = __ldg(trow + t);
            if (tgt >= 0) {  // absent slot: no positive, no negatives
              if (q == 0) {
                id = (int32_t)(tgt - a.lo_t);
                pos = true;
              } else {
                id = (int32_t)draw_below(key, (uint64_t)(t * a.n_neg + (q - 1)), a.n_t);
              }
            }
          } else if (q == 0) {  // fused pool: cnt > 0, so no slot is absent
            id = (int32_t)(__ldg(a.adj + first + draw_below(pkey, (uint64_t)t, cnt)) - a.lo_t);
            pos = true;
          } else {
            id = (int32_t)draw_below(key, (uint64_t)(t * a.n_neg + (q - 1)), a.n_t);
          }
        }
        mine[p] = id;
        unsigned b = __ballot_sync(g.gmask, pos);
        if (G < 32) b = (b >> gbase) & ((1u << (G < 32 ? G : 0)) - 1u);
        wpos |= b << (p * G);
      }
    };
    for (int c0 = 0; c0 < tot; c0 += kWin) {
      draw_window(c0);
      int32_t win[kWin];
#pragma unroll
      for (int w = 0; w < kWin; ++w) win[w] = __shfl_sync(g.gmask, mine[w / G], w % G, G);
      const unsigned wpos_cur = wpos;
#pragma unroll 1
      for (int h = 0; h < kWin / kChunk; ++h) {  // not unrolled: one copy of the chunk code
        int32_t ids[kChunk];
#pragma unroll
        for (int j = 0; j < kChunk; ++j) ids[j] = h ? win[kChunk + j] : win[j];
        if (!(ids[0] >= 0 || ids[1] >= 0 || ids[2] >= 0 || ids[3] >= 0)) continue;
        if (!loaded) {
          S.load(a.Msrc + i * (int64_t)a.dim, g.gl, a.dim);
          keep.save(S, g.gl);
          loaded = true;
        }
        const unsigned pos_mask = (wpos_cur >> (h * kChunk)) & ((1u << kChunk) - 1u);
        pos_count += __popc(pos_mask);
        neg_count += (ids[0] >= 0) + (ids[1] >= 0) + (ids[2] >= 0) + (ids[3] >= 0) -
                     __popc(pos_mask);
        run_chunk<Row, EXACT>(S, i, ids, pos_mask, a.Mtgt, a.dim, lr, reuse, diagonal, true, g,
                              bad, fast, atomic);
      }
    }
    if (loaded) keep.writeback(S, a.Msrc + i * (int64_t)a.dim, g.gl, a.dim, atomic && !EXACT);
  }
  if (g.gl == 0) {
    if (pos_count) atomicAdd(reinterpret_cast<unsigned long long *>(a.status + 2), pos_count);
    if (neg_count) atomicAdd(reinterpret_cast<unsigned long long *>(a.status + 3), neg_count);
    if (bad) {
      atomicOr(reinterpret_cast<unsigned long long *>(a.status), 1ull);
      atomicMin(reinterpret_cast<long long *>(a.status + 1), 0ll);
    }
  }
}

// ---------------------------------------------------------------------------
// Fixed sample lists: source src[i] is updated against samples[i*k + j]
// (j ascending, -1 = skip) with label labels[j]; single-array semantics of
// update_embedding (trainer.py:137-142).  One group chains one source.
// ---------------------------------------------------------------------------
struct ListArgs {
  float *M;
  int dim;
  int64_t n_src;
  const int64_t *__restrict__ src;
  int k;
  const int64_t *__restrict__ samples;
  const int8_t *__restrict__ labels;
  double lr;
  bool reuse;
  bool fast;
  bool atomic;
  int64_t max_groups;
  int64_t *status;
};

template <class Row, bool EXACT>
__global__ void __launch_bounds__(kBlock, EXACT ? 1 : Row::kMinBlocks) apply_lists_kernel(ListArgs a) {
  const GroupCtx g = group_ctx<Row>();
  const Slots<Row> sl(a.max_groups);
  if (sl.warp_idle()) return;
  bool bad = false;
  for (int64_t base = sl.warp_base; base < a.n_src; base += sl.eff) {
    const int64_t i = base + (sl.gid - sl.warp_base);
    if (!sl.enabled || i >= a.n_src) continue;
    const int64_t v = a.src[i];
    Row S;
    S.load(a.M + v * (int64_t)a.dim, g.gl, a.dim);
    const Row S0 = S;
    for (int c0 = 0; c0 < a.k; c0 += kChunk) {
      int32_t ids[kChunk];
      unsigned pos_mask = 0;
#pragma unroll
      for (int j = 0; j < kChunk; ++j) {
        const int idx = c0 + j;
        ids[j] = idx < a.k ? (int32_t)a.samples[i * a.k + idx] : -1;
        if (idx < a.k && a.labels[idx]) pos_mask |= 1u << j;
      }
      run_chunk<Row, EXACT>(S, v, ids, pos_mask, a.M, a.dim, a.lr, a.reuse, true, false, g, bad,
                            a.fast, a.atomic);
    }
    writeback_source(S, S0, a.M + v * (int64_t)a.dim, g.gl, a.dim, a.atomic && !EXACT);
  }
  if (bad && g.gl == 0) {
    atomicOr(reinterpret_cast<unsigned long long *>(a.status), 1ull);
    atomicMin(reinterpret_cast<long long *>(a.status + 1), 0ll);
  }
}

// ---------------------------------------------------------------------------
// Per-layout kernel table.
// ---------------------------------------------------------------------------
using PassFn = void (*)(PassArgs);
using PoolFn = void (*)(PoolArgs);
using ListFn = void (*)(ListArgs);

struct Variant {
  int G = 0;
  bool s0_smem = false;  // pass KIND 0/2 and pool kernels take kBlock/G*dim floats of smem
  PassFn pass = nullptr;       // throughput (full occupancy)
  PassFn pass_pipe = nullptr;  // latency (capped launches)
  PoolFn pool = nullptr;
  ListFn lists = nullptr;
  // HOT instantiations (default flags fixed at compile time); null if absent
  PassFn pass_hot = nullptr;
  PassFn pass_ahead_hot = nullptr;  // KIND 2
  PassFn pass_staged_hot = nullptr;  // KIND 3
  PassFn pass_staged_hot_f64 = nullptr;  // KIND 3 with the fp64 sigmoid
  PassFn pass_staged_hot_ppr = nullptr;  // KIND 3, fp64 sigmoid, PPR positives
  PassFn pass_hot_f64 = nullptr;
  PassFn pass_ahead_hot_f64 = nullptr;
  PassFn pass_pipe_hot_f64 = nullptr;
  PoolFn pool_hot_f64 = nullptr;
  PoolFn pool_hot_diag_f64 = nullptr;
  PoolFn pool_bal_hot_f64 = nullptr;
  PoolFn pool_bal_hot_diag_f64 = nullptr;
  PassFn pass_pipe_hot = nullptr;
  PoolFn pool_hot = nullptr;       // off-diagonal pair
  PoolFn pool_hot_diag = nullptr;  // diagonal pair (Msrc == Mtgt)
  PoolFn pool_bal_hot = nullptr;   // balanced pools
  PoolFn pool_bal_hot_diag = nullptr;
};

template <class Row, bool EXACT, bool WITH_HOT = false>
Variant make_variant() {
  Variant v;
  v.G = Row::G;
  v.s0_smem = Row::kStageable && !EXACT;
  v.pass = train_passes_kernel<Row, EXACT, 0, false>;
  v.pass_pipe = train_passes_kernel<Row, EXACT, 1, false>;
  v.pool = train_pool_kernel<Row, EXACT, 0>;
  v.lists = apply_lists_kernel<Row, EXACT>;
  if constexpr (WITH_HOT && !EXACT) {
    v.pass_hot = train_passes_kernel<Row, false, 0, true>;
    v.pass_ahead_hot = train_passes_kernel<Row, false, 2, true>;
    v.pass_staged_hot = train_passes_kernel<Row, false, 3, true>;
    v.pass_staged_hot_f64 = train_passes_kernel<Row, false, 3, true, true>;
    v.pass_staged_hot_ppr = train_passes_kernel<Row, false, 3, true, true, true>;
    v.pass_hot_f64 = train_passes_kernel<Row, false, 0, true, true>;
    v.pass_ahead_hot_f64 = train_passes_kernel<Row, false, 2, true, true>;
    v.pass_pipe_hot_f64 = train_passes_kernel<Row, false, 1, true, true>;
    v.pool_hot_f64 = train_pool_kernel<Row, false, 1, true>;
    v.pool_hot_diag_f64 = train_pool_kernel<Row, false, 2, true>;
    v.pool_bal_hot_f64 = train_pool_kernel<Row, false, 3, true>;
    v.pool_bal_hot_diag_f64 = train_pool_kernel<Row, false, 4, true>;
    v.pass_pipe_hot = train_passes_kernel<Row, false, 1, true>;
    v.pool_hot = train_pool_kernel<Row, false, 1>;
    v.pool_hot_diag = train_pool_kernel<Row, false, 2>;
    v.pool_bal_hot = train_pool_kernel<Row, false, 3>;
    v.pool_bal_hot_diag = train_pool_kernel<Row, false, 4>;
  }
  return v;
}

// Fast layouts (tree dot): VecRow<G, NV>, dim = 4*G*NV.
Variant vec_variant(int G, int NV);  // returns G == 0 if not instantiated
// Any-dim layouts (ScalarRow<NS>, dim <= 32*NS); exact = serial dot.
Variant scalar_variant(int NS, bool exact);

}  // namespace tk
}  // namespace gb
