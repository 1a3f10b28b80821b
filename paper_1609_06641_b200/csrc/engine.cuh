// engine.cuh — compile-time tile engine for the batched dyadic WHT (CHW).
//
// Model.  The reference cascade (transforms.hpp:126-143) is, op
// for op, the level-synchronous butterfly network "for t = 0..m-1 combine
// (j, j|2^t) as ((a+b)k, (a-b)k), then y[i] = v[rev_m(i)]" (
// restated in oracle/chw_oracle.c:chw_oracle_network_f64 and pinned bitwise by
// tests/test_oracle.py).  A kernel therefore only decides WHERE each index bit
// of a tile lives at each moment:
//
//   * a "tile" is a set of 2^T elements addressed by T tile-local bits;
//   * a Layout assigns every tile bit to a register-index bit (the first E_BITS
//     entries), a lane bit (next 5) or a warp bit (the rest);
//   * a butterfly on tile bit b is register arithmetic when b is a register bit,
//     a warp shuffle when b is a lane bit;
//   * changing Layout is a round trip through shared memory under an XOR swizzle
//     chosen so that the lanes of each access hit distinct banks;
//   * a position Map turns tile bits into global element offsets (natural order
//     on the way in, bit-reversed = dyadic order on the way out), so the
//     reversal is folded into the store addresses.
//
// Everything about a tile is resolved at compile time: register indices are
// constants after unrolling, so the thread's data never leaves registers except
// for the explicit shared-memory transposes.
#pragma once

#include <cstdint>
#include <type_traits>
#include <utility>
#include <cuda_bf16.h>

#define CHW_HD __host__ __device__ __forceinline__

namespace chwb {

// ---------------------------------------------------------------------------
// Compile-time integer lists.
// ---------------------------------------------------------------------------
template <int... V>
struct BL {
  static constexpr int N = sizeof...(V);
  CHW_HD static constexpr int at(int k) {
    constexpr int a[sizeof...(V) + 1] = {V..., -1};
    return a[k];
  }
};

// Concatenation of two list types (anything with N and at()).
template <class A, class B>
struct Cat {
  static constexpr int N = A::N + B::N;
  CHW_HD static constexpr int at(int k) { return k < A::N ? A::at(k) : B::at(k - A::N); }
};

// Compile-time loop: f(std::integral_constant<int, I>) for I = 0..N-1.  The
// register-indexed loops below use it so every per-register offset is a C++
// constant expression (folded by the front end) instead of an unrolled loop
// that NVVM has to simplify — E = 128 tiles compile an order of magnitude
// faster this way.
template <class F, int... I>
__device__ __forceinline__ void static_for_impl(F& f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
}

template <class L>
CHW_HD constexpr int find(int v) {
  for (int k = 0; k < L::N; ++k)
    if (L::at(k) == v) return k;
  return -1;
}

// ---------------------------------------------------------------------------
// Layout: Reg lists the tile bit held by each register-index bit; Thr lists the
// tile bit held by each thread-index bit (lanes = first 5 entries).
// ---------------------------------------------------------------------------
template <class Reg, class Thr>
struct Layout {
  using R = Reg;
  using Th = Thr;
  static constexpr int E_BITS = Reg::N;
  static constexpr int E = 1 << E_BITS;
  static constexpr int T_BITS = Reg::N + Thr::N;
  static constexpr int NT = 1 << Thr::N;
  CHW_HD static constexpr int slot(int tile_bit) { return find<Reg>(tile_bit); }
};

// Tile bit -> element position maps.
struct IdMap {
  CHW_HD static constexpr int pos(int k) { return k; }
};
// Dyadic (Paley) output order: in-row bit b -> bit M-1-b (orderings.hpp:45-52,
// natural_to_dyadic :70-78); row bits (>= M) unchanged.
template <int M>
struct RevMap {
  CHW_HD static constexpr int pos(int k) { return k < M ? M - 1 - k : k; }
};

// Sequency output order (orderings.hpp:82-102): out[s] =
// dyadic[gray(s)], i.e. the element at dyadic in-row position p is stored at
// gray^-1(p) = p ^ p>>1 ^ p>>2 ^ ... — a GF(2)-linear map of the position, not
// a bit permutation.  A map with kLinear applies lin() to the position that
// Base::pos() gives; lin() is linear (XOR-additive), so a store address is
// lin(thread part ^ tile-outer part) ^ lin(register part): one runtime value
// per thread and a compile-time constant per register (stores are scalar:
// the low address bits depend on every position bit).
template <class Base, int M>
struct SeqMap {
  static constexpr bool kLinear = true;
  CHW_HD static constexpr int pos(int k) { return Base::pos(k); }
  CHW_HD static constexpr uint32_t lin(uint32_t p) {
    const uint32_t mask = M >= 32 ? 0xffffffffu : ((1u << M) - 1u);
    uint32_t lo = p & mask;
    lo ^= lo >> 1;
    lo ^= lo >> 2;
    lo ^= lo >> 4;
    lo ^= lo >> 8;
    lo ^= lo >> 16;
    return lo | (p & ~mask);
  }
};
template <class Map, class = void>
struct IsLinearMap : std::false_type {};
template <class Map>
struct IsLinearMap<Map, std::void_t<decltype(Map::kLinear)>> : std::integral_constant<bool, Map::kLinear> {};

template <class L, class Map>
CHW_HD constexpr uint32_t reg_off(int r) {
  uint32_t o = 0;
  for (int k = 0; k < L::E_BITS; ++k)
    if ((r >> k) & 1) o |= 1u << Map::pos(L::R::at(k));
  return o;
}

template <class L, class Map>
__device__ __forceinline__ uint32_t thr_off(uint32_t t) {
  uint32_t o = 0;
#pragma unroll
  for (int k = 0; k < L::Th::N; ++k) o |= ((t >> k) & 1u) << Map::pos(L::Th::at(k));
  return o;
}

// Bits a thread offset may set (so register offsets can be ADDed when disjoint).
template <class L, class Map>
CHW_HD constexpr uint32_t thr_mask() {
  uint32_t o = 0;
  for (int k = 0; k < L::Th::N; ++k) o |= 1u << Map::pos(L::Th::at(k));
  return o;
}

// Largest VB such that tile bits at element positions 0..VB-1 are held by
// register bits (so 2^VB consecutive elements sit in registers of one thread).
template <class L, class Map>
CHW_HD constexpr int vec_bits(int cap) {
  int vb = 0;
  while (vb < cap) {
    bool found = false;
    for (int k = 0; k < L::E_BITS; ++k)
      if (Map::pos(L::R::at(k)) == vb) found = true;
    if (!found) break;
    ++vb;
  }
  return vb;
}
// Register-index bit holding element-position bit q.
template <class L, class Map>
CHW_HD constexpr int reg_bit_for_pos(int q) {
  for (int k = 0; k < L::E_BITS; ++k)
    if (Map::pos(L::R::at(k)) == q) return k;
  return -1;
}
// Register index of the q-th element of the vector whose first element is r.
template <class L, class Map>
CHW_HD constexpr int vec_elem(int r, int q, int vb) {
  int x = r;
  for (int b = 0; b < vb; ++b)
    if ((q >> b) & 1) x |= 1 << reg_bit_for_pos<L, Map>(b);
  return x;
}
// Does register index r start a vector (all vector bits clear)?
template <class L, class Map>
CHW_HD constexpr bool vec_head(int r, int vb) {
  for (int b = 0; b < vb; ++b)
    if ((r >> reg_bit_for_pos<L, Map>(b)) & 1) return false;
  return true;
}

// ---------------------------------------------------------------------------
// Linear XOR swizzle on word addresses: y = x ^ sum_i bit(x, src_i) << dst_i.
// ---------------------------------------------------------------------------
template <int... P>
struct Swz {
  CHW_HD static constexpr uint32_t apply(uint32_t x) {
    constexpr int a[sizeof...(P) + 2] = {P..., -1, -1};
    uint32_t y = x;
    for (int i = 0; i + 1 < (int)sizeof...(P); i += 2) y ^= ((x >> a[i]) & 1u) << a[i + 1];
    return y;
  }
  // Bits the swizzle may touch given possible input bits `mask`.
  CHW_HD static constexpr uint32_t image(uint32_t mask) {
    constexpr int a[sizeof...(P) + 2] = {P..., -1, -1};
    uint32_t y = mask;
    for (int i = 0; i + 1 < (int)sizeof...(P); i += 2)
      if ((mask >> a[i]) & 1u) y |= 1u << a[i + 1];
    return y;
  }
};
using NoSwz = Swz<>;

// ---------------------------------------------------------------------------
// Element I/O types.
// ---------------------------------------------------------------------------
template <class T>
struct IoTraits;
template <>
struct IoTraits<double> {
  using C = double;  // compute type
  static constexpr int VMAX = 1;  // log2 elements per 16 B
};
template <>
struct IoTraits<float> {
  using C = float;
  static constexpr int VMAX = 2;
};
template <>
struct IoTraits<__nv_bfloat16> {
  using C = float;
  static constexpr int VMAX = 3;
};

// Cache operators for global traffic: kNC = read-only path (ld.global.nc),
// kStream = evict-first streaming (ld/st.global.cs: data touched once),
// kL2 = cache in L2 only (ld/st.global.cg: the fused kernels' L2-resident
// intermediate, never served from a possibly stale L1).
enum class Cache : int { kNC = 0, kStream = 1, kL2 = 2, kL2Last = 3 };

// kL2Last: L1-bypassing access with an L2 evict_last policy (createpolicy), for
// intermediates that must survive in L2 while streaming traffic passes by.
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float ld_l2last(const float* ptr) {
  float v;
  asm volatile("ld.global.cg.L2::cache_hint.f32 %0, [%1], %2;"
               : "=f"(v)
               : "l"(ptr), "l"(l2_evict_last_policy()));
  return v;
}
__device__ __forceinline__ float4 ld_l2last(const float4* ptr) {
  float4 v;
  asm volatile("ld.global.cg.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(ptr), "l"(l2_evict_last_policy()));
  return v;
}
__device__ __forceinline__ void st_l2last(float* ptr, float v) {
  asm volatile("st.global.cg.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(ptr), "f"(v),
               "l"(l2_evict_last_policy())
               : "memory");
}
__device__ __forceinline__ void st_l2last(float4* ptr, float4 v) {
  asm volatile("st.global.cg.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(l2_evict_last_policy())
               : "memory");
}

template <Cache CO, class V>
__device__ __forceinline__ V gload(const V* p) {
  if constexpr (CO == Cache::kNC)
    return __ldg(p);
  else if constexpr (CO == Cache::kStream)
    return __ldcs(p);
  else if constexpr (CO == Cache::kL2Last)
    return ld_l2last(p);
  else
    return __ldcg(p);
}
template <Cache CO, class V>
__device__ __forceinline__ void gstore(V* p, V v) {
  if constexpr (CO == Cache::kStream)
    __stcs(p, v);
  else if constexpr (CO == Cache::kL2)
    __stcg(p, v);
  else if constexpr (CO == Cache::kL2Last)
    st_l2last(p, v);
  else
    *p = v;
}

// Vector load of 2^VB consecutive T converted to C.
template <class T, int VB, Cache CO = Cache::kNC>
struct VecIO;

template <Cache CO>
struct VecIO<double, 0, CO> {
  __device__ __forceinline__ static void ld(const double* p, double* o) { o[0] = gload<CO>(p); }
  __device__ __forceinline__ static void st(double* p, const double* v) { gstore<CO>(p, v[0]); }
};
template <Cache CO>
struct VecIO<double, 1, CO> {
  __device__ __forceinline__ static void ld(const double* p, double* o) {
    const double2 v = gload<CO>(reinterpret_cast<const double2*>(p));
    o[0] = v.x;
    o[1] = v.y;
  }
  __device__ __forceinline__ static void st(double* p, const double* v) {
    gstore<CO>(reinterpret_cast<double2*>(p), make_double2(v[0], v[1]));
  }
};
template <Cache CO>
struct VecIO<float, 0, CO> {
  __device__ __forceinline__ static void ld(const float* p, float* o) { o[0] = gload<CO>(p); }
  __device__ __forceinline__ static void st(float* p, const float* v) { gstore<CO>(p, v[0]); }
};
template <Cache CO>
struct VecIO<float, 1, CO> {
  __device__ __forceinline__ static void ld(const float* p, float* o) {
    const float2 v = gload<CO>(reinterpret_cast<const float2*>(p));
    o[0] = v.x;
    o[1] = v.y;
  }
  __device__ __forceinline__ static void st(float* p, const float* v) {
    gstore<CO>(reinterpret_cast<float2*>(p), make_float2(v[0], v[1]));
  }
};
template <Cache CO>
struct VecIO<float, 2, CO> {
  __device__ __forceinline__ static void ld(const float* p, float* o) {
    const float4 v = gload<CO>(reinterpret_cast<const float4*>(p));
    o[0] = v.x;
    o[1] = v.y;
    o[2] = v.z;
    o[3] = v.w;
  }
  __device__ __forceinline__ static void st(float* p, const float* v) {
    gstore<CO>(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
  }
};
// bf16: 2^VB elements packed; converted to/from fp32 registers.
template <int VB, Cache CO>
struct VecIO<__nv_bfloat16, VB, CO> {
  static constexpr int N = 1 << VB;
  __device__ __forceinline__ static void ld(const __nv_bfloat16* p, float* o) {
    if constexpr (VB == 0) {
      o[0] = __uint_as_float(((uint32_t)gload<CO>(reinterpret_cast<const unsigned short*>(p))) << 16);
    } else if constexpr (VB == 1) {
      const uint32_t w = gload<CO>(reinterpret_cast<const unsigned int*>(p));
      o[0] = __uint_as_float(w << 16);
      o[1] = __uint_as_float(w & 0xffff0000u);
    } else if constexpr (VB == 2) {
      const uint2 w = gload<CO>(reinterpret_cast<const uint2*>(p));
      o[0] = __uint_as_float(w.x << 16);
      o[1] = __uint_as_float(w.x & 0xffff0000u);
      o[2] = __uint_as_float(w.y << 16);
      o[3] = __uint_as_float(w.y & 0xffff0000u);
    } else {
      const uint4 w = gload<CO>(reinterpret_cast<const uint4*>(p));
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        o[2 * i] = __uint_as_float(ws[i] << 16);
        o[2 * i + 1] = __uint_as_float(ws[i] & 0xffff0000u);
      }
    }
  }
  __device__ __forceinline__ static uint32_t pack2(float a, float b) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);  // round-to-nearest-even
    return *reinterpret_cast<const uint32_t*>(&h);
  }
  __device__ __forceinline__ static void st(__nv_bfloat16* p, const float* v) {
    if constexpr (VB == 0) {
      const __nv_bfloat16 h = __float2bfloat16_rn(v[0]);
      gstore<CO>(reinterpret_cast<unsigned short*>(p), *reinterpret_cast<const unsigned short*>(&h));
    } else if constexpr (VB == 1) {
      gstore<CO>(reinterpret_cast<unsigned int*>(p), (unsigned int)pack2(v[0], v[1]));
    } else if constexpr (VB == 2) {
      gstore<CO>(reinterpret_cast<uint2*>(p), make_uint2(pack2(v[0], v[1]), pack2(v[2], v[3])));
    } else {
      gstore<CO>(reinterpret_cast<uint4*>(p),
                 make_uint4(pack2(v[0], v[1]), pack2(v[2], v[3]), pack2(v[4], v[5]), pack2(v[6], v[7])));
    }
  }
};

// int64 support (the reference's exact integer path).
template <>
struct IoTraits<long long> {
  using C = long long;
  static constexpr int VMAX = 1;
};
template <Cache CO>
struct VecIO<long long, 0, CO> {
  __device__ __forceinline__ static void ld(const long long* p, long long* o) { o[0] = gload<CO>(p); }
  __device__ __forceinline__ static void st(long long* p, const long long* v) { gstore<CO>(p, v[0]); }
};
template <Cache CO>
struct VecIO<long long, 1, CO> {
  __device__ __forceinline__ static void ld(const long long* p, long long* o) {
    const longlong2 v = gload<CO>(reinterpret_cast<const longlong2*>(p));
    o[0] = v.x;
    o[1] = v.y;
  }
  __device__ __forceinline__ static void st(long long* p, const long long* v) {
    longlong2 x;
    x.x = v[0];
    x.y = v[1];
    gstore<CO>(reinterpret_cast<longlong2*>(p), x);
  }
};
// Shared-memory vector access of 2^VB compute-type words.
template <class C, int VB>
struct SmemVec;
template <class C>
struct SmemVec<C, 0> {
  __device__ __forceinline__ static void st(C* p, const C* v) { *p = v[0]; }
  __device__ __forceinline__ static void ld(const C* p, C* o) { o[0] = *p; }
};
template <>
struct SmemVec<float, 1> {
  __device__ __forceinline__ static void st(float* p, const float* v) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  }
  __device__ __forceinline__ static void ld(const float* p, float* o) {
    const float2 x = *reinterpret_cast<const float2*>(p);
    o[0] = x.x;
    o[1] = x.y;
  }
};
template <>
struct SmemVec<float, 2> {
  __device__ __forceinline__ static void st(float* p, const float* v) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
  __device__ __forceinline__ static void ld(const float* p, float* o) {
    const float4 x = *reinterpret_cast<const float4*>(p);
    o[0] = x.x;
    o[1] = x.y;
    o[2] = x.z;
    o[3] = x.w;
  }
};
template <>
struct SmemVec<double, 1> {
  __device__ __forceinline__ static void st(double* p, const double* v) {
    *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
  }
  __device__ __forceinline__ static void ld(const double* p, double* o) {
    const double2 x = *reinterpret_cast<const double2*>(p);
    o[0] = x.x;
    o[1] = x.y;
  }
};

template <>
struct SmemVec<long long, 1> {
  __device__ __forceinline__ static void st(long long* p, const long long* v) {
    longlong2 x;
    x.x = v[0];
    x.y = v[1];
    *reinterpret_cast<longlong2*>(p) = x;
  }
  __device__ __forceinline__ static void ld(const long long* p, long long* o) {
    const longlong2 x = *reinterpret_cast<const longlong2*>(p);
    o[0] = x.x;
    o[1] = x.y;
  }
};
// ---------------------------------------------------------------------------
// Butterflies.
// ---------------------------------------------------------------------------
// Reference scaling constant (common.hpp:29).
constexpr double kInvSqrt2 = 0.70710678118654752440;

// One butterfly with the reference operand order: lower index a, upper b,
// s = (a+b)k, d = (a-b)k (transforms.hpp:62-70).  PER_STAGE applies k in every
// butterfly (the f64 Orthonormal path, bit-exact with the reference); otherwise
// scaling is deferred to a single multiply at the store.  The _rn intrinsics
// forbid FMA contraction so the op sequence is the reference's exactly.
template <bool PER_STAGE>
__device__ __forceinline__ void bf(double& a, double& b) {
  const double s = __dadd_rn(a, b);
  const double d = __dsub_rn(a, b);
  if constexpr (PER_STAGE) {
    a = __dmul_rn(s, kInvSqrt2);
    b = __dmul_rn(d, kInvSqrt2);
  } else {
    a = s;
    b = d;
  }
}
template <bool PER_STAGE>
__device__ __forceinline__ void bf(float& a, float& b) {
  const float s = __fadd_rn(a, b);
  const float d = __fsub_rn(a, b);
  if constexpr (PER_STAGE) {
    a = __fmul_rn(s, (float)kInvSqrt2);
    b = __fmul_rn(d, (float)kInvSqrt2);
  } else {
    a = s;
    b = d;
  }
}

// Integer butterfly: exact, two's-complement (inputs bounded as common.hpp:17-18).
template <bool PER_STAGE>
__device__ __forceinline__ void bf(long long& a, long long& b) {
  const long long s = a + b;
  const long long d = a - b;
  a = s;
  b = d;
}


// Two fp32 butterflies in one packed FADD2 pair (sm_100 add/sub.rn.f32x2):
// (a0, a1) +/- (b0, b1), each lane rounded exactly like __fadd_rn/__fsub_rn.
__device__ __forceinline__ void bf2(float& a0, float& a1, float& b0, float& b1) {
  uint64_t A, B, S, D;
  asm("mov.b64 %0, {%1, %2};" : "=l"(A) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(B) : "f"(b0), "f"(b1));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(S) : "l"(A), "l"(B));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(D) : "l"(A), "l"(B));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(S));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(b0), "=f"(b1) : "l"(D));
}

// Two fp32 products a*s, b*s in one packed FMUL2 (sm_100 mul.rn.f32x2),
// each rounded exactly like __fmul_rn.
__device__ __forceinline__ void mul2(float& a, float& b, float s) {
  uint64_t A, S, P;
  asm("mov.b64 %0, {%1, %2};" : "=l"(A) : "f"(a), "f"(b));
  asm("mov.b64 %0, {%1, %1};" : "=l"(S) : "f"(s));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(P) : "l"(A), "l"(S));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(P));
}

// The butterfly between the two halves of one register pair, (a, b) ->
// (a + b, a - b), as ONE packed FFMA2: (b, b) * (1, -1) + (a, a).  ptxas folds
// the broadcasts into operand modifiers (FFMA2 R, Rb.F32, Rc.F32x2, Ra.F32); a
// product by +-1 is exact, so each half is rounded exactly like
// __fadd_rn / __fsub_rn.  Used for register bit 0, which the (r, r|1) pairing
// of the other bits cannot pack (64 scalar FADDs less per 128-value level).
#ifndef CHW_BF_SELF
#define CHW_BF_SELF 1
#endif
__device__ __forceinline__ void bf_self(float& a, float& b) {
  uint64_t LL, HH, C, D;
  asm("mov.b64 %0, {%1, %1};" : "=l"(LL) : "f"(a));
  asm("mov.b64 %0, {%1, %1};" : "=l"(HH) : "f"(b));
  asm("mov.b64 %0, {%1, %2};" : "=l"(C) : "f"(1.0f), "f"(-1.0f));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(D) : "l"(HH), "l"(C), "l"(LL));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(D));
}

// Butterflies on the listed tile bits, in list order (order matters only for
// bit-exact f64; f32/bf16 are order-free up to rounding).  fp32 butterflies on
// register bits other than bit 0 are issued in pairs (registers r, r^1) as
// packed FADD2 instructions: half the FP issue slots, identical results.
template <class L, class Bits, bool PER_STAGE, class C>
__device__ __forceinline__ void butterflies(C (&v)[L::E]) {
  if constexpr (std::is_same<C, float>::value && !PER_STAGE && L::E >= 4) {
    static_for<Bits::N>([&](auto I) {
      constexpr int k = L::slot(Bits::at(decltype(I)::value));
      static_assert(k >= 0, "butterfly bit must be a register bit");
      if constexpr (k > 0) {
        static_for<L::E / 2>([&](auto H) {
          constexpr int r = 2 * decltype(H)::value;
          if constexpr (!((r >> k) & 1)) bf2(v[r], v[r | 1], v[r | (1 << k)], v[(r | (1 << k)) | 1]);
        });
      } else {
        // register bit 0: the butterfly inside each (r, r|1) pair, one FFMA2
        // (bf_self).  Pairing (r, r|2) for it instead fights the (r, r|1)
        // pairs of every other bit (measured: the repacking MOVs cost more
        // than the saved FADDs, cfg5 0.53 -> 0.49).
        static_for<L::E>([&](auto R) {
          constexpr int r = decltype(R)::value;
          if constexpr (!((r >> k) & 1)) {
#if CHW_BF_SELF
            bf_self(v[r], v[r | 1]);
#else
            bf<PER_STAGE>(v[r], v[r | (1 << k)]);
#endif
          }
        });
      }
    });
  } else {
    static_for<Bits::N>([&](auto I) {
      constexpr int k = L::slot(Bits::at(decltype(I)::value));
      static_assert(k >= 0, "butterfly bit must be a register bit");
      static_for<L::E>([&](auto R) {
        constexpr int r = decltype(R)::value;
        if constexpr (!((r >> k) & 1)) bf<PER_STAGE>(v[r], v[r | (1 << k)]);
      });
    });
  }
}

// Butterfly on a lane bit (tile bit held by thread bit `tb` < 5) via shuffles.
template <class L, int TILE_BIT, bool PER_STAGE, class C>
__device__ __forceinline__ void shfl_butterfly(C (&v)[L::E], uint32_t tid) {
  constexpr int tb = find<typename L::Th>(TILE_BIT);
  static_assert(tb >= 0 && tb < 5, "shuffle butterfly needs a lane bit");
  const bool upper = (tid >> tb) & 1u;
#pragma unroll
  for (int r = 0; r < L::E; ++r) {
    const C o = __shfl_xor_sync(0xffffffffu, v[r], 1 << tb);
    C a = upper ? o : v[r];
    C b = upper ? v[r] : o;
    bf<PER_STAGE>(a, b);
    v[r] = upper ? b : a;
  }
}

// ---------------------------------------------------------------------------
// Global <-> register and shared <-> register moves.
// ---------------------------------------------------------------------------
// Load a tile from global memory in layout L; element offset of tile bit k is
// Map::pos(k) within the tile (tile base pointer already applied).
template <class L, class Map, Cache CO = Cache::kNC, class T, class C>
__device__ __forceinline__ void load_global(const T* __restrict__ base, C (&v)[L::E], uint32_t tid) {
  constexpr int VB = vec_bits<L, Map>(IoTraits<T>::VMAX);
  const uint32_t tb = thr_off<L, Map>(tid);
  static_for<L::E>([&](auto R) {
    constexpr int r = decltype(R)::value;
    if constexpr (vec_head<L, Map>(r, VB)) {
      constexpr uint32_t ro = reg_off<L, Map>(r);
      C tmp[1 << VB];
      VecIO<T, VB, CO>::ld(base + (tb + ro), tmp);
      static_for<(1 << VB)>([&](auto Q) {
        constexpr int q = decltype(Q)::value;
        v[vec_elem<L, Map>(r, q, VB)] = tmp[q];
      });
    }
  });
}

// Predicated variant for a partial last tile: element valid iff its offset < limit.
template <class L, class Map, class T, class C>
__device__ __forceinline__ void load_global_pred(const T* __restrict__ base, C (&v)[L::E],
                                                 uint32_t tid, uint32_t limit) {
  constexpr int VB = vec_bits<L, Map>(IoTraits<T>::VMAX);
  const uint32_t tb = thr_off<L, Map>(tid);
#pragma unroll
  for (int r = 0; r < L::E; ++r) {
    if (!vec_head<L, Map>(r, VB)) continue;
    C tmp[1 << VB];
    const uint32_t off = tb + reg_off<L, Map>(r);
    if (off < limit) {
      VecIO<T, VB>::ld(base + off, tmp);
    } else {
#pragma unroll
      for (int q = 0; q < (1 << VB); ++q) tmp[q] = C(0);
    }
#pragma unroll
    for (int q = 0; q < (1 << VB); ++q) v[vec_elem<L, Map>(r, q, VB)] = tmp[q];
  }
}

// Store a tile to global memory, multiplying by `scale` when SCALE.  `outer`
// is the position of the tile's fixed (non-tile) bits inside the row: added
// to the address for bit-permutation maps, folded through lin() for linear
// maps (SeqMap).
template <class L, class Map, bool SCALE, Cache CO = Cache::kNC, class T, class C>
__device__ __forceinline__ void store_global(T* __restrict__ base, const C (&v)[L::E], uint32_t tid,
                                             C scale, uint32_t outer = 0) {
  if constexpr (IsLinearMap<Map>::value) {
    // When the position bits 0..VB-1 are register bits, the 2^VB values of a
    // vector group land in one aligned 2^VB-element block (lin maps the low
    // VB position bits into themselves), in an order fixed by the block's
    // low address bits b: slot q holds the value whose lin() is q ^ b.  The
    // thread permutes its registers with selects and issues one vector store.
    constexpr int VB = vec_bits<L, Map>(IoTraits<T>::VMAX);
    constexpr int NV = 1 << VB;
    const uint32_t tb = Map::lin(thr_off<L, Map>(tid) ^ outer);
    static_for<L::E>([&](auto R) {
      constexpr int r = decltype(R)::value;
      if constexpr (vec_head<L, Map>(r, VB)) {
        constexpr uint32_t ro = Map::lin(reg_off<L, Map>(r));
        const uint32_t addr = tb ^ ro;
        C e[NV];  // e[c]: the group's value whose low address bits (lin) are c
        static_for<NV>([&](auto A) {
          constexpr int a = decltype(A)::value;
          constexpr int cidx = (int)(Map::lin((uint32_t)a) & (NV - 1));
          e[cidx] = v[vec_elem<L, Map>(r, a, VB)];
        });
        C tmp[NV];
        const uint32_t b = addr & (NV - 1);
        static_for<NV>([&](auto Q) {
          constexpr int q = decltype(Q)::value;
          // tmp[q] = e[q ^ b] with b a runtime value: a select tree on b's bits
          C s[NV];
          static_for<NV>([&](auto K) { s[decltype(K)::value] = e[decltype(K)::value ^ q]; });
          static_for<VB>([&](auto Bt) {
            constexpr int bit = decltype(Bt)::value;
            const bool on = (b >> bit) & 1u;
            static_for<(NV >> (bit + 1))>([&](auto J) {
              constexpr int j = decltype(J)::value;
              s[j] = on ? s[j * 2 + 1] : s[j * 2];
            });
          });
          tmp[q] = SCALE ? s[0] * scale : s[0];
        });
        VecIO<T, VB, CO>::st(base + (addr & ~(uint32_t)(NV - 1)), tmp);
      }
    });
  } else {
    constexpr int VB = vec_bits<L, Map>(IoTraits<T>::VMAX);
    const uint32_t tb = thr_off<L, Map>(tid) + outer;
    static_for<L::E>([&](auto R) {
      constexpr int r = decltype(R)::value;
      if constexpr (vec_head<L, Map>(r, VB)) {
        constexpr uint32_t ro = reg_off<L, Map>(r);
        C tmp[1 << VB];
        static_for<(1 << VB)>([&](auto Q) {
          constexpr int q = decltype(Q)::value;
          tmp[q] = v[vec_elem<L, Map>(r, q, VB)];
        });
        if constexpr (SCALE) {
          if constexpr (std::is_same<C, float>::value && VB >= 1) {
            static_for<(1 << VB) / 2>([&](auto Q) { mul2(tmp[2 * decltype(Q)::value], tmp[2 * decltype(Q)::value + 1], scale); });
          } else {
            static_for<(1 << VB)>([&](auto Q) { tmp[decltype(Q)::value] *= scale; });
          }
        }
        VecIO<T, VB, CO>::st(base + (tb + ro), tmp);
      }
    });
  }
}

template <class L, class Map, bool SCALE, class T, class C>
__device__ __forceinline__ void store_global_pred(T* __restrict__ base, const C (&v)[L::E],
                                                  uint32_t tid, C scale, uint32_t limit) {
  // `limit` bounds the tile-local (pre-map) offset: the valid elements of a
  // partial last tile are its first `limit` rows' worth of tile bits.
  if constexpr (IsLinearMap<Map>::value) {
    const uint32_t tp = thr_off<L, Map>(tid);
    const uint32_t tb = Map::lin(tp);
    static_for<L::E>([&](auto R) {
      constexpr int r = decltype(R)::value;
      constexpr uint32_t rp = reg_off<L, Map>(r);
      constexpr uint32_t ro = Map::lin(rp);
      if ((tp + rp) < limit) {
        C tmp[1] = {v[r]};
        if constexpr (SCALE) tmp[0] *= scale;
        VecIO<T, 0>::st(base + (tb ^ ro), tmp);
      }
    });
  } else {
    constexpr int VB = vec_bits<L, Map>(IoTraits<T>::VMAX);
    const uint32_t tb = thr_off<L, Map>(tid);
#pragma unroll
    for (int r = 0; r < L::E; ++r) {
      if (!vec_head<L, Map>(r, VB)) continue;
      C tmp[1 << VB];
#pragma unroll
      for (int q = 0; q < (1 << VB); ++q) {
        const C x = v[vec_elem<L, Map>(r, q, VB)];
        tmp[q] = SCALE ? x * scale : x;
      }
      const uint32_t off = tb + reg_off<L, Map>(r);
      if (off < limit) VecIO<T, VB>::st(base + off, tmp);
    }
  }
}

// Shared memory: tile-local index j lives at word S::apply(j).
template <class L, class S, int VBCAP>
CHW_HD constexpr int smem_vec_bits() {
  int vb = vec_bits<L, IdMap>(VBCAP);
  while (vb > 0) {
    bool ok = true;
    for (int b = 0; b < vb; ++b)
      if (S::image(1u << b) != (1u << b)) ok = false;
    for (int b = vb; b < 31; ++b)
      if (S::image(1u << b) & ((1u << vb) - 1)) ok = false;
    if (ok) break;
    --vb;
  }
  return vb;
}

template <class C>
struct SmemCap {
  static constexpr int V = sizeof(C) == 8 ? 1 : 2;
};

template <class L, class S, class C>
__device__ __forceinline__ void smem_store(C* sm, const C (&v)[L::E], uint32_t tid) {
  constexpr int VB = smem_vec_bits<L, S, SmemCap<C>::V>();
  constexpr uint32_t tmask = S::image(thr_mask<L, IdMap>());
  const uint32_t sb = S::apply(thr_off<L, IdMap>(tid));
  static_for<L::E>([&](auto R) {
    constexpr int r = decltype(R)::value;
    if constexpr (vec_head<L, IdMap>(r, VB)) {
      constexpr uint32_t so = S::apply(reg_off<L, IdMap>(r));
      const uint32_t a = (so & tmask) ? (sb ^ so) : (sb + so);
      C tmp[1 << VB];
      static_for<(1 << VB)>([&](auto Q) {
        constexpr int q = decltype(Q)::value;
        tmp[q] = v[vec_elem<L, IdMap>(r, q, VB)];
      });
      SmemVec<C, VB>::st(sm + a, tmp);
    }
  });
}

template <class L, class S, class C>
__device__ __forceinline__ void smem_load(const C* sm, C (&v)[L::E], uint32_t tid) {
  constexpr int VB = smem_vec_bits<L, S, SmemCap<C>::V>();
  constexpr uint32_t tmask = S::image(thr_mask<L, IdMap>());
  const uint32_t sb = S::apply(thr_off<L, IdMap>(tid));
  static_for<L::E>([&](auto R) {
    constexpr int r = decltype(R)::value;
    if constexpr (vec_head<L, IdMap>(r, VB)) {
      constexpr uint32_t so = S::apply(reg_off<L, IdMap>(r));
      const uint32_t a = (so & tmask) ? (sb ^ so) : (sb + so);
      C tmp[1 << VB];
      SmemVec<C, VB>::ld(sm + a, tmp);
      static_for<(1 << VB)>([&](auto Q) {
        constexpr int q = decltype(Q)::value;
        v[vec_elem<L, IdMap>(r, q, VB)] = tmp[q];
      });
    }
  });
}

}  // namespace chwb
