// Counter-based generators for the WoS walker.
//
// Philox4x64-10 reproduces the reference's rng.philox4x64 (rng.py:57-82) and
// _kernels.philox_block (_kernels.py:60-82) bit for bit: same multipliers, same
// round (x0,x1,x2,x3) <- (hi(M1 x2)^x1^k0, lo(M1 x2), hi(M0 x0)^x3^k1, lo(M0 x0)),
// key bumped after each round. Used by the REPLAY modes.
//
// Philox4x32 (Random123 constants) drives the NATIVE_F32 mode: 32-bit multiplies
// map to one IMAD.WIDE.U32 each, a 3-input XOR to one LOP3. 10 rounds by default,
// 7 on request (kPhiloxRoundsFast below).
#pragma once
#include <stdint.h>

namespace wos {

__device__ __forceinline__ void philox4x64(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                                           uint64_t k0, uint64_t k1, uint64_t out[4]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
    uint64_t hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
    uint64_t hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
    uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// rng.to_uniform (rng.py:100-102): top 53 bits -> [0, 1)
__device__ __forceinline__ double u01_53(uint64_t w) {
  return (double)(w >> 11) * 1.1102230246251565e-16;
}

// One Philox4x32 round with round key (k0, k1).
__device__ __forceinline__ void philox4x32_round(uint4& c, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint64_t p0 = (uint64_t)M0 * c.x;  // IMAD.WIDE.U32
  const uint64_t p1 = (uint64_t)M1 * c.z;
  c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ k0, (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ k1, (uint32_t)p0);
}

// Round counts of the NATIVE stream: 10 (Random123's default, the production stream)
// or 7 (opt-in: the fewest rounds Random123 reports Crush-resistant for Philox4x32,
// WalkConfig.philox_rounds = 7). Rounds 7..9 sit behind one kernel-uniform branch.
constexpr int kPhiloxRoundsDefault = 10;
constexpr int kPhiloxRoundsFast = 7;

__device__ __forceinline__ uint4 philox4x32(uint4 c, uint32_t k0, uint32_t k1, int rounds = 10) {
  for (int r = 0; r < rounds; ++r) {
    philox4x32_round(c, k0, k1);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// Same with a precomputed round-key schedule (rk0[r] = k0 + r W0, rk1[r] = k1 + r W1).
// With the schedule in the kernel parameters the XORs take c[] operands directly.
__device__ __forceinline__ uint4 philox4x32_rk(uint4 c, const uint32_t* rk0, const uint32_t* rk1, int rounds) {
#pragma unroll
  for (int r = 0; r < kPhiloxRoundsFast; ++r) philox4x32_round(c, rk0[r], rk1[r]);
  if (rounds > kPhiloxRoundsFast) {
#pragma unroll
    for (int r = kPhiloxRoundsFast; r < kPhiloxRoundsDefault; ++r) philox4x32_round(c, rk0[r], rk1[r]);
  }
  return c;
}

// A walk draws blocks at counters (c0, b, c2, c3): c0 = low point id, b = the block
// index (2 floor(step / jumps per block)), c2 = low traj id, c3 = the high words mixed;
// only b varies along a walk. Philox multiplies words 0 and 2 of its state, so with the
// varying word in position 1:
//   round 0 multiplies c0 and c2 — both products are per-walk constants;
//   round 1 multiplies x0' = hi(M1 c2) ^ b ^ k0 (varies) and x2' (constant);
//   round 2 multiplies x0'' (constant again) and x2'' (varies).
// Precomputing the constant products once per walk (four IMAD.WIDE at the walk start)
// leaves two of the first six multiplies per block; the output is bit-identical to
// philox4x32 on the counter (c0, b, c2, c3).
struct PhiloxPre {
  uint32_t a0;   // hi(M1 c2) ^ k0(0)               x0' = a0 ^ b
  uint32_t e1;   // lo(M0 c0) ^ k1(1)               x2'' = hi(M0 x0') ^ e1
  uint32_t b1k;  // lo(M1 x2') ^ k0(2)              state word 0 after round 2 = hi(M1 x2'') ^ b1k
  uint32_t ch2;  // hi(M0 x0'') ^ k1(2)             state word 2 after round 2 = ch2 ^ lo(M0 x0')
  uint32_t cl;   // lo(M0 x0'')                     state word 3 after round 2
};

__device__ __forceinline__ PhiloxPre philox_pre(uint32_t c0, uint32_t c2, uint32_t c3, uint32_t k00, uint32_t k10,
                                                uint32_t k01, uint32_t k11, uint32_t k02, uint32_t k12) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint64_t p1 = (uint64_t)M1 * c2;  // round 0
  const uint64_t p0 = (uint64_t)M0 * c0;
  const uint32_t x1 = (uint32_t)p1;
  const uint32_t x2 = (uint32_t)(p0 >> 32) ^ c3 ^ k10;
  const uint64_t s = (uint64_t)M1 * x2;  // round 1, word 2 (constant)
  const uint32_t b0 = (uint32_t)(s >> 32) ^ x1 ^ k01;
  const uint64_t t = (uint64_t)M0 * b0;  // round 2, word 0 (constant)
  return PhiloxPre{(uint32_t)(p1 >> 32) ^ k00, (uint32_t)p0 ^ k11, (uint32_t)s ^ k02,
                   (uint32_t)(t >> 32) ^ k12, (uint32_t)t};
}

// The same fold split once more for walks that share (c0, c3) — a unit's walks differ
// only in c2: the c2-free part (p0 = M0 c0 and s = M1 x2) once per unit, the rest
// (two multiplies instead of four) per walk. Bit-identical to philox_pre.
struct PhiloxUnit {
  uint32_t e1;   // lo(M0 c0) ^ k1(1)
  uint32_t b1k;  // lo(M1 x2) ^ k0(2)
  uint32_t sk;   // hi(M1 x2) ^ k0(1)
};

__device__ __forceinline__ PhiloxUnit philox_pre_unit(uint32_t c0, uint32_t c3, uint32_t k10, uint32_t k01,
                                                      uint32_t k11, uint32_t k02) {
  const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
  const uint32_t x2 = (uint32_t)(p0 >> 32) ^ c3 ^ k10;
  const uint64_t s = (uint64_t)0xCD9E8D57u * x2;
  return PhiloxUnit{(uint32_t)p0 ^ k11, (uint32_t)s ^ k02, (uint32_t)(s >> 32) ^ k01};
}

__device__ __forceinline__ PhiloxPre philox_pre_walk(uint32_t c2, const PhiloxUnit& u, uint32_t k00,
                                                     uint32_t k12) {
  const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
  const uint32_t b0 = u.sk ^ (uint32_t)p1;
  const uint64_t t = (uint64_t)0xD2511F53u * b0;
  return PhiloxPre{(uint32_t)(p1 >> 32) ^ k00, u.e1, u.b1k, (uint32_t)(t >> 32) ^ k12, (uint32_t)t};
}

// rounds 0-2 from the precomputed words: the state entering round 3
__device__ __forceinline__ uint4 philox_pre_r012(uint32_t b, const PhiloxPre& p) {
  const uint64_t q = (uint64_t)0xD2511F53u * (p.a0 ^ b);                // round 1, word 0
  const uint64_t r = (uint64_t)0xCD9E8D57u * ((uint32_t)(q >> 32) ^ p.e1);  // round 2, word 2
  return make_uint4((uint32_t)(r >> 32) ^ p.b1k, (uint32_t)r, p.ch2 ^ (uint32_t)q, p.cl);
}

__device__ __forceinline__ uint4 philox4x32_rk_pre(uint32_t b, const PhiloxPre& p, const uint32_t* rk0,
                                                   const uint32_t* rk1, int rounds) {
  uint4 c = philox_pre_r012(b, p);
#pragma unroll
  for (int r = 3; r < kPhiloxRoundsFast; ++r) philox4x32_round(c, rk0[r], rk1[r]);
  if (rounds > kPhiloxRoundsFast) {
#pragma unroll
    for (int r = kPhiloxRoundsFast; r < kPhiloxRoundsDefault; ++r) philox4x32_round(c, rk0[r], rk1[r]);
  }
  return c;
}

// multi-instance walks: the launch-uniform k0 schedule from the kernel parameters (ptxas
// keeps it in uniform registers), the per-instance k1 bumped per round
__device__ __forceinline__ uint4 philox4x32_pre_k0(uint32_t b, const PhiloxPre& p, const uint32_t* rk0, uint32_t k1,
                                                   int rounds) {
  uint4 c = philox_pre_r012(b, p);
#pragma unroll
  for (int r = 3; r < kPhiloxRoundsFast; ++r) philox4x32_round(c, rk0[r], k1 + (uint32_t)r * 0xBB67AE85u);
  if (rounds > kPhiloxRoundsFast) {
#pragma unroll
    for (int r = kPhiloxRoundsFast; r < kPhiloxRoundsDefault; ++r)
      philox4x32_round(c, rk0[r], k1 + (uint32_t)r * 0xBB67AE85u);
  }
  return c;
}

__device__ __forceinline__ uint4 philox4x32_pre(uint32_t b, const PhiloxPre& p, uint32_t k0, uint32_t k1,
                                                int rounds) {
  uint4 c = philox_pre_r012(b, p);
  k0 += 3u * 0x9E3779B9u;
  k1 += 3u * 0xBB67AE85u;
#pragma unroll
  for (int r = 3; r < kPhiloxRoundsFast; ++r) {
    philox4x32_round(c, k0, k1);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  if (rounds > kPhiloxRoundsFast) {
#pragma unroll
    for (int r = kPhiloxRoundsFast; r < kPhiloxRoundsDefault; ++r) {
      philox4x32_round(c, k0, k1);
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
  }
  return c;
}

// NATIVE uniform: (w >> 9) * 2^-23 in [0, 1), exact in fp32 (one LOP3 + one FADD).
__device__ __forceinline__ float u01_23(uint32_t w) {
  return __uint_as_float(0x3f800000u | (w >> 9)) - 1.0f;
}

}  // namespace wos
