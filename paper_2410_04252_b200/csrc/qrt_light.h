// libqrt — register-resident gate passes for runs of 1-/2-qubit and diagonal
// gates (the hardware-efficient-ansatz shape: RY/RZ on every qubit, CZ
// brickwork).  Shared by the host planner (qrt_gates.cu) and the kernel
// (qrt_light.cu).
//
// A light pass works on the same 2^12-amplitude tiles as gate_pass_kernel
// (positions B, the lowest four always included), but the amplitudes live in
// registers: 256 threads x 16 amplitudes.  A *stage* picks four tile bits S
// as the register bits; every gate of the stage has its dense targets in S
// (diagonal gates may target any position), so it is applied without
// touching shared memory.  Between stages the tile is transposed through
// shared memory once; the first stage loads straight from HBM and the last
// stores straight to HBM when S avoids the four coalescing positions.  A
// pass of m stages therefore costs one HBM round trip (32 B/amplitude) plus
// m-1 shared-memory round trips, whatever the number of gates.
//
// +-1 diagonal gates (CZ, CCZ, Z, ...) cost no fp64 work: their signs are
// kept pending — one bit per thread when they do not depend on a register
// bit (such signs commute with every gate applied in registers), a 16-bit
// slot mask otherwise — and applied with integer XORs on the sign bits only
// when a dense gate on an affected register bit follows (the host decides
// statically) or the tile leaves the registers.
#pragma once

#include <cstdint>

#include "qrt_internal.h"

namespace qrt {

inline constexpr int kLightRegBits = 4;                                 // 16 amplitudes per thread
inline constexpr int kLightThreads = 1 << (kTileBits - kLightRegBits);  // 256
inline constexpr int kLightMaxStages = 8;
inline constexpr int kLightMaxOps = 224;
inline constexpr int kLightMaxMats = 896;  // double2 entries in the launch parameters
inline constexpr int kLightMaxDiagK = 6;

// kL1 / kL2: dense 1-/2-qubit gate on register bits.
// kLDiag:    phase diagonal, k <= 2.
// kLSignU:   +-1 diagonal without register targets: flips the thread's sign bit.
// kLSignS:   +-1 diagonal with register targets and <= 2 other targets: slot mask table.
// kLSignG:   any other +-1 diagonal (k <= 6): slot mask evaluated per slot.
enum LightKind : std::int8_t { kL1 = 0, kL2 = 1, kLDiag = 2, kLSignU = 3, kLSignS = 4, kLSignG = 5 };

// LightOp::code: 0-3 dense 1-qubit on register bit q; 4-9 dense 2-qubit on
// register-bit pair (0,1) (0,2) (0,3) (1,2) (1,3) (2,3); then the diagonal
// kinds; 14-17 dense 1-qubit with a real first column (phase-folded) on
// register bit q; kCodeFlush set = apply pending slot signs first.
inline constexpr int kCodeSignU = 10, kCodeSignS = 11, kCodeSignG = 12, kCodeDiag = 13, kCodeReal1 = 14,
                     kCodeFlush = 64;

struct LightOp {
    std::uint64_t tab;  // kLSignU: bit f = sign of fixed-bit value f; kLSignS: 16-bit slot masks per f;
                        // kLSignG: the -1 entries of the diagonal
    std::int16_t mat;   // kL1/kL2/kLDiag: first double2 in LightParams::mats
    std::int8_t kind, k;
    std::int8_t q0, q1;  // dense: register bits of matrix bits 0 / 1 (q0 < q1 for kL2)
    std::int8_t flush;   // apply pending slot signs before this op
    std::int8_t code;    // dispatch case (see kCode*), computed on the host
    std::int8_t realcol; // kL1: first column real
    std::int8_t nsrc;    // fixed (non-register) targets
    std::int8_t src[kLightMaxDiagK];  // bit of the thread word W holding fixed target i
    std::int8_t rq[kLightMaxDiagK];   // kLDiag/kLSignG: register bit of target j, 4 if fixed
    std::int8_t fj[kLightMaxDiagK];   // kLDiag/kLSignG: target index j of fixed target i
};

struct LightStage {
    std::int8_t S[kLightRegBits];               // tile bit of register bit q
    std::int8_t tb[kTileBits - kLightRegBits];  // tile bit of thread-index bit i
    std::int16_t op_begin, op_count;
};

// Thread word W = tile index (bits 0..11) | the CTA's outer index (bit 12 + i
// <-> outer_pos[i]): every fixed diagonal target is one bit of W.
struct LightParams {
    amp_t* ptrs[kMaxLocalPEs];
    int c;  // tile bits 0..c-1 are positions 0..c-1
    int n_outer;
    int n_stages;
    int direct_in;   // stage 0 loads registers straight from HBM
    int direct_out;  // last stage stores registers straight to HBM
    int tiles_per_pe;
    std::int8_t tile_pos[kTileBits];
    std::int8_t outer_pos[64];
    LightStage st[kLightMaxStages];
    LightOp ops[kLightMaxOps];
    double2 mats[kLightMaxMats];
};

struct FusedSource;
void launch_light_pass(const LightParams& P, int total_tiles, cudaStream_t stream, int device,
                       const FusedSource* fs = nullptr);

}  // namespace qrt
