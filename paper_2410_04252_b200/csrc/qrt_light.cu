// libqrt — register-resident light gate passes (see qrt_light.h).
//
// Reference semantics: apply_gate_narrow (dist_sim.cpp:163-201) for every
// gate of the pass, in an order that never swaps two gates sharing a qubit.
// One CTA = one 2^12-amplitude tile = 256 threads x 16 amplitudes.

#include "qrt_fused.h"
#include "qrt_light.h"

// 1: prefetch the next op's dispatch code (measured slower: 30q HEA gates
// 454 -> 490 ms, same-box A/B profiles/r2/lpf — the op loop already runs on
// the uniform datapath, and the extra live value costs registers)
#ifndef QRT_LIGHT_PREFETCH
#define QRT_LIGHT_PREFETCH 0
#endif

namespace qrt {

namespace {

using u64 = std::uint64_t;

__device__ __forceinline__ int swz(int e) {
    const int x = e >> 3;
    return e ^ ((x ^ (x >> 3) ^ (x >> 6) ^ (x >> 9)) & 7);
}

__device__ __forceinline__ double2 cmul(const double2 u, const double2 a) {
    return make_double2(fma(u.x, a.x, -u.y * a.y), fma(u.x, a.y, u.y * a.x));
}
__device__ __forceinline__ double2 cmac2(const double2 u, const double2 a, const double2 w, const double2 b) {
    double2 r;
    r.x = fma(u.x, a.x, fma(-u.y, a.y, fma(w.x, b.x, -w.y * b.y)));
    r.y = fma(u.x, a.y, fma(u.y, a.x, fma(w.x, b.y, w.y * b.x)));
    return r;
}

// In place (see dense1r): y-only partials, then y', then x'.
template <int Q>
__device__ __forceinline__ void dense1(double2 (&a)[16], const double2* __restrict__ m) {
    const double2 m00 = m[0], m01 = m[1], m10 = m[2], m11 = m[3];
    const double n00 = -m00.y, n01 = -m01.y, n10 = -m10.y, n11 = -m11.y;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        if ((r >> Q) & 1) continue;
        const int s = r | (1 << Q);
        asm("{\n"
            ".reg .f64 p0, p1, p2, p3;\n"
            "mul.rn.f64 p0, %5, %3;\n"       // x'.x <- m01.x y.x - m01.y y.y
            "fma.rn.f64 p0, %4, %2, p0;\n"
            "mul.rn.f64 p1, %6, %2;\n"       // x'.y <- m01.x y.y + m01.y y.x
            "fma.rn.f64 p1, %4, %3, p1;\n"
            "mul.rn.f64 p2, %8, %3;\n"       // y'.x <- m11.x y.x - m11.y y.y
            "fma.rn.f64 p2, %7, %2, p2;\n"
            "mul.rn.f64 p3, %9, %2;\n"       // y'.y <- m11.x y.y + m11.y y.x
            "fma.rn.f64 p3, %7, %3, p3;\n"
            "fma.rn.f64 p2, %13, %1, p2;\n"  // - m10.y x.y
            "fma.rn.f64 p3, %12, %0, p3;\n"  // + m10.y x.x
            "fma.rn.f64 %2, %11, %0, p2;\n"  // y'.x = m10.x x.x + ...
            "fma.rn.f64 %3, %11, %1, p3;\n"  // y'.y = m10.x x.y + ...
            "fma.rn.f64 p0, %15, %1, p0;\n"  // - m00.y x.y
            "fma.rn.f64 p1, %14, %0, p1;\n"  // + m00.y x.x
            "fma.rn.f64 %0, %10, %0, p0;\n"  // x'.x = m00.x x.x + ...
            "fma.rn.f64 %1, %10, %1, p1;\n"  // x'.y = m00.x x.y + ...
            "}\n"
            : "+d"(a[r].x), "+d"(a[r].y), "+d"(a[s].x), "+d"(a[s].y)
            : "d"(m01.x), "d"(n01), "d"(m01.y), "d"(m11.x), "d"(n11), "d"(m11.y), "d"(m00.x), "d"(m10.x),
              "d"(m10.y), "d"(n10), "d"(m00.y), "d"(n00));
    }
}

// Dense 1-qubit gate whose first column is real (m00, m10 real): 6 fp64
// operations per amplitude instead of 8.
// In-place form: the y-only partial sums first, then y' and x' overwrite
// their own registers, so every slot keeps its register across the op switch
// (the C++ form left ~2 register copies per amplitude at the switch join).
template <int Q>
__device__ __forceinline__ void dense1r(double2 (&a)[16], const double2* __restrict__ m) {
    const double m00 = m[0].x, m10 = m[2].x;
    const double2 m01 = m[1], m11 = m[3];
    const double n01 = -m01.y, n11 = -m11.y;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        if ((r >> Q) & 1) continue;
        const int s = r | (1 << Q);
        asm("{\n"
            ".reg .f64 p0, p1, p2, p3;\n"
            "mul.rn.f64 p0, %5, %3;\n"
            "fma.rn.f64 p0, %4, %2, p0;\n"
            "mul.rn.f64 p1, %6, %2;\n"
            "fma.rn.f64 p1, %4, %3, p1;\n"
            "mul.rn.f64 p2, %11, %3;\n"
            "fma.rn.f64 p2, %10, %2, p2;\n"
            "mul.rn.f64 p3, %7, %2;\n"
            "fma.rn.f64 p3, %10, %3, p3;\n"
            "fma.rn.f64 %2, %9, %0, p2;\n"
            "fma.rn.f64 %3, %9, %1, p3;\n"
            "fma.rn.f64 %0, %8, %0, p0;\n"
            "fma.rn.f64 %1, %8, %1, p1;\n"
            "}\n"
            : "+d"(a[r].x), "+d"(a[r].y), "+d"(a[s].x), "+d"(a[s].y)
            : "d"(m01.x), "d"(n01), "d"(m01.y), "d"(m11.y), "d"(m00), "d"(m10), "d"(m11.x), "d"(n11));
    }
}

// Matrix bit 0 <-> register bit Q0, matrix bit 1 <-> register bit Q1 (Q0 < Q1).
template <int Q0, int Q1>
__device__ __forceinline__ void dense2(double2 (&a)[16], const double2* __restrict__ m) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        if (((r >> Q0) & 1) || ((r >> Q1) & 1)) continue;
        const int i0 = r, i1 = r | (1 << Q0), i2 = r | (1 << Q1), i3 = r | (1 << Q0) | (1 << Q1);
        const double2 x0 = a[i0], x1 = a[i1], x2 = a[i2], x3 = a[i3];
        double2 y[4];
#pragma unroll
        for (int row = 0; row < 4; ++row) {
            const double2* u = m + 4 * row;
            double2 acc = cmac2(u[0], x0, u[1], x1);
            const double2 t = cmac2(u[2], x2, u[3], x3);
            acc.x += t.x;
            acc.y += t.y;
            y[row] = acc;
        }
        a[i0] = y[0];
        a[i1] = y[1];
        a[i2] = y[2];
        a[i3] = y[3];
    }
}

// Pending +-1 signs: bit r set = register slot r still owes a negation.
// Applied by XOR on the sign bits (integer pipe), not as fp64 negations.
__device__ __forceinline__ void apply_signs(double2 (&a)[16], unsigned& pend) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const int s = static_cast<int>((pend >> r) & 1u) << 31;
        a[r].x = __hiloint2double(__double2hiint(a[r].x) ^ s, __double2loint(a[r].x));
        a[r].y = __hiloint2double(__double2hiint(a[r].y) ^ s, __double2loint(a[r].y));
    }
    pend = 0;
}

// Pending +-1 signs folded into the slot mask: the thread-uniform bit g
// flips every slot.
__device__ __forceinline__ void flush_all(double2 (&a)[16], unsigned& pend, unsigned& g) {
    pend ^= 0u - g;
    g = 0;
    apply_signs(a, pend);
}

// Value of the fixed (non-register) targets of a diagonal op: bit i = bit
// src[i] of the thread word W.
__device__ __forceinline__ int fixed_value(const LightOp& op, std::uint64_t W) {
    const int ns = op.nsrc;
    int f = 0;
    if (ns > 0) f |= static_cast<int>((W >> op.src[0]) & 1ull);
    if (ns > 1) f |= static_cast<int>((W >> op.src[1]) & 1ull) << 1;
    for (int i = 2; i < ns; ++i) f |= static_cast<int>((W >> op.src[i]) & 1ull) << i;
    return f;
}

// Diagonal index of slot r: fixed targets from f, register targets from r.
__device__ __forceinline__ int diag_index(const LightOp& op, int f, int r) {
    int m = 0;
    const int k = op.k, ns = op.nsrc;
    for (int i = 0; i < ns; ++i) m |= ((f >> i) & 1) << op.fj[i];
    for (int j = 0; j < k; ++j)
        if (op.rq[j] < 4) m |= ((r >> op.rq[j]) & 1) << j;
    return m;
}

// FUSED: the pass gathers its tile through a pending QR (qrt_fused.h); a
// separate instantiation so the common path carries no extra registers.
template <bool FUSED>
__global__ void __launch_bounds__(kLightThreads, 2)
    light_pass_kernel(const __grid_constant__ LightParams P, const FusedSource* __restrict__ fs_arg) {
    const FusedSource* __restrict__ fs = FUSED ? fs_arg : nullptr;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int E = 1 << kTileBits;
    double2* tile = reinterpret_cast<double2*>(smem_raw);
    u64* tab = reinterpret_cast<u64*>(tile + E);
    const int c = P.c;
    const int t = threadIdx.x;
    u64 cta = 0;
    const u64 b = static_cast<u64>(blockIdx.x % P.tiles_per_pe);  // bit i <-> outer_pos[i]
    for (int i = 0; i < P.n_outer; ++i) cta |= ((b >> i) & 1ull) << P.outer_pos[i];
    const u64 wout = b << kTileBits;  // outer bits of the thread word W
    amp_t* __restrict__ v = P.ptrs[blockIdx.x / P.tiles_per_pe];
    const int nt = 1 << (kTileBits - c);
    const int cmask = (1 << c) - 1;
    if (!P.direct_in || !P.direct_out || fs) {
        for (int h = t; h < nt; h += kLightThreads) {
            u64 o = 0;
            for (int i = c; i < kTileBits; ++i) o |= static_cast<u64>((h >> (i - c)) & 1) << P.tile_pos[i];
            tab[h] = o;
        }
        __syncthreads();
    }
    u64* fwords = tab + nt;  // fused QR tables (host sizes shared memory for them)
    if (fs) fused_tables(*fs, tab, nt, cta, fs->pe_begin + static_cast<int>(blockIdx.x / P.tiles_per_pe), fwords);
    amp_t* __restrict__ vout = fs ? fs->dst[blockIdx.x / P.tiles_per_pe] : v;

    double2 a[16];
    unsigned pend = 0;  // pending slot signs
    unsigned g = 0;     // pending thread-uniform sign
    int ebase = 0;      // tile index of register slot 0
    int swq[4];         // swizzled tile offset of register bit q (swz is linear over GF(2))
    auto map_stage = [&](const LightStage& S) {
        ebase = 0;
#pragma unroll
        for (int i = 0; i < kTileBits - kLightRegBits; ++i) ebase |= ((t >> i) & 1) << S.tb[i];
#pragma unroll
        for (int q = 0; q < 4; ++q) swq[q] = swz(1 << S.S[q]);
    };
    auto sslot = [&](int sb, int r) {
        int o = sb;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if ((r >> q) & 1) o ^= swq[q];
        return o;
    };
    auto gofs = [&](int e) {  // tile index -> offset inside the PE
        u64 o = cta;
#pragma unroll
        for (int i = 0; i < kTileBits; ++i)
            if ((e >> i) & 1) o |= 1ull << P.tile_pos[i];
        return o;
    };

    // ---- stage 0 input
    map_stage(P.st[0]);
    if (P.direct_in && !FUSED) {
        const u64 g0 = gofs(ebase);
        u64 gq[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) gq[q] = 1ull << P.tile_pos[P.st[0].S[q]];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            u64 o = g0;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if ((r >> q) & 1) o |= gq[q];
            a[r] = __ldcs(&v[o]);
        }
    } else {
        for (int e = t; e < E; e += kLightThreads) {
            const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&tile[swz(e)]));
            const amp_t* src = fs ? fused_src(*fs, fwords, e, cmask, c) : &v[cta | tab[e >> c] | (e & cmask)];
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src));
        }
        asm volatile("cp.async.wait_all;\n" ::);
        __syncthreads();
        const int sb = swz(ebase);
#pragma unroll
        for (int r = 0; r < 16; ++r) a[r] = tile[sslot(sb, r)];
    }

    for (int s = 0; s < P.n_stages; ++s) {
        const LightStage& S = P.st[s];
        if (s > 0) {
            // transpose through shared memory: previous mapping out, this one in
            flush_all(a, pend, g);
            {
                const int sb = swz(ebase);
                __syncthreads();  // readers of the previous transpose are done
#pragma unroll
                for (int r = 0; r < 16; ++r) tile[sslot(sb, r)] = a[r];
            }
            __syncthreads();
            map_stage(S);
            const int sb = swz(ebase);
#pragma unroll
            for (int r = 0; r < 16; ++r) a[r] = tile[sslot(sb, r)];
        }
        const u64 W = static_cast<u64>(ebase) | wout;
        const int o_end = S.op_begin + S.op_count;
#if QRT_LIGHT_PREFETCH
        // the next op's dispatch code is loaded while this op computes (it heads
        // each op's load chain: code -> dispatch -> matrix offset -> matrix)
        int code_n = 0;
        if (S.op_count > 0) code_n = P.ops[S.op_begin].code;
#endif
        for (int o = S.op_begin; o < o_end; ++o) {
            const LightOp& op = P.ops[o];
            // one host-computed case code per op (jump table), flush bit on top
#if QRT_LIGHT_PREFETCH
            const int code = code_n;
            const int mat = op.mat;
            if (o + 1 < o_end) code_n = P.ops[o + 1].code;
#else
            const int code = op.code;
            const int mat = op.mat;
#endif
            if (code & kCodeFlush) apply_signs(a, pend);
            switch (code & ~kCodeFlush) {
                case 0: dense1<0>(a, P.mats + mat); break;
                case 1: dense1<1>(a, P.mats + mat); break;
                case 2: dense1<2>(a, P.mats + mat); break;
                case 3: dense1<3>(a, P.mats + mat); break;
                case 4: dense2<0, 1>(a, P.mats + mat); break;
                case 5: dense2<0, 2>(a, P.mats + mat); break;
                case 6: dense2<0, 3>(a, P.mats + mat); break;
                case 7: dense2<1, 2>(a, P.mats + mat); break;
                case 8: dense2<1, 3>(a, P.mats + mat); break;
                case 9: dense2<2, 3>(a, P.mats + mat); break;
                case kCodeReal1 + 0: dense1r<0>(a, P.mats + mat); break;
                case kCodeReal1 + 1: dense1r<1>(a, P.mats + mat); break;
                case kCodeReal1 + 2: dense1r<2>(a, P.mats + mat); break;
                case kCodeReal1 + 3: dense1r<3>(a, P.mats + mat); break;
                case kCodeSignU: g ^= static_cast<unsigned>(op.tab >> fixed_value(op, W)) & 1u; break;
                case kCodeSignS: pend ^= static_cast<unsigned>(op.tab >> (16 * fixed_value(op, W))) & 0xffffu; break;
                case kCodeSignG: {
                    const int f = fixed_value(op, W);
                    unsigned mask = 0;
#pragma unroll
                    for (int r = 0; r < 16; ++r)
                        mask |= static_cast<unsigned>((op.tab >> diag_index(op, f, r)) & 1ull) << r;
                    pend ^= mask;
                    break;
                }
                default: {
                    // phase diagonal (k <= 2): two entries live at a time
                    const int f = fixed_value(op, W);
                    const double2* d = P.mats + mat;
                    const int halves = op.k > 1 ? 2 : 1;
#pragma unroll 1
                    for (int hb = 0; hb < halves; ++hb) {
                        const double2 d0 = d[2 * hb], d1 = d[2 * hb + 1];
#pragma unroll
                        for (int r = 0; r < 16; ++r) {
                            const int m = diag_index(op, f, r);
                            if ((m >> 1) == hb) a[r] = cmul((m & 1) ? d1 : d0, a[r]);
                        }
                    }
                    break;
                }
            }
        }
    }

    // ---- last stage output
    flush_all(a, pend, g);
    if (P.direct_out) {
        const u64 g0 = gofs(ebase);
        u64 gq[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) gq[q] = 1ull << P.tile_pos[P.st[P.n_stages - 1].S[q]];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            u64 o = g0;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if ((r >> q) & 1) o |= gq[q];
            __stcs(&vout[o], a[r]);
        }
    } else {
        const int sb = swz(ebase);
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 16; ++r) tile[sslot(sb, r)] = a[r];
        __syncthreads();
        for (int e = t; e < E; e += kLightThreads) __stcs(&vout[cta | tab[e >> c] | (e & cmask)], tile[swz(e)]);
    }
}

}  // namespace

void launch_light_pass(const LightParams& P, int total_tiles, cudaStream_t stream, int device, const FusedSource* fs) {
    static bool attr_done[64] = {};
    const std::size_t nt = std::size_t{1} << (kTileBits - P.c);
    const std::size_t smem = (std::size_t{1} << kTileBits) * sizeof(double2) +
                             (nt + (fs ? kFusedSmemWords + nt : 0)) * sizeof(std::uint64_t);
    if (!attr_done[device]) {
        QRT_CUDA(cudaFuncSetAttribute(light_pass_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
        QRT_CUDA(cudaFuncSetAttribute(light_pass_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
        attr_done[device] = true;
    }
    if (fs)
        light_pass_kernel<true><<<total_tiles, kLightThreads, smem, stream>>>(P, fs);
    else
        light_pass_kernel<false><<<total_tiles, kLightThreads, smem, stream>>>(P, nullptr);
    QRT_CUDA(cudaGetLastError());
}

}  // namespace qrt
