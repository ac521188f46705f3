// common.cuh — device helpers shared by every kernel of the λ(ω)/BB engine.
//
//  * 32-byte sector I/O: sm_100a's 256-bit LDG/STG (LDG.E.ENL2.256 / STG.E.ENL2.256)
//    move one whole DRAM sector per thread.
//  * submask_bits(): the gasket membership of a run of cells as a bit-mask. The
//    reference tests membership per cell through a byte raster
//    (MemberMask, fractal.hpp:105-125); for the gasket it is the bit test
//    x & (n-1-y) == 0 (tests/acceptance.cpp:88-102), i.e. "x is a submask of y".
//  * λ(ω) in closed form: with X(v) = bit 2j set iff base-3
//    digit j of v is 2 and Y(v) = bit 2j set iff digit j >= 1,
//        λx = X(ωx) | X(ωy) << 1,   λy = Y(ωx) | Y(ωy) << 1.
//    This is the reference's digit loop (block_map.cpp:77-111: odd μ consume
//    digits of ωx, even μ digits of ωy, τ = H[β] with H = {(0,0),(0,1),(1,1)},
//    Δ = τ·2^(μ-1)) with the per-level sum turned into bit placement.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace nbbgpu {

struct Sector {
    uint32_t w[8];
};

__device__ __forceinline__ Sector ldg_sector(const void* p) {
    Sector r;
    asm volatile(
        "ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]),
          "=r"(r.w[6]), "=r"(r.w[7])
        : "l"(p));
    return r;
}

// Coherent (non-.nc) variant, for grids written earlier in the same kernel.
__device__ __forceinline__ Sector ld_sector(const void* p) {
    Sector r;
    asm volatile(
        "ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]),
          "=r"(r.w[6]), "=r"(r.w[7])
        : "l"(p)
        : "memory");
    return r;
}

__device__ __forceinline__ void stg_sector(void* p, const Sector& v) {
    asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]),
                 "r"(v.w[1]), "r"(v.w[2]), "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]),
                 "r"(v.w[7])
                 : "memory");
}

// Bit i (0 <= i < 32) set iff i is a submask of m (m < 32): the member bits of
// a 32-cell run whose row selector restricted to the run is m.
__device__ __forceinline__ uint32_t submask_bits(uint32_t m) {
    uint32_t f = 1u;
    if (m & 1u) f |= f << 1;
    if (m & 2u) f |= f << 2;
    if (m & 4u) f |= f << 4;
    if (m & 8u) f |= f << 8;
    if (m & 16u) f |= f << 16;
    return f;
}

__host__ __device__ __forceinline__ bool gasket_member(int64_t x, int64_t y, int64_t n) {
    return x >= 0 && y >= 0 && x < n && y < n && (x & (n - 1 - y)) == 0;
}


// ---- generic NBB specs (vicsek, carpet, …) ---------------------------------------
// Table-driven descriptor for the per-cell kernels; the gasket keeps the bit-test and
// closed-form fast paths (`gasket` = 1).
struct DevSpec {
    int k, s;
    int ox[9], oy[9];
    int replica_at[9];  // step-box cell cy*s + cx -> replica index, -1 if empty
    int gasket;
};

// is_member (fractal.cpp:194-214): descend the replica chain; false outside the embedding
__device__ __forceinline__ bool member_spec(const DevSpec& sp, int64_t x, int64_t y, int level) {
    int64_t n = 1;
    for (int i = 0; i < level; ++i) n *= sp.s;
    if (sp.gasket) return gasket_member(x, y, n);
    if (x < 0 || y < 0 || x >= n || y >= n) return false;
    int64_t scale = n / sp.s;
    for (int mu = level; mu >= 1; --mu) {
        const int cx = (int)(x / scale), cy = (int)(y / scale);
        if (sp.replica_at[cy * sp.s + cx] < 0) return false;
        x -= cx * scale;
        y -= cy * scale;
        scale /= sp.s;
    }
    return true;
}

// lambda_map (block_map.cpp:77-111): odd levels consume base-k digits of ωx, even of ωy
__device__ __forceinline__ void lambda_spec(const DevSpec& sp, uint64_t ox, uint64_t oy, int level,
                                            int64_t& x, int64_t& y) {
    int64_t px = 0, py = 0, scale = 1;
    for (int mu = 1; mu <= level; ++mu) {
        int beta;
        if (mu & 1) {
            beta = (int)(ox % (uint64_t)sp.k);
            ox /= (uint64_t)sp.k;
        } else {
            beta = (int)(oy % (uint64_t)sp.k);
            oy /= (uint64_t)sp.k;
        }
        px += sp.ox[beta] * scale;
        py += sp.oy[beta] * scale;
        scale *= sp.s;
    }
    x = px;
    y = py;
}

// ---- λ(ω) ------------------------------------------------------------------
// LUT over 6 base-3 digits: entry v (< 729) = X6(v) | Y6(v) << 16, X6/Y6 < 2^11.
__constant__ uint32_t c_xy729[729];

__host__ __device__ __forceinline__ uint32_t xy6_arith(uint32_t v) {
    uint32_t X = 0, Y = 0;
    for (int j = 0; j < 6; ++j) {
        const uint32_t q = v / 3u;
        const uint32_t d = v - 3u * q;
        X |= (d == 2u ? 1u : 0u) << (2 * j);
        Y |= (d != 0u ? 1u : 0u) << (2 * j);
        v = q;
    }
    return X | (Y << 16);
}

// X(v), Y(v) for v < 3^12 from a 729-entry table (constant or shared memory).
__device__ __forceinline__ void xy_from_table(const uint32_t* tab, uint32_t v, uint32_t& X,
                                              uint32_t& Y) {
    const uint32_t hi = __umulhi(v, 0x59E60383u) >> 8;  // v / 729, exact for v <= 3^12
    const uint32_t lo = v - hi * 729u;
    const uint32_t a = tab[lo];
    const uint32_t b = hi ? tab[hi] : 0u;
    X = (a & 0xFFFFu) | ((b & 0xFFFFu) << 12);
    Y = (a >> 16) | ((b >> 16) << 12);
}

// Arithmetic X/Y for any 32-bit v (no table; used where indices diverge and no
// table is staged).
__device__ __forceinline__ void xy_arith(uint32_t v, uint32_t& X, uint32_t& Y) {
    X = 0;
    Y = 0;
    for (int j = 0; v != 0u; ++j) {
        const uint32_t q = __umulhi(v, 0xAAAAAAABu) >> 1;
        const uint32_t d = v - 3u * q;
        X |= (d == 2u ? 1u : 0u) << (2 * j);
        Y |= (d != 0u ? 1u : 0u) << (2 * j);
        v = q;
    }
}

__device__ __forceinline__ void lambda_from_xy(uint32_t Xx, uint32_t Yx, uint32_t Xy, uint32_t Yy,
                                               uint32_t& lx, uint32_t& ly) {
    lx = Xx | (Xy << 1);
    ly = Yx | (Yy << 1);
}

// λ via the constant-memory table: warp-uniform ω -> one broadcast per lookup.
__device__ __forceinline__ void lambda_const(uint32_t ox, uint32_t oy, uint32_t& lx, uint32_t& ly) {
    uint32_t Xx, Yx, Xy, Yy;
    xy_from_table(c_xy729, ox, Xx, Yx);
    xy_from_table(c_xy729, oy, Xy, Yy);
    lambda_from_xy(Xx, Yx, Xy, Yy, lx, ly);
}

__device__ __forceinline__ void lambda_arith(uint32_t ox, uint32_t oy, uint32_t& lx, uint32_t& ly) {
    uint32_t Xx, Yx, Xy, Yy;
    xy_arith(ox, Xx, Yx);
    xy_arith(oy, Xy, Yy);
    lambda_from_xy(Xx, Yx, Xy, Yy, lx, ly);
}

// Division by a runtime constant d (< 2^31) for dividends < 2^32 via a host-
// precomputed magic (Granlund–Montgomery round-up): q = umulhi(x, m) >> s.
struct FastDiv {
    uint32_t d;
    uint32_t m;
    uint32_t s;
};

__device__ __forceinline__ uint32_t fastdiv(uint32_t x, const FastDiv& f) {
    return f.m == 0u ? (x >> f.s) : (__umulhi(x, f.m) >> f.s);
}

// 4 alive bits of a sector of four int64 cells.
__device__ __forceinline__ uint32_t alive4_i64(const Sector& v) {
    return ((v.w[0] | v.w[1]) != 0u ? 1u : 0u) | ((v.w[2] | v.w[3]) != 0u ? 2u : 0u) |
           ((v.w[4] | v.w[5]) != 0u ? 4u : 0u) | ((v.w[6] | v.w[7]) != 0u ? 8u : 0u);
}

// 4 bits (byte nonzero) of one 32-bit word of uint8 cells.
__device__ __forceinline__ uint32_t alive4_u8(uint32_t w) {
    const uint32_t t = (((w & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | w) & 0x80808080u;
    return ((t >> 7) * 0x00204081u) >> 21 & 0xFu;
}

// 32 alive bits of a sector of 32 uint8 cells.
__device__ __forceinline__ uint32_t alive32_u8(const Sector& v) {
    uint32_t b = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) b |= alive4_u8(v.w[i]) << (4 * i);
    return b;
}

// Sector of four int64 cells holding (nib >> i) & 1.
__device__ __forceinline__ Sector expand4_i64(uint32_t nib) {
    Sector s;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        s.w[2 * i] = (nib >> i) & 1u;
        s.w[2 * i + 1] = 0u;
    }
    return s;
}

// Sector of 32 uint8 cells holding bit i of `bits`.
__device__ __forceinline__ Sector expand32_u8(uint32_t bits) {
    Sector s;
#pragma unroll
    for (int i = 0; i < 8; ++i) s.w[i] = (((bits >> (4 * i)) & 0xFu) * 0x00204081u) & 0x01010101u;
    return s;
}

// Masked int64 sum of a sector (bit i of nib selects cell i).
__device__ __forceinline__ uint64_t masked_sum4(const Sector& v, uint32_t nib) {
    uint64_t s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint64_t c = (uint64_t)v.w[2 * i] | ((uint64_t)v.w[2 * i + 1] << 32);
        s += (nib >> i & 1u) ? c : 0ull;
    }
    return s;
}

// Life-like update of 32 cells held bit-sliced: the 8 neighbour words, the
// centre word and the rule masks (bit v of birth/survive: count v -> alive).
// count = number of set neighbour bits per position, computed by a carry-save
// adder tree; the rule is then a 5-input truth table (centre, count bits)
// evaluated as a mux tree over constant leaves.
__device__ __forceinline__ uint32_t life_rule(uint32_t n0, uint32_t n1, uint32_t n2, uint32_t n3,
                                              uint32_t n4, uint32_t n5, uint32_t n6, uint32_t n7,
                                              uint32_t centre, uint32_t birth, uint32_t survive) {
    // full adders over (n0,n1,n2), (n3,n4,n5); half adder over (n6,n7)
    const uint32_t s0 = n0 ^ n1 ^ n2, c0 = (n0 & n1) | (n2 & (n0 ^ n1));
    const uint32_t s1 = n3 ^ n4 ^ n5, c1 = (n3 & n4) | (n5 & (n3 ^ n4));
    const uint32_t s2 = n6 ^ n7, c2 = n6 & n7;
    // ones column
    const uint32_t b0 = s0 ^ s1 ^ s2, k0 = (s0 & s1) | (s2 & (s0 ^ s1));
    // twos column: c0 + c1 + c2 + k0 (each weight 2) -> t0 (2s), t1 (4s), t2 (8s)
    const uint32_t u0 = c0 ^ c1 ^ c2, v0 = (c0 & c1) | (c2 & (c0 ^ c1));
    const uint32_t b1 = u0 ^ k0, w0 = u0 & k0;
    const uint32_t b2 = v0 ^ w0, b3 = v0 & w0;
    // leaves: for count v, alive -> survive bit v, dead -> birth bit v
    uint32_t leaf[9];
#pragma unroll
    for (int v = 0; v < 9; ++v) {
        const uint32_t sv = (survive >> v & 1u) ? 0xFFFFFFFFu : 0u;
        const uint32_t bv = (birth >> v & 1u) ? 0xFFFFFFFFu : 0u;
        leaf[v] = (centre & sv) | (~centre & bv);
    }
    // mux tree over b0 (counts 0..7 in pairs), b1, b2; count 8 = b3 (then b0..b2 = 0)
    const uint32_t m01 = (b0 & leaf[1]) | (~b0 & leaf[0]);
    const uint32_t m23 = (b0 & leaf[3]) | (~b0 & leaf[2]);
    const uint32_t m45 = (b0 & leaf[5]) | (~b0 & leaf[4]);
    const uint32_t m67 = (b0 & leaf[7]) | (~b0 & leaf[6]);
    const uint32_t m03 = (b1 & m23) | (~b1 & m01);
    const uint32_t m47 = (b1 & m67) | (~b1 & m45);
    const uint32_t m07 = (b2 & m47) | (~b2 & m03);
    return (b3 & leaf[8]) | (~b3 & m07);
}

// A Life-like rule as the constants of two count-indexed mux trees, S for live centres and B for
// dead ones (leaf v = 0 or ~0: bit v of survive / birth). Level-0 node k of a tree is
// leaf[2k] ^ (b0 & (leaf[2k] ^ leaf[2k + 1])): every constant enters one logic op as a
// constant-bank operand (the table is a kernel parameter), so a runtime rule costs no per-cell
// materialisation of its 18 leaf masks (life_rule's `bit ? ~0 : 0` per leaf and cell).
struct RuleTab {
    uint32_t sd[4], se[4], s8;  // survive tree: leaf[2k] ^ leaf[2k + 1], leaf[2k], leaf[8]
    uint32_t bd[4], be[4], b8;  // birth tree
};
__host__ __device__ inline RuleTab make_rule_tab(uint32_t birth, uint32_t survive) {
    RuleTab t{};
    auto leaf = [](uint32_t m, int v) { return ((m >> v) & 1u) ? 0xFFFFFFFFu : 0u; };
    for (int k = 0; k < 4; ++k) {
        t.se[k] = leaf(survive, 2 * k);
        t.sd[k] = leaf(survive, 2 * k) ^ leaf(survive, 2 * k + 1);
        t.be[k] = leaf(birth, 2 * k);
        t.bd[k] = leaf(birth, 2 * k) ^ leaf(birth, 2 * k + 1);
    }
    t.s8 = leaf(survive, 8);
    t.b8 = leaf(birth, 8);
    return t;
}
// life_rule with the rule as a RuleTab (same adder tree; bit-identical results)
__device__ __forceinline__ uint32_t life_rule_tab(uint32_t n0, uint32_t n1, uint32_t n2, uint32_t n3, uint32_t n4,
                                                  uint32_t n5, uint32_t n6, uint32_t n7, uint32_t centre,
                                                  const RuleTab& t) {
    const uint32_t s0 = n0 ^ n1 ^ n2, c0 = (n0 & n1) | (n2 & (n0 ^ n1));
    const uint32_t s1 = n3 ^ n4 ^ n5, c1 = (n3 & n4) | (n5 & (n3 ^ n4));
    const uint32_t s2 = n6 ^ n7, c2 = n6 & n7;
    const uint32_t b0 = s0 ^ s1 ^ s2, k0 = (s0 & s1) | (s2 & (s0 ^ s1));
    const uint32_t u0 = c0 ^ c1 ^ c2, v0 = (c0 & c1) | (c2 & (c0 ^ c1));
    const uint32_t b1 = u0 ^ k0, w0 = u0 & k0;
    const uint32_t b2 = v0 ^ w0, b3 = v0 & w0;
    auto tree = [&](const uint32_t* d, const uint32_t* e, uint32_t l8) {
        const uint32_t m0 = e[0] ^ (b0 & d[0]), m1 = e[1] ^ (b0 & d[1]);
        const uint32_t m2 = e[2] ^ (b0 & d[2]), m3 = e[3] ^ (b0 & d[3]);
        const uint32_t q0 = (b1 & m1) | (~b1 & m0), q1 = (b1 & m3) | (~b1 & m2);
        const uint32_t o = (b2 & q1) | (~b2 & q0);
        return (b3 & l8) | (~b3 & o);  // count 8: b0 = b1 = b2 = 0
    };
    const uint32_t sv = tree(t.sd, t.se, t.s8), bv = tree(t.bd, t.be, t.b8);
    return (centre & sv) | (~centre & bv);
}

}  // namespace nbbgpu
