// gz_bits.cuh -- bit-word helpers shared by the v4 solver (gz_tilesolve.cuh):
// per-site bit words over chain positions (bit t-1 <-> position t, NW words per
// site), the arc-mask planes, and the extraction closure (maxflow.py:267-320
// restated as a prefix reach over the final residual masks).
#pragma once

namespace gz2 {

using namespace gz;

__device__ __forceinline__ unsigned long long gtimer();

}  // namespace gz2

// device watchdog: true once the solve has run longer than p.watchdog_ns
__device__ __forceinline__ bool gz2_watchdog_expired(const gz::Prob &p) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return p.watchdog_ns && t - p.t_start_ns > p.watchdog_ns;
}

namespace gz2 {

struct Bits2 {
    uint32_t *mask;   // [13][NW][P] indexed like gz::Arc: 0 chain-up, 1..4 same-level R L D U,
                      // 5..8 diagonal-up (reverse inhibit) R L D U, 9..12 inhibit diagonal-down R L D U
    uint32_t *V, *F0, *F1, *A, *IN, *EX, *RL;   // [NW][P]
    int32_t *R0, *R1;                            // reach prefix length [P]
    int NW;
};

template <int NW>
struct BW {
    uint32_t w[NW];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < NW; ++i) w[i] = 0u;
    }
    __device__ __forceinline__ bool any() const {
        uint32_t a = 0;
#pragma unroll
        for (int i = 0; i < NW; ++i) a |= w[i];
        return a != 0u;
    }
    __device__ __forceinline__ void load(const uint32_t *base, int P, int c) {
#pragma unroll
        for (int i = 0; i < NW; ++i) w[i] = base[(size_t)i * P + c];
    }
    __device__ __forceinline__ void store(uint32_t *base, int P, int c) const {
#pragma unroll
        for (int i = 0; i < NW; ++i) base[(size_t)i * P + c] = w[i];
    }
    // toward higher positions (bit b -> b+1)
    __device__ __forceinline__ BW shl1() const {
        BW r;
#pragma unroll
        for (int i = NW - 1; i >= 0; --i) r.w[i] = (w[i] << 1) | (i > 0 ? (w[i - 1] >> 31) : 0u);
        return r;
    }
    // toward lower positions (bit b -> b-1)
    __device__ __forceinline__ BW shr1() const {
        BW r;
#pragma unroll
        for (int i = 0; i < NW; ++i) r.w[i] = (w[i] >> 1) | (i + 1 < NW ? (w[i + 1] << 31) : 0u);
        return r;
    }
    __device__ __forceinline__ int top() const {   // highest set bit index or -1
#pragma unroll
        for (int i = NW - 1; i >= 0; --i)
            if (w[i]) return 32 * i + 31 - __clz(w[i]);
        return -1;
    }
    __device__ __forceinline__ bool test(int b) const { return (w[b >> 5] >> (b & 31)) & 1u; }
    __device__ __forceinline__ void set(int b) { w[b >> 5] |= 1u << (b & 31); }
    __device__ __forceinline__ void clr(int b) { w[b >> 5] &= ~(1u << (b & 31)); }
    // bits [lo, hi) set
    __device__ __forceinline__ static BW range(int lo, int hi) {
        BW r;
#pragma unroll
        for (int i = 0; i < NW; ++i) {
            int a = lo - 32 * i, b = hi - 32 * i;
            a = a < 0 ? 0 : (a > 32 ? 32 : a);
            b = b < 0 ? 0 : (b > 32 ? 32 : b);
            uint32_t mb = b >= 32 ? 0xffffffffu : ((1u << b) - 1u);
            uint32_t ma = a >= 32 ? 0xffffffffu : ((1u << a) - 1u);
            r.w[i] = mb & ~ma;
        }
        return r;
    }
};

template <int NW>
__device__ __forceinline__ BW<NW> operator&(BW<NW> a, const BW<NW> &b) {
#pragma unroll
    for (int i = 0; i < NW; ++i) a.w[i] &= b.w[i];
    return a;
}
template <int NW>
__device__ __forceinline__ BW<NW> operator|(BW<NW> a, const BW<NW> &b) {
#pragma unroll
    for (int i = 0; i < NW; ++i) a.w[i] |= b.w[i];
    return a;
}
template <int NW>
__device__ __forceinline__ BW<NW> andnot(BW<NW> a, const BW<NW> &b) {
#pragma unroll
    for (int i = 0; i < NW; ++i) a.w[i] &= ~b.w[i];
    return a;
}


// ---------------------------------------------------------------------------
// extraction on the final masks: reach prefix r (positions lo+1 .. lo+r).
// Arc-mask word (arc q, word w) of site c.  PACK (16-lane chains, NW = 1): the
// 16-bit masks of arcs 2k and 2k+1 share word k (7 words per site instead of
// 13: fewer bytes for every mask build, BFS region load and reach pass).
template <bool PACK, int NW>
__device__ __forceinline__ uint32_t mask_word(const uint32_t *mask, int P, int q, int w, int c) {
    if (PACK) return (mask[(size_t)(q >> 1) * P + c] >> ((q & 1) * 16)) & 0xffffu;
    return mask[((size_t)q * NW + w) * P + c];
}
template <bool PACK, int NW>
__device__ __forceinline__ BW<NW> mask_bw(const uint32_t *mask, int P, int q, int c) {
    BW<NW> r;
#pragma unroll
    for (int w = 0; w < NW; ++w) r.w[w] = mask_word<PACK, NW>(mask, P, q, w, c);
    return r;
}

template <bool WIN, int NW, bool PACK = false>
__device__ int bit_close_up(const Bits2 &b, int P, int c, int lo, int hi, int r) {
    if (r <= 0) return 0;
    const BW<NW> cu = mask_bw<PACK, NW>(b.mask, P, A_UP, c);
    while (lo + r < hi && cu.test(lo + r - 1)) ++r;
    return r;
}

template <bool WIN, int NW, bool PACK = false>
__device__ bool bit_reach_iter(const Prob &p, const Bits2 &b, int c, int32_t *R) {
    const int P = p.P;
    const int y = c / p.G, g = c - y * p.G;
    const bool has[4] = {g + 1 < p.G, g > 0, y + 1 < p.Y, y > 0};
    const int nc[4] = {c + 1, c - 1, c + p.G, c - p.G};
    int lo = 0, hi = p.L;
    if (WIN) { lo = p.lo[c]; hi = p.hi[c]; }
    const int r0 = R[c];
    int r = r0;
    BW<NW> T;
    T.zero();
    bool anyn = false;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (!has[i]) continue;
        const int rn = R[nc[i]];
        if (rn <= 0) continue;
        const int lon = WIN ? p.lo[nc[i]] : 0;
        BW<NW> Rn = BW<NW>::range(lon, lon + rn);
        const int j = i ^ 1;   // direction from the neighbour back to c
        const BW<NW> s = mask_bw<PACK, NW>(b.mask, P, A_SR + j, nc[i]);
        const BW<NW> dd = mask_bw<PACK, NW>(b.mask, P, A_DR + j, nc[i]);
        const BW<NW> uu = mask_bw<PACK, NW>(b.mask, P, A_UR + j, nc[i]);
        T = T | (Rn & s) | (Rn & dd).shr1() | (Rn & uu).shl1();
        anyn = true;
    }
    if (anyn) {
        T = T & BW<NW>::range(lo, hi);
        const int top = T.top();
        if (top >= 0 && top + 1 - lo > r) r = bit_close_up<WIN, NW, PACK>(b, P, c, lo, hi, top + 1 - lo);
    }
    if (r == r0) return false;
    R[c] = r;   // in place: see the reach loop in gz_tilesolve.cuh
    return true;
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

}  // namespace gz2
