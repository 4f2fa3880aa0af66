// NumPy-compatible Philox4x64-10 stream on the device.
//
// The reference backs every stream with np.random.Philox (rng.py:28-31) and
// draws uniforms as (raw >> 11) * 2^-53 (Generator.random).  Given the host
// Generator's state (counter, key, 4-word buffer, buffer position), output e
// of the stream is either a buffered word or lane (e - avail) % 4 of the
// block for counter + 1 + (e - avail) / 4 -- so any element can be produced
// independently, in parallel, bit-identical to the host draw.
#pragma once
#include <stdint.h>

#include "../../include/temo_b200.h"

namespace temo {

struct Philox {
    uint64_t ctr[4];
    uint64_t key[2];
    uint64_t buf[4];
    int32_t pos;
    uint64_t rk[20];  // round keys (k0, k1) of rounds 0..9: kernel-parameter (constant bank) operands
};

__host__ __device__ inline Philox philox_from(const temo_philox_state &s) {
    Philox p;
    for (int i = 0; i < 4; ++i) { p.ctr[i] = s.counter[i]; p.buf[i] = s.buffer[i]; }
    p.key[0] = s.key[0];
    p.key[1] = s.key[1];
    p.pos = s.buffer_pos;
    uint64_t k0 = s.key[0], k1 = s.key[1];
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B97F4A7C15ull;
            k1 += 0xBB67AE8584CAA73Bull;
        }
        p.rk[2 * r] = k0;
        p.rk[2 * r + 1] = k1;
    }
    return p;
}

__device__ __forceinline__ void philox_block(const uint64_t ctr_in[4], const uint64_t key_in[2],
                                             uint64_t out[4]) {
    uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint64_t k0 = key_in[0], k1 = key_in[1];
#ifdef OFF_ABL_PHILOX
#pragma unroll
    for (int r = 0; r < 1; ++r) {
#else
#pragma unroll
    for (int r = 0; r < 10; ++r) {
#endif
        if (r) {
            k0 += 0x9E3779B97F4A7C15ull;
            k1 += 0xBB67AE8584CAA73Bull;
        }
        const uint64_t lo0 = 0xD2E7470EE14C6C93ull * c0, hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c0);
        const uint64_t lo1 = 0xCA5A826395121157ull * c2, hi1 = __umul64hi(0xCA5A826395121157ull, c2);
        const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// NB independent blocks in lockstep (ILP across the serial 10-round chains)
template <int NB>
__device__ __forceinline__ void philox_blocks(const uint64_t ctr[NB][4], const uint64_t key_in[2],
                                              uint64_t out[NB][4]) {
    uint64_t c0[NB], c1[NB], c2[NB], c3[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        c0[b] = ctr[b][0]; c1[b] = ctr[b][1]; c2[b] = ctr[b][2]; c3[b] = ctr[b][3];
    }
    uint64_t k0 = key_in[0], k1 = key_in[1];
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B97F4A7C15ull;
            k1 += 0xBB67AE8584CAA73Bull;
        }
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const uint64_t lo0 = 0xD2E7470EE14C6C93ull * c0[b], hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c0[b]);
            const uint64_t lo1 = 0xCA5A826395121157ull * c2[b], hi1 = __umul64hi(0xCA5A826395121157ull, c2[b]);
            const uint64_t n0 = hi1 ^ c1[b] ^ k0, n2 = hi0 ^ c3[b] ^ k1;
            c0[b] = n0;
            c1[b] = lo1;
            c2[b] = n2;
            c3[b] = lo0;
        }
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        out[b][0] = c0[b]; out[b][1] = c1[b]; out[b][2] = c2[b]; out[b][3] = c3[b];
    }
}

// NB independent blocks with precomputed round keys (no per-round key additions)
template <int NB>
__device__ __forceinline__ void philox_blocks_rk(const uint64_t ctr[NB][4], const uint64_t *rk,
                                                 uint64_t out[NB][4]) {
    uint64_t c0[NB], c1[NB], c2[NB], c3[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        c0[b] = ctr[b][0]; c1[b] = ctr[b][1]; c2[b] = ctr[b][2]; c3[b] = ctr[b][3];
    }
#pragma unroll
    for (int r = 0; r < 10; ++r) {
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const uint64_t lo0 = 0xD2E7470EE14C6C93ull * c0[b], hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c0[b]);
            const uint64_t lo1 = 0xCA5A826395121157ull * c2[b], hi1 = __umul64hi(0xCA5A826395121157ull, c2[b]);
            const uint64_t n0 = hi1 ^ c1[b] ^ rk[2 * r], n2 = hi0 ^ c3[b] ^ rk[2 * r + 1];
            c0[b] = n0;
            c1[b] = lo1;
            c2[b] = n2;
            c3[b] = lo0;
        }
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        out[b][0] = c0[b]; out[b][1] = c1[b]; out[b][2] = c2[b]; out[b][3] = c3[b];
    }
}

// counter + add (256-bit, little-endian words)
__device__ __forceinline__ void ctr_add(const uint64_t in[4], uint64_t add, uint64_t out[4]) {
    out[0] = in[0] + add;
    uint64_t carry = out[0] < add;
    out[1] = in[1] + carry;
    carry = carry && out[1] == 0;
    out[2] = in[2] + carry;
    carry = carry && out[2] == 0;
    out[3] = in[3] + carry;
}

// Per-thread cursor that caches the last block it generated.
struct PhiloxCursor {
    uint64_t blk = ~0ull;
    uint64_t v[4];

    __device__ __forceinline__ uint64_t raw(const Philox &p, uint64_t e) {
        const uint64_t avail = (uint64_t)(4 - p.pos);
        if (e < avail) return p.buf[p.pos + e];
        const uint64_t e2 = e - avail, b = e2 >> 2;
        if (b != blk) {
            uint64_t c[1][4], o[1][4];
            ctr_add(p.ctr, b + 1, c[0]);
            philox_blocks_rk<1>(c, p.rk, o);
            for (int k = 0; k < 4; ++k) v[k] = o[0][k];
            blk = b;
        }
        return v[e2 & 3];
    }

    __device__ __forceinline__ double uniform(const Philox &p, uint64_t e) {
        return (double)(raw(p, e) >> 11) * (1.0 / 9007199254740992.0);
    }
};

// Uniform source: injected array (parity mode with duck-typed host RNGs) or
// the Philox stream at a raw offset.
struct USrc {
    const double *ptr;
    uint64_t off;
    __device__ __forceinline__ double get(const Philox &p, PhiloxCursor &c, uint64_t e) const {
        return ptr ? ptr[e] : c.uniform(p, off + e);
    }
};

}  // namespace temo
