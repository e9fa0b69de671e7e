// frames.cuh -- synthetic BSC frames, bit-identical to the reference's
// counter-based frame streams, generated where they are decoded.
//
// The reference draws frame `idx` of a grid point as (bench._frame_inputs,
// bench.py:123-130; channel.rng_stream, channel.py:29-35):
//     key   = Generator(Philox(key=SeedSequence((seed,*path,idx,0)).generate_state(2,u64)))
//                 .integers(0, 2, size=n, dtype=uint8)
//     flips = Generator(Philox(key=SeedSequence((seed,*path,idx,1)).generate_state(2,u64)))
//                 .random(n) < e
// i.e. numpy 2.3's SeedSequence (pool of 4 uint32, hashmix / mix), Philox
// 4x64-10 with a zero counter that is incremented before each 4-word block,
// the 32-bit draws split from 64-bit outputs low half first, integers(0, 2,
// uint8) = Lemire's bounded draw on buffered bytes (range 2: the top bit of
// each byte, never rejecting), random() = (w >> 11) * 2^-53.  So with w_k the
// k-th 64-bit Philox output of a stream:
//     key bit i  = bit 8*(i%8)+7 of w_{i/8}        (block i/32, counter i/32+1)
//     flip bit i = (double)(w_i >> 11) * 2^-53 < e  (block i/4,  counter i/4+1)
// Each output position depends only on its own counter, so the generator is
// embarrassingly parallel: one thread makes one 32-bit word of a packed
// BitBlock row (1 Philox block for the key, 8 for the flips).  Everything
// here is __host__ __device__ so the host build pins it against numpy on CPU
// (tests/test_frames.py) and the device build is checked against that.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace mbp {
namespace frames {

constexpr int kMaxEntropyWords = 24;

struct Key2 { uint64_t k0, k1; };

__host__ __device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b)
{
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// Philox 4x64, 10 rounds (Random123 constants)
__host__ __device__ __forceinline__ void philox4x64_10(uint64_t c[4], Key2 k)
{
    const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
    const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#ifdef __CUDA_ARCH__
#pragma unroll
#endif
    for (int r = 0; r < 10; ++r) {
        if (r) { k.k0 += W0; k.k1 += W1; }
        const uint64_t lo0 = M0 * c[0], hi0 = mulhi64(M0, c[0]);
        const uint64_t lo1 = M1 * c[2], hi1 = mulhi64(M1, c[2]);
        const uint64_t n0 = hi1 ^ c[1] ^ k.k0, n2 = hi0 ^ c[3] ^ k.k1;
        c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    }
}

// numpy SeedSequence(entropy).generate_state(2, uint64), entropy given as the
// concatenation of its uint32 words (_coerce_to_uint32_array)
__host__ __device__ __forceinline__ Key2 seed_sequence_key(const uint32_t* w, int len)
{
    const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
    const uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
    uint32_t hc = INIT_A;
    auto hashmix = [&](uint32_t v) {
        v ^= hc;
        hc *= MULT_A;
        v *= hc;
        v ^= v >> 16;
        return v;
    };
    auto mix = [](uint32_t x, uint32_t y) {
        uint32_t r = MIX_L * x - MIX_R * y;
        r ^= r >> 16;
        return r;
    };
    uint32_t pool[4];
    for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < len ? w[i] : 0u);
    for (int s = 0; s < 4; ++s)
        for (int d = 0; d < 4; ++d)
            if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
    for (int s = 4; s < len; ++s)
        for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(w[s]));
    uint32_t hb = INIT_B, st[4];
    for (int i = 0; i < 4; ++i) {
        uint32_t v = pool[i] ^ hb;
        hb *= MULT_B;
        v *= hb;
        v ^= v >> 16;
        st[i] = v;
    }
    return Key2{(uint64_t)st[0] | ((uint64_t)st[1] << 32), (uint64_t)st[2] | ((uint64_t)st[3] << 32)};
}

// entropy words of (prefix..., idx, purpose): a non-negative int is its
// little-endian 32-bit words, 0 being one zero word
__host__ __device__ __forceinline__ Key2 frame_key(const uint32_t* prefix, int plen, uint64_t idx, uint32_t purpose)
{
    uint32_t w[kMaxEntropyWords];
    int len = 0;
    for (int i = 0; i < plen; ++i) w[len++] = prefix[i];
    w[len++] = (uint32_t)idx;
    if (idx >> 32) w[len++] = (uint32_t)(idx >> 32);
    w[len++] = purpose;
    return seed_sequence_key(w, len);
}

// 32 key bits starting at bit 32*j: Philox block j (counter j+1)
__host__ __device__ __forceinline__ uint32_t key_word(Key2 k, uint64_t j)
{
    uint64_t c[4] = {j + 1, 0, 0, 0};
    philox4x64_10(c, k);
    uint32_t out = 0;
#ifdef __CUDA_ARCH__
#pragma unroll
#endif
    for (int q = 0; q < 4; ++q)
        for (int b = 0; b < 8; ++b) out |= (uint32_t)((c[q] >> (8 * b + 7)) & 1u) << (8 * q + b);
    return out;
}

// 32 flip bits starting at bit 32*j: Philox blocks 8j .. 8j+7
__host__ __device__ __forceinline__ uint32_t flip_word(Key2 k, uint64_t j, double e)
{
    uint32_t out = 0;
#ifdef __CUDA_ARCH__
#pragma unroll 2
#endif
    for (int blk = 0; blk < 8; ++blk) {
        uint64_t c[4] = {8 * j + blk + 1, 0, 0, 0};
        philox4x64_10(c, k);
        for (int q = 0; q < 4; ++q)
            out |= (uint32_t)((double)(c[q] >> 11) * (1.0 / 9007199254740992.0) < e) << (4 * blk + q);
    }
    return out;
}

struct FrameArgs {
    uint32_t prefix[kMaxEntropyWords - 3];
    int plen;
    int n;
    long long nb;        // row bytes ceil(n/8)
    long long first;     // frame index of row 0
    long long batch;
    double e;
};

// keys[f] = (frame_key(.., first+f, 0), frame_key(.., first+f, 1))
__global__ void frame_keys_kernel(FrameArgs A, Key2* __restrict__ keys)
{
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2 * A.batch) return;
    keys[t] = frame_key(A.prefix, A.plen, (uint64_t)(A.first + (t >> 1)), (uint32_t)(t & 1));
}

// one thread per (frame, 32-bit word): packed key and noisy rows
__global__ void frame_bits_kernel(FrameArgs A, const Key2* __restrict__ keys, uint8_t* __restrict__ key_rows,
                                  uint8_t* __restrict__ noisy_rows)
{
    const long long words = (A.n + 31) / 32;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= words * A.batch) return;
    const long long f = t / words, j = t - f * words;
    const Key2 kk = keys[2 * f], kf = keys[2 * f + 1];
    uint32_t kw = key_word(kk, (uint64_t)j);
    uint32_t fw = flip_word(kf, (uint64_t)j, A.e);
    const int rem = A.n - (int)(32 * j);
    if (rem < 32) {   // zero padding bits (bits.py: padding must be zero)
        const uint32_t mask = (1u << rem) - 1u;
        kw &= mask;
        fw &= mask;
    }
    const uint32_t yw = kw ^ fw;
    const long long base = f * A.nb + 4 * j;
    if ((A.nb & 3) == 0) {
        *reinterpret_cast<uint32_t*>(key_rows + base) = kw;
        *reinterpret_cast<uint32_t*>(noisy_rows + base) = yw;
    } else {
        for (int b = 0; b < 4 && 4 * j + b < A.nb; ++b) {
            key_rows[base + b] = (uint8_t)(kw >> (8 * b));
            noisy_rows[base + b] = (uint8_t)(yw >> (8 * b));
        }
    }
}

}  // namespace frames
}  // namespace mbp
