// Shared-memory FFT building blocks for the TVOLAP kernels (sm_100a).
//
// The reference transforms a real 4L block through a 2L-point complex radix-2
// DIT plus a pack/untangle step (proj/src/spectral.cpp:99-125, inverse
// :127-158). Here the same half-length trick runs as a Stockham auto-sort
// FFT in shared memory: radix-4 stages (radix-2 for an odd power), one
// butterfly per thread per stage, ping-ponging between two smem buffers so no
// bit-reversal pass is needed. Twiddles come from an fp64-computed table
// rounded once to fp32 (SURVEY.md §7 hard part 1), so the fp32 transform error
// stays ~1e-7 relative.
#pragma once

#include <cuda_runtime.h>

#include <cmath>

namespace tvb {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
    return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
    return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

// acc += h * x for two packed bins (one float4 = two complex64), plus the Nyquist product of the
// first one (only kept for the packed bin 0 = (Re X_0, Re X_N), spectral.cpp:121-123):
// engine.cpp:85-92 / spectral.cpp:160-166.
__device__ __forceinline__ void cmac4(float4& acc, float& aux, const float4 h, const float4 x) {
    acc.x = fmaf(h.x, x.x, acc.x);
    acc.x = fmaf(-h.y, x.y, acc.x);
    acc.y = fmaf(h.x, x.y, acc.y);
    acc.y = fmaf(h.y, x.x, acc.y);
    acc.z = fmaf(h.z, x.z, acc.z);
    acc.z = fmaf(-h.w, x.w, acc.z);
    acc.w = fmaf(h.z, x.w, acc.w);
    acc.w = fmaf(h.w, x.z, acc.w);
    aux = fmaf(h.y, x.y, aux);
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }

// Radix of the Stockham stage that starts at sub-transform length Ns: 8 while possible, but a
// remaining factor of 16 is done as 4 x 4 rather than 8 x 2 (a radix-2 pass costs more per
// point than a radix-8 one). 1024 = 8.8.4.4, 512 = 8.8.8, 256 = 8.8.4, 64 = 8.8.
__host__ __device__ __forceinline__ int fft_radix(int N, int Ns) {
    const int rem = N / Ns;
    if (rem == 16) return 4;
    return (rem & 7) == 0 ? 8 : ((rem & 3) == 0 ? 4 : 2);
}

// Number of Stockham stages for length N (decides which ping-pong buffer holds the result).
__host__ __device__ __forceinline__ int fft_stage_count(int N) {
    int k = 0;
    for (int Ns = 1; Ns < N; Ns *= fft_radix(N, Ns)) ++k;
    return k;
}

// Intermediate Stockham stages store to a swizzled layout (low 3 index bits XOR bits 3..5):
// a permutation inside aligned groups of 8 elements that spreads the stride-R stores of the
// early stages over the shared-memory banks. The first stage reads and the last stage writes
// the natural layout, so callers never see it.
__device__ __forceinline__ int fsw(int i, bool on) { return on ? (i ^ ((i >> 3) & 7)) : i; }

// Host side: the stage twiddle table for length N (fp64 angles, rounded once), N entries.
template <class F2, class MAKE>
inline void fft_stage_twiddles(int N, F2* out, MAKE make) {
    const double pi = 3.14159265358979323846264338327950288;
    for (int Ns = 1; Ns < N;) {
        const int R = fft_radix(N, Ns);
        for (int k = 0; k < Ns; ++k)
            for (int r = 1; r < R; ++r) {
                const double a = -2.0 * pi * (double)k * (double)r / (double)(Ns * R);
                out[(Ns - 1) + k * (R - 1) + (r - 1)] = make(std::cos(a), std::sin(a));
            }
        Ns *= R;
    }
    out[N - 1] = make(0.0, 0.0);  // unused pad entry (the table has N - 1 live entries)
}

template <bool INV>
__device__ __forceinline__ float2 twmul(float2 v, float2 w) {
    return INV ? cmulc(v, w) : cmul(v, w);
}

// In-register 4-point DFT (sign -1 forward, +1 inverse).
template <bool INV>
__device__ __forceinline__ void dft4(float2& v0, float2& v1, float2& v2, float2& v3) {
    const float2 a0 = cadd(v0, v2), a1 = csub(v0, v2);
    const float2 a2 = cadd(v1, v3), a3 = csub(v1, v3);
    v0 = cadd(a0, a2);
    v2 = csub(a0, a2);
    if (INV) {  // y1 = a1 + i a3, y3 = a1 - i a3
        v1 = make_float2(a1.x - a3.y, a1.y + a3.x);
        v3 = make_float2(a1.x + a3.y, a1.y - a3.x);
    } else {    // y1 = a1 - i a3, y3 = a1 + i a3
        v1 = make_float2(a1.x + a3.y, a1.y - a3.x);
        v3 = make_float2(a1.x - a3.y, a1.y + a3.x);
    }
}

// In-register 8-point DFT: radix-2 split n = n1 + 4 n2, then two 4-point DFTs
// (even outputs from b0..b3, odd outputs from W8^n1 * b(n1+4)).
template <bool INV>
__device__ __forceinline__ void dft8(float2 (&v)[8]) {
    constexpr float c = 0.70710678118654752440f;
    float2 b[8];
#pragma unroll
    for (int n = 0; n < 4; ++n) {
        b[n] = cadd(v[n], v[n + 4]);
        b[n + 4] = csub(v[n], v[n + 4]);
    }
    // W8^1, W8^2, W8^3 (conjugated for the inverse)
    if (INV) {
        b[5] = make_float2((b[5].x - b[5].y) * c, (b[5].x + b[5].y) * c);
        b[6] = make_float2(-b[6].y, b[6].x);
        b[7] = make_float2(-(b[7].x + b[7].y) * c, (b[7].x - b[7].y) * c);
    } else {
        b[5] = make_float2((b[5].x + b[5].y) * c, (b[5].y - b[5].x) * c);
        b[6] = make_float2(b[6].y, -b[6].x);
        b[7] = make_float2((b[7].y - b[7].x) * c, -(b[7].x + b[7].y) * c);
    }
    dft4<INV>(b[0], b[1], b[2], b[3]);
    dft4<INV>(b[4], b[5], b[6], b[7]);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[2 * k] = b[k];
        v[2 * k + 1] = b[k + 4];
    }
}

// One Stockham stage: nf transforms, sub-transform length Ns -> Ns*R.
template <bool INV>
__device__ __forceinline__ void fft_stage(const float2* src, float2* dst, int N, int Ns, int nf,
                                          const float2* __restrict__ tw, bool prune, int tid, int nthreads) {
    const int R = fft_radix(N, Ns);
    const int nb = N / R;
    const bool zero_hi = prune && Ns == 1;  // legs r >= R/2 read the zero upper half
    const int lgnb = 31 - __clz(nb);
    const bool rs = Ns > 1, ws = Ns * R < N;  // read / write the swizzled intermediate layout
    const float2* tws = tw + (Ns - 1);        // this stage's twiddles: [k][r-1], k < Ns, r < R
    for (int jj = tid; jj < nb * nf; jj += nthreads) {
        const int f = jj >> lgnb, j = jj & (nb - 1);
        const float2* sf = src + (size_t)f * N;
        float2* df = dst + (size_t)f * N;
        const int k = j & (Ns - 1);
        const int idxD = (j - k) * R + k;
        if (R == 8) {
            float2 v[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) v[r] = (zero_hi && r >= 4) ? make_float2(0.f, 0.f) : sf[fsw(j + r * nb, rs)];
            if (Ns > 1) {
                const float2* w = tws + k * 7;
#pragma unroll
                for (int r = 1; r < 8; ++r) v[r] = twmul<INV>(v[r], w[r - 1]);
            }
            dft8<INV>(v);
#pragma unroll
            for (int r = 0; r < 8; ++r) df[fsw(idxD + r * Ns, ws)] = v[r];
        } else if (R == 4) {
            float2 v0 = sf[fsw(j, rs)];
            float2 v1 = sf[fsw(j + nb, rs)];
            float2 v2 = zero_hi ? make_float2(0.f, 0.f) : sf[fsw(j + 2 * nb, rs)];
            float2 v3 = zero_hi ? make_float2(0.f, 0.f) : sf[fsw(j + 3 * nb, rs)];
            if (Ns > 1) {
                const float2* w = tws + k * 3;
                v1 = twmul<INV>(v1, w[0]);
                v2 = twmul<INV>(v2, w[1]);
                v3 = twmul<INV>(v3, w[2]);
            }
            dft4<INV>(v0, v1, v2, v3);
            df[fsw(idxD, ws)] = v0;
            df[fsw(idxD + Ns, ws)] = v1;
            df[fsw(idxD + 2 * Ns, ws)] = v2;
            df[fsw(idxD + 3 * Ns, ws)] = v3;
        } else {
            float2 v0 = sf[fsw(j, rs)];
            float2 v1 = zero_hi ? make_float2(0.f, 0.f) : sf[fsw(j + nb, rs)];
            if (Ns > 1) v1 = twmul<INV>(v1, tws[k]);
            df[fsw(idxD, ws)] = cadd(v0, v1);
            df[fsw(idxD + Ns, ws)] = csub(v0, v1);
        }
    }
    __syncthreads();
}

// Batched Stockham FFT of `nf` length-N transforms stored back to back in `a`
// (N a power of two >= 2), `b` the ping-pong buffer. `tw` is the stage twiddle table built by
// fft_stage_twiddles(): stage with sub-length Ns and radix R keeps W^(k r) for k < Ns, 1 <= r < R
// contiguously per k at offset Ns - 1 (N - 1 entries in all), so each thread reads consecutive
// entries and a warp's twiddle loads spread over the banks.
// Radix-8 stages (radix-4/2 for the remainder): each thread keeps one butterfly's
// 8 points in registers, so a 512-point transform is 3 shared-memory passes.
// When `prune` is set the upper half of every input is taken as zero and never
// read (the engine's 4L block is zero-padded past 2L, proj/src/engine.cpp:77-80).
// NC != 0 fixes N at compile time: the stages unroll and all index math folds.
// All threads of the CTA must call this; returns the buffer holding the result.
template <bool INV, int NC = 0>
__device__ float2* fft_batch(float2* a, float2* b, int N, int nf, const float2* __restrict__ tw, bool prune, int tid,
                             int nthreads) {
    float2* src = a;
    float2* dst = b;
    if constexpr (NC != 0) {
        (void)N;
        int Ns = 1;
#pragma unroll
        for (int st = 0; st < 12; ++st) {
            if (Ns >= NC) break;
            fft_stage<INV>(src, dst, NC, Ns, nf, tw, prune, tid, nthreads);
            float2* t = src;
            src = dst;
            dst = t;
            Ns *= fft_radix(NC, Ns);
        }
    } else {
        for (int Ns = 1; Ns < N;) {
            fft_stage<INV>(src, dst, N, Ns, nf, tw, prune, tid, nthreads);
            float2* t = src;
            src = dst;
            dst = t;
            Ns *= fft_radix(N, Ns);
        }
    }
    return src;
}

// One warp, one transform, in place in a warp-private smem buffer (no CTA barriers): every
// Stockham stage gathers this lane's butterflies into registers, __syncwarp, scatters the
// outputs over the same buffer, __syncwarp. Each butterfly does exactly the operations of
// fft_stage (same twiddles, same radix kernels), so results are bit-identical to fft_batch.
// The first stage reads its inputs through `load0(n)` (natural order, n < N/2: the upper half
// is zero, `prune`); the result is left in natural order in `buf`.
__host__ __device__ constexpr int fft_radix_c(int N, int Ns) {
    return (N / Ns == 16) ? 4 : (((N / Ns) & 7) == 0 ? 8 : (((N / Ns) & 3) == 0 ? 4 : 2));
}

template <bool INV, int N, int Ns, class LOAD0>
__device__ __forceinline__ void fft_warp_stages(float2* buf, const float2* __restrict__ tw, int lane,
                                                const LOAD0& load0) {
    if constexpr (Ns < N) {
        constexpr int R = fft_radix_c(N, Ns);
        constexpr int nb = N / R;
        constexpr int BPL = (nb + 31) / 32;  // butterflies per lane
        constexpr bool rs = Ns > 1, ws = Ns * R < N;
        const float2* tws = tw + (Ns - 1);
        float2 v[BPL][R];
#pragma unroll
        for (int b = 0; b < BPL; ++b) {
            const int j = lane + 32 * b;
            if (nb >= 32 || j < nb) {
                const int k = j & (Ns - 1);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if constexpr (Ns == 1)
                        v[b][r] = r < R / 2 ? load0(j + r * nb) : make_float2(0.f, 0.f);
                    else
                        v[b][r] = buf[fsw(j + r * nb, rs)];
                }
                if constexpr (Ns > 1) {
#pragma unroll
                    for (int r = 1; r < R; ++r) v[b][r] = twmul<INV>(v[b][r], tws[k * (R - 1) + (r - 1)]);
                }
                if constexpr (R == 8) {
                    dft8<INV>(v[b]);
                } else if constexpr (R == 4) {
                    dft4<INV>(v[b][0], v[b][1], v[b][2], v[b][3]);
                } else {
                    const float2 t0 = cadd(v[b][0], v[b][1]), t1 = csub(v[b][0], v[b][1]);
                    v[b][0] = t0;
                    v[b][1] = t1;
                }
            }
        }
        __syncwarp();
#pragma unroll
        for (int b = 0; b < BPL; ++b) {
            const int j = lane + 32 * b;
            if (nb >= 32 || j < nb) {
                const int k = j & (Ns - 1);
                const int idxD = (j - k) * R + k;
#pragma unroll
                for (int r = 0; r < R; ++r) buf[fsw(idxD + r * Ns, ws)] = v[b][r];
            }
        }
        __syncwarp();
        fft_warp_stages<INV, N, Ns * R>(buf, tw, lane, load0);
    }
}

// ---------------------------------------------------------------- register-resident warp FFT
// W_32^j = exp(-2 pi i j / 32) (fp64 values rounded once; quarter turns exact).
__device__ __forceinline__ float2 w32c(int j) {
    constexpr float c[32] = {
        1.f, 9.807852507e-01f, 9.238795042e-01f, 8.314695954e-01f, 7.071067691e-01f, 5.555702448e-01f,
        3.826834261e-01f, 1.950903237e-01f, 0.f, -1.950903237e-01f, -3.826834261e-01f, -5.555702448e-01f,
        -7.071067691e-01f, -8.314695954e-01f, -9.238795042e-01f, -9.807852507e-01f, -1.f, -9.807852507e-01f,
        -9.238795042e-01f, -8.314695954e-01f, -7.071067691e-01f, -5.555702448e-01f, -3.826834261e-01f,
        -1.950903237e-01f, 0.f, 1.950903237e-01f, 3.826834261e-01f, 5.555702448e-01f, 7.071067691e-01f,
        8.314695954e-01f, 9.238795042e-01f, 9.807852507e-01f};
    return make_float2(c[j & 31], c[(j + 8) & 31]);  // -sin(x) = cos(x + pi / 2)
}

// In-register DFT of R = 1..32 points, natural order in and out (sign -1 forward, +1 inverse).
// 16 = 4 x 4 and 32 = 8 x 4 four-step splits with compile-time twiddles. HALF: the upper half
// of the input is zero (pruned transforms): the first butterfly level keeps x +- 0 = x (equal
// values; only the sign of a zero can differ) instead of adding zeros.
template <bool INV, int R, bool HALF = false>
__device__ __forceinline__ void dft_reg(float2 (&v)[R]) {
    if constexpr (R == 2) {
        const float2 t0 = HALF ? v[0] : cadd(v[0], v[1]), t1 = HALF ? v[0] : csub(v[0], v[1]);
        v[0] = t0;
        v[1] = t1;
    } else if constexpr (R == 4 && HALF) {
        const float2 a0 = v[0], a2 = v[1];  // dft4 with v2 = v3 = 0: a1 = a0, a3 = a2
        v[0] = cadd(a0, a2);
        v[2] = csub(a0, a2);
        if (INV) {
            v[1] = make_float2(a0.x - a2.y, a0.y + a2.x);
            v[3] = make_float2(a0.x + a2.y, a0.y - a2.x);
        } else {
            v[1] = make_float2(a0.x + a2.y, a0.y - a2.x);
            v[3] = make_float2(a0.x - a2.y, a0.y + a2.x);
        }
    } else if constexpr (R == 4) {
        dft4<INV>(v[0], v[1], v[2], v[3]);
    } else if constexpr (R == 8 && HALF) {
        // dft8 with v4..v7 = 0: b[n] = b[n + 4] = v[n]
        constexpr float c = 0.70710678118654752440f;
        float2 b[8];
#pragma unroll
        for (int n = 0; n < 4; ++n) b[n] = b[n + 4] = v[n];
        if (INV) {
            b[5] = make_float2((b[5].x - b[5].y) * c, (b[5].x + b[5].y) * c);
            b[6] = make_float2(-b[6].y, b[6].x);
            b[7] = make_float2(-(b[7].x + b[7].y) * c, (b[7].x - b[7].y) * c);
        } else {
            b[5] = make_float2((b[5].x + b[5].y) * c, (b[5].y - b[5].x) * c);
            b[6] = make_float2(b[6].y, -b[6].x);
            b[7] = make_float2((b[7].y - b[7].x) * c, -(b[7].x + b[7].y) * c);
        }
        dft4<INV>(b[0], b[1], b[2], b[3]);
        dft4<INV>(b[4], b[5], b[6], b[7]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[2 * k] = b[k];
            v[2 * k + 1] = b[k + 4];
        }
    } else if constexpr (R == 8) {
        dft8<INV>(v);
    } else if constexpr (R == 16 || R == 32) {
        constexpr int A = R / 4;  // inner DFT length over a (n = 4 a + b), then 4-point DFTs over b
        float2 y[4][A];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
#pragma unroll
            for (int a = 0; a < A; ++a) y[b][a] = v[4 * a + b];
            dft_reg<INV, A, HALF>(y[b]);  // HALF: v[4a + b] = 0 for a >= A / 2
#pragma unroll
            for (int ka = 1; ka < A; ++ka)
                if (b > 0) y[b][ka] = twmul<INV>(y[b][ka], w32c((32 / R) * b * ka));
        }
#pragma unroll
        for (int ka = 0; ka < A; ++ka) {
            dft4<INV>(y[0][ka], y[1][ka], y[2][ka], y[3][ka]);
#pragma unroll
            for (int kb = 0; kb < 4; ++kb) v[ka + A * kb] = y[kb][ka];
        }
    }
}

// Host side: the four-step tables appended after the stage table (tw[N .. 2N + 32)):
// tw4[k1 * 32 + t] = W_N^(t k1) for k1 < N / 32, then W_32^j for j < 32.
template <class F2, class MAKE>
inline void fft_warp_twiddles(int N, F2* out, MAKE make) {
    const double pi = 3.14159265358979323846264338327950288;
    const int n1 = N / 32;
    for (int i = 0; i < N; ++i) out[i] = make(0.0, 0.0);
    for (int k1 = 0; k1 < n1; ++k1)
        for (int t = 0; t < 32; ++t) {
            const double a = -2.0 * pi * (double)t * (double)k1 / (double)N;
            out[k1 * 32 + t] = make(std::cos(a), std::sin(a));
        }
    for (int j = 0; j < 32; ++j) {
        const double a = -2.0 * pi * (double)j / 32.0;
        out[N + j] = make(std::cos(a), std::sin(a));
    }
}

__host__ __device__ constexpr int bitrev_c(int x, int bits) {
    int r = 0;
    for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1) << (bits - 1 - i);
    return r;
}

// One N-point transform per warp (64 <= N <= 1024) with the data in registers: N = N1 x 32,
// lane t takes x[32 n1 + t] (`load(n)`; with PRUNE the upper half is zero and never loaded),
// an N1-point DFT in registers, twiddles W_N^(t k1), one swizzled transpose through the
// warp's buffer, N1-point DFTs over the columns (B = 32 / N1 lanes per column) and a B-point
// DFT across those lanes with shuffles. The result is left in natural order in buf[0 .. N).
// tw4 = the four-step tables (fft_warp_twiddles). Roughly half the instructions of the
// radix-8 Stockham passes and no CTA barriers.
template <bool INV, int N, bool PRUNE, int NB = 1, class LOAD, bool INPLACE = false>
__device__ __forceinline__ void fft_warp4(float2* buf, const float2* __restrict__ tw4, int lane, const LOAD& load) {
    // INPLACE: `load` may read `buf` (every lane's inputs are loaded before any lane stores)
    // NB transforms in lockstep (independent instruction streams for ILP): transform t uses
    // buf + t N and reads its input through load(t, n).
    static_assert(N >= 64 && N <= 1024, "warp FFT covers 64..1024 points");
    constexpr int N1 = N / 32, B = 32 / N1;
    constexpr int lgB = B == 1 ? 0 : B == 2 ? 1 : B == 4 ? 2 : B == 8 ? 3 : 4;
    float2 v[NB][N1];
#pragma unroll
    for (int t = 0; t < NB; ++t)
#pragma unroll
        for (int n1 = 0; n1 < N1; ++n1)
            v[t][n1] = (PRUNE && n1 >= N1 / 2) ? make_float2(0.f, 0.f) : load(t, 32 * n1 + lane);
    if constexpr (INPLACE) __syncwarp();
#pragma unroll
    for (int t = 0; t < NB; ++t) {
        dft_reg<INV, N1, PRUNE>(v[t]);
#pragma unroll
        for (int k1 = 1; k1 < N1; ++k1) v[t][k1] = twmul<INV>(v[t][k1], tw4[k1 * 32 + lane]);
#pragma unroll
        for (int k1 = 0; k1 < N1; ++k1) buf[t * N + k1 * 32 + (lane ^ ((B * k1) & 31))] = v[t][k1];
    }
    __syncwarp();
    const int k1 = lane >> lgB, b = lane & (B - 1);
#pragma unroll
    for (int t = 0; t < NB; ++t) {
#pragma unroll
        for (int a = 0; a < N1; ++a) v[t][a] = buf[t * N + k1 * 32 + B * (a ^ k1) + b];
        dft_reg<INV, N1>(v[t]);
    }
    if constexpr (B > 1) {
        const float2* w32 = tw4 + N;
#pragma unroll
        for (int c = 1; c < N1; ++c) {
            const float2 w = w32[(b * c) & 31];
#pragma unroll
            for (int t = 0; t < NB; ++t)
                if (b) v[t][c] = twmul<INV>(v[t][c], w);
        }
#pragma unroll
        for (int hs = B / 2; hs >= 1; hs /= 2) {  // radix-2 DIF across the column's lanes
            const bool upper = (b & hs) != 0;
            const float2 w = w32[(b & (hs - 1)) * (16 / hs)];
#pragma unroll
            for (int t = 0; t < NB; ++t)
#pragma unroll
                for (int c = 0; c < N1; ++c) {
                    float2 o;
                    o.x = __shfl_xor_sync(0xffffffffu, v[t][c].x, hs);
                    o.y = __shfl_xor_sync(0xffffffffu, v[t][c].y, hs);
                    // the last level (hs = 1) multiplies by W^0 = 1: skipped (equal values)
                    v[t][c] = upper ? (hs == 1 ? csub(o, v[t][c]) : twmul<INV>(csub(o, v[t][c]), w))
                                    : cadd(v[t][c], o);
                }
        }
    }
    __syncwarp();
    int h = 0;
#pragma unroll
    for (int i = 0; i < lgB; ++i) h |= ((b >> i) & 1) << (lgB - 1 - i);
#pragma unroll
    for (int t = 0; t < NB; ++t)
#pragma unroll
        for (int c = 0; c < N1; ++c) buf[t * N + k1 + N1 * c + N1 * N1 * h] = v[t][c];
    __syncwarp();
}

// Single transform (nf = 1).
template <bool INV, int NC = 0>
__device__ float2* fft_stockham(float2* a, float2* b, int N, const float2* __restrict__ tw, bool prune, int tid,
                                int nthreads) {
    return fft_batch<INV, NC>(a, b, N, 1, tw, prune, tid, nthreads);
}

// Untangle bin k (0 <= k <= N) of the real 2N-point transform from the
// half-length complex spectrum Z (spectral.cpp:113-120):
//   X_k = E_k + pack_k * O_k,  E = (Z_k + conj Z_{N-k})/2,  O = -i (Z_k - conj Z_{N-k})/2.
__device__ __forceinline__ float2 untangle(const float2* Z, int N, int k, const float2* __restrict__ pk) {
    const float2 zk = Z[k & (N - 1)];
    const float2 zm = Z[(N - k) & (N - 1)];
    const float2 even = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
    // odd = -0.5 i (zk - conj zm) = 0.5 * ((zk.y + zm.y), -(zk.x - zm.x))
    const float2 odd = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
    return cadd(even, cmul(pk[k], odd));
}

// Packed form used everywhere on the device: bin 0 carries (Re X_0, Re X_N)
// (both purely real, spectral.cpp:121-123), bins 1..N-1 are X_k.
__device__ __forceinline__ float2 untangle_packed(const float2* Z, int N, int k, const float2* __restrict__ pk) {
    if (k == 0) {
        const float2 z0 = Z[0];
        return make_float2(z0.x + z0.y, z0.x - z0.y);
    }
    return untangle(Z, N, k, pk);
}

// Untangle a whole packed spectrum into dst[0..N) (16-byte aligned): two bins per thread and
// one 16-byte store, no per-element address arithmetic beyond the bin index.
template <int NC = 0>
__device__ __forceinline__ void untangle_store(const float2* Z, int N, const float2* __restrict__ pk,
                                               float2* __restrict__ dst, int tid, int nthreads) {
    if constexpr (NC != 0) N = NC;
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (int k2 = tid; k2 < N / 2; k2 += nthreads) {
        const float2 a = untangle_packed(Z, N, 2 * k2, pk);
        const float2 b = untangle(Z, N, 2 * k2 + 1, pk);
        d4[k2] = make_float4(a.x, a.y, b.x, b.y);
    }
}

// One warp untangles a whole packed spectrum into dst[0 .. N) by bin pairs (k, N - k): both bins
// come from the same (Z_k, Z_{N-k}), and since pack_{N-k} = -conj(pack_k),
// X_{N-k} = conj(E_k - pack_k O_k) — half the loads and flops of untangling every bin alone.
// Used by the K4 warp transforms (side, in-stream, fused and in-kernel — all identical).
__device__ __forceinline__ void untangle_pairs_warp(const float2* Z, int N, const float2* __restrict__ pk,
                                                    float2* __restrict__ dst, int lane) {
    for (int k = lane; k <= N / 2; k += 32) {
        if (k == 0) {
            const float2 z0 = Z[0];
            dst[0] = make_float2(z0.x + z0.y, z0.x - z0.y);
            continue;
        }
        const float2 zk = Z[k], zm = Z[N - k];
        const float2 even = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
        const float2 odd = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
        const float2 po = cmul(pk[k], odd);
        dst[k] = cadd(even, po);
        if (k != N / 2) dst[N - k] = make_float2(even.x - po.x, -(even.y - po.y));
    }
}

// untangle_pairs_warp over the warp's own buffer (Z == dst): a lane reads both bins of its pair
// (k, N - k) before writing them, and pairs are disjoint across lanes. Same operations.
__device__ __forceinline__ void untangle_pairs_inplace_warp(float2* Z, int N, const float2* __restrict__ pk,
                                                            int lane) {
    for (int k = lane; k <= N / 2; k += 32) {
        if (k == 0) {
            const float2 z0 = Z[0];
            Z[0] = make_float2(z0.x + z0.y, z0.x - z0.y);
            continue;
        }
        const float2 zk = Z[k], zm = Z[N - k];
        const float2 even = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
        const float2 odd = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
        const float2 po = cmul(pk[k], odd);
        Z[k] = cadd(even, po);
        if (k != N / 2) Z[N - k] = make_float2(even.x - po.x, -(even.y - po.y));
    }
    __syncwarp();
}

// Tangle bin k < N for the inverse (spectral.cpp:142-148), from a packed
// spectrum Y:  z_k = E + i O,  E = (X_k + conj X_{N-k})/2,
// O = (X_k - conj X_{N-k})/2 * conj(pack_k).
__device__ __forceinline__ float2 tangle_packed(const float2* Y, int N, int k, const float2* __restrict__ pk) {
    float2 xk, xm;  // xm = conj(X_{N-k})
    if (k == 0) {
        xk = make_float2(Y[0].x, 0.f);
        xm = make_float2(Y[0].y, 0.f);
    } else {
        xk = Y[k];
        const float2 t = Y[N - k];
        xm = make_float2(t.x, -t.y);
    }
    const float2 even = make_float2(0.5f * (xk.x + xm.x), 0.5f * (xk.y + xm.y));
    const float2 odd = cmulc(make_float2(0.5f * (xk.x - xm.x), 0.5f * (xk.y - xm.y)), pk[k]);
    return make_float2(even.x - odd.y, even.y + odd.x);
}

}  // namespace tvb
