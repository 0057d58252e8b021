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

namespace tvb {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
    return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }

// Stockham FFT of N complex points (N a power of two >= 2) held in `a`,
// using `b` as the ping-pong buffer. tw[t] = e^{-2 pi i t / N}, t < N.
// INV selects the conjugate-twiddle (unscaled) inverse. When `prune` is set the
// input's upper half a[N/2..N) is taken as zero and never read (the engine's
// 4L block is zero-padded past 2L, proj/src/engine.cpp:77-80). All threads of
// the CTA must call this (it contains __syncthreads); returns the buffer that
// holds the result in natural order.
template <bool INV>
__device__ float2* fft_stockham(float2* a, float2* b, int N, const float2* __restrict__ tw, bool prune, int tid,
                                int nthreads) {
    float2* src = a;
    float2* dst = b;
    for (int Ns = 1; Ns < N;) {
        const int R = ((N / Ns) & 3) == 0 ? 4 : 2;
        const int nb = N / R;       // butterflies this stage
        const int stride = nb;      // input stride between the R legs
        const int tstep = N / (Ns * R);
        const bool zero_hi = prune && Ns == 1;
        for (int j = tid; j < nb; j += nthreads) {
            const int k = j & (Ns - 1);
            const int idxD = (j - k) * R + k;
            if (R == 4) {
                float2 v0 = src[j];
                float2 v1 = src[j + stride];
                float2 v2 = zero_hi ? make_float2(0.f, 0.f) : src[j + 2 * stride];
                float2 v3 = zero_hi ? make_float2(0.f, 0.f) : src[j + 3 * stride];
                if (Ns > 1) {
                    const int t1 = k * tstep;
                    const float2 w1 = tw[t1], w2 = tw[2 * t1], w3 = tw[3 * t1];
                    if (INV) {
                        v1 = cmulc(v1, w1);
                        v2 = cmulc(v2, w2);
                        v3 = cmulc(v3, w3);
                    } else {
                        v1 = cmul(v1, w1);
                        v2 = cmul(v2, w2);
                        v3 = cmul(v3, w3);
                    }
                }
                const float2 a0 = cadd(v0, v2), a1 = csub(v0, v2);
                const float2 a2 = cadd(v1, v3), a3 = csub(v1, v3);
                dst[idxD] = cadd(a0, a2);
                dst[idxD + 2 * Ns] = csub(a0, a2);
                if (INV) {  // y1 = a1 + i a3, y3 = a1 - i a3
                    dst[idxD + Ns] = make_float2(a1.x - a3.y, a1.y + a3.x);
                    dst[idxD + 3 * Ns] = make_float2(a1.x + a3.y, a1.y - a3.x);
                } else {    // y1 = a1 - i a3, y3 = a1 + i a3
                    dst[idxD + Ns] = make_float2(a1.x + a3.y, a1.y - a3.x);
                    dst[idxD + 3 * Ns] = make_float2(a1.x - a3.y, a1.y + a3.x);
                }
            } else {
                float2 v0 = src[j];
                float2 v1 = zero_hi ? make_float2(0.f, 0.f) : src[j + stride];
                if (Ns > 1) {
                    const float2 w1 = tw[k * tstep];
                    v1 = INV ? cmulc(v1, w1) : cmul(v1, w1);
                }
                dst[idxD] = cadd(v0, v1);
                dst[idxD + Ns] = csub(v0, v1);
            }
        }
        __syncthreads();
        float2* t = src;
        src = dst;
        dst = t;
        Ns *= R;
    }
    return src;
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
