// kohler_luma.cuh — colour ingest (luma_kernel).
// Part of the single translation unit kohler_kernels.cu (included there,
// in this order, after the shared constants and parameter blocks).
#pragma once

namespace {

// ---------------------------------------------------------------------------
// Colour ingest: Rec. 601 integer luma of interleaved
// RGB, exactly the reference's luma601 (proj/src/pnm.cpp:63-68), used by
// read_pnm for P6/P3 input (:110-136):
//     v = min((299 r + 587 g + 114 b + 500) / 1000, 255)
// HBM-bound (3 B read + 1 B written per pixel).  One thread converts 16
// pixels: three 16-byte loads, the weighted sums by two DP2A per pixel
// (16-bit weights x 8-bit samples, FMA pipe), the division by 1000 as one
// IMAD.HI with ceil(2^32 / 1000) (exact for t < 2^18: 704 t < 2^32), one
// 16-byte store.  Ragged row ends / unaligned buffers take a per-pixel loop.
// ---------------------------------------------------------------------------
struct LumaParams {
    const uint8_t* rgb;
    size_t rpitch, rstride;   // bytes between rows / images of the RGB input
    uint8_t* gray;
    size_t gpitch, gstride;
    int w, rows, n;
    int vec;                  // all bases / pitches / strides 16-byte aligned
    long long items;          // n * rows * ceil(w / 16)
    int nchunk;
};

constexpr uint32_t kLumaMagic = 4294968u;  // ceil(2^32 / 1000)

__device__ __forceinline__ uint32_t luma_div(uint32_t t) { return __umulhi(t, kLumaMagic); }

__device__ __forceinline__ uint32_t luma1(uint32_t r, uint32_t g, uint32_t b)
{
    return luma_div(299u * r + 587u * g + 114u * b + 500u);
}

// four pixels from three words r0 g0 b0 r1 | g1 b1 r2 g2 | b2 r3 g3 b3 -> packed bytes
__device__ __forceinline__ uint32_t luma4(uint32_t w0, uint32_t w1, uint32_t w2)
{
    constexpr uint32_t A = 299u | 587u << 16, B = 114u, C = 299u << 16, D = 587u | 114u << 16;
    const uint32_t p0 = luma_div(__dp2a_hi(B, w0, __dp2a_lo(A, w0, 500u)));
    const uint32_t p1 = luma_div(__dp2a_lo(D, w1, __dp2a_hi(C, w0, 500u)));
    const uint32_t p2 = luma_div(__dp2a_lo(B, w2, __dp2a_hi(A, w1, 500u)));
    const uint32_t p3 = luma_div(__dp2a_hi(D, w2, __dp2a_lo(C, w2, 500u)));
    return __byte_perm(p0 | p1 << 8, p2 | p3 << 8, 0x5410);
}

__global__ void __launch_bounds__(256) luma_kernel(const LumaParams p)
{
    for (long long it = (long long)blockIdx.x * blockDim.x + threadIdx.x; it < p.items;
         it += (long long)gridDim.x * blockDim.x) {
        const long long rowi = it / p.nchunk;
        const int c = (int)(it - rowi * p.nchunk);
        const int img = (int)(rowi / p.rows), y = (int)(rowi - (long long)img * p.rows);
        const uint8_t* src = p.rgb + (size_t)img * p.rstride + (size_t)y * p.rpitch + (size_t)c * 48;
        uint8_t* dst = p.gray + (size_t)img * p.gstride + (size_t)y * p.gpitch + (size_t)c * 16;
        const int x0 = c * 16;
        if (p.vec && x0 + 16 <= p.w) {
            const uint4 a = __ldg(reinterpret_cast<const uint4*>(src));
            const uint4 b = __ldg(reinterpret_cast<const uint4*>(src) + 1);
            const uint4 d = __ldg(reinterpret_cast<const uint4*>(src) + 2);
            uint4 o;
            o.x = luma4(a.x, a.y, a.z);
            o.y = luma4(a.w, b.x, b.y);
            o.z = luma4(b.z, b.w, d.x);
            o.w = luma4(d.y, d.z, d.w);
            *reinterpret_cast<uint4*>(dst) = o;
        } else {
            const int e = min(16, p.w - x0);
            for (int i = 0; i < e; ++i)
                dst[i] = (uint8_t)luma1(src[3 * i], src[3 * i + 1], src[3 * i + 2]);
        }
    }
}

} // namespace
