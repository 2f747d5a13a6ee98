// common.cuh — shared device/host definitions for the sm_100a 3DGS² Newton path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>

#include "ngs_b200.h"

namespace ngsb {

constexpr int kTile = 16;                 // rasterizer.hpp:18 kTileSize
constexpr int kTilePixels = kTile * kTile;
constexpr double kNearPlaneEps = 1e-6;    // camera.hpp:11
constexpr double kSigmaMargin = 1e-4;     // scene.hpp:10
constexpr double kColorOffset = 0.5;      // sh.hpp:21
// Largest (tile, splat) pair count of one view: the onesweep look-back packs running
// counts into 30 bits (sort.cu kCountMask) and offsets are int.
constexpr int kMaxPairs = (1 << 30) - 1;
// Device error-flag bits (ngs_context::check_err maps them onto status codes).
constexpr int kErrNonPD = 1, kErrDegenerate = 2, kErrQuat = 4, kErrPairLimit = 8, kErrFixedRange = 16;

// Error carrying an ngs_status; thrown by host code, mapped at the C-ABI edge.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        throw Error(NGS_ERR_CUDA, std::string(what) + " failed at " + file + ":" + std::to_string(line) +
                                      ": " + cudaGetErrorString(e));
    }
}
#define CUDA_CHECK(x) ::ngsb::cuda_check((x), #x, __FILE__, __LINE__)
#define CUDA_LAUNCH_CHECK() ::ngsb::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// Opt a kernel into at least `bytes` of dynamic shared memory on the current device. Function
// attributes are per device, so the high-water mark is kept per (kernel, device).
inline void ensure_dynamic_smem(const void* kernel, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> granted;
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice", __FILE__, __LINE__);
    std::lock_guard<std::mutex> lock(mu);
    size_t& g = granted[{kernel, dev}];
    if (bytes > g) {
        cuda_check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)),
                   "cudaFuncSetAttribute", __FILE__, __LINE__);
        g = bytes;
    }
}

// Camera constants uploaded per view (camera.hpp:17-45), FP64.
struct CameraDev {
    double view[16];       // row-major world->camera
    double proj[16];       // row-major camera->clip
    double view_proj[16];  // proj * view
    double center[3];      // camera position in world space
    int width, height;
    int tile;              // tile edge in pixels (16, or 8 for small views; binning result identical)
    int tiles_x, tiles_y;
};

// Device-side scene, FP32 SoA.
struct SceneDev {
    int n;
    int sh_degree;
    int n_coeffs;          // (deg+1)^2
    float bg[3];
    float4* pos_sigma;     // x, y, z, sigma
    float4* scale;         // sx, sy, sz, 0
    float4* quat;          // w, x, y, z
    float* sh;             // [48][n] coefficient-major: sh[(16*ch + i)*n + k]
};

// Projected record of one kernel in one view (forward-pass payload), 48 B.
//   a = (pixel.x, pixel.y, Q00, Q01), b = (Q11, sigma, c0, c1), c = (c2, cov00, cov01, cov11)
struct ViewRecordsDev {
    float4* a;
    float4* b;
    float4* c;
    double* depth;         // camera-space depth (FP64, sort key source)
    int4* rect;            // tile rect [tx0, ty0, tx1, ty1] inclusive; tx0 > tx1 => not binned
    int* tiles_touched;
    uint8_t* flags;        // bit0 projected (entry exists), bits1-3 channel clamped
};

enum RecordFlag : uint8_t { kProjected = 1, kClamp0 = 2, kClamp1 = 4, kClamp2 = 8 };

// ---- order-independent scalar sums -------------------------------------------
// Report scalars (loss sums, delta norms) are summed from per-block partials. With
// FP64 atomics the result depends on block order; instead every partial is added
// exactly into a 128-bit two's-complement fixed-point number (binary point 2^-88,
// four 32-bit chunks in 64-bit counters: integer atomics are associative), so the
// same partials give bitwise the same sum in any order. Word 4 flags a non-finite or
// out-of-range (|x| >= 2^38) partial: the sum then reads as NaN (the trainer's
// "non-finite update" abort, trainer.hpp:200-205).
constexpr int kExactWords = 5;
constexpr int kExactShift = 88;

__device__ __forceinline__ void exact_add(unsigned long long* w, double x) {
    if (x == 0.0) return;
    if (!(fabs(x) < 0x1p38)) {
        atomicOr(w + 4, 1ull);
        return;
    }
    int e;
    const double m = frexp(x, &e);                                  // |m| in [0.5, 1)
    const long long mi = static_cast<long long>(ldexp(m, 53));       // exact
    const int sh = e - 53 + kExactShift;                            // <= 73
    __int128 v = static_cast<__int128>(mi);
    v = sh >= 0 ? (v << sh) : (sh > -127 ? (v >> (-sh)) : (mi < 0 ? -1 : 0));  // truncation below 2^-88
    const unsigned __int128 u = static_cast<unsigned __int128>(v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const unsigned long long chunk = static_cast<unsigned long long>((u >> (32 * i)) & 0xffffffffull);
        if (chunk) atomicAdd(w + i, chunk);
    }
}

// Host: the exact sum rounded once to FP64 (NaN if flagged).
inline double exact_value(const unsigned long long* w) {
    if (w[4]) return __builtin_nan("");
    unsigned __int128 u = 0;
    for (int q = 0; q < 4; ++q) u += static_cast<unsigned __int128>(w[q]) << (32 * q);
    const bool neg = static_cast<__int128>(u) < 0;
    if (neg) u = ~u + 1;
    // long double keeps 64 significant bits: one rounding to it, then to double, is exact
    // enough for a report scalar (the same bits on every run either way).
    const long double mag = static_cast<long double>(u) * 0x1p-88L;
    return static_cast<double>(neg ? -mag : mag);
}

// ---- small device math -----------------------------------------------------

__host__ __device__ inline double mrow(const double* m, int r, int c) { return m[4 * r + c]; }

}  // namespace ngsb
