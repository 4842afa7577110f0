// sv_consts.h -- constants and enums shared by the host code, the nvcc-built
// kernels and the kernels compiled at run time by NVRTC (gate_jit.cpp): no
// includes, nothing host-only.
#pragma once

#ifdef __CUDACC_RTC__
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
#endif

#ifndef SV_TILE_BITS_C64
#define SV_TILE_BITS_C64 13
#endif
#ifndef SV_GATE_TILE_BITS_C64
#define SV_GATE_TILE_BITS_C64 13
#endif

namespace sv {

constexpr int kTileBitsC64 = SV_TILE_BITS_C64;  // 2^13 x 8 B = 64 KiB smem tile
constexpr int kRegBitsC64 = 5;     // 32 amplitudes per thread, 256 threads
constexpr int kTileBitsC128 = 12;  // 2^12 x 16 B = 64 KiB smem tile
constexpr int kRegBitsC128 = 4;    // 16 amplitudes per thread, 256 threads
// minimum unprocessed low slots kept in a strided tile: 2^c amplitudes = 64 B
// contiguous runs (c64: 8 x 8 B, c128: 4 x 16 B)
constexpr int kCarryC64 = 3;
constexpr int kCarryC128 = 2;
// gate-circuit tiles (gates.cu) may be smaller than the WHT tiles
constexpr int kGateTileBitsC64 = SV_GATE_TILE_BITS_C64;

enum MidOp { MID_NONE = 0, MID_ORACLE = 1, MID_F0 = 2 };

}  // namespace sv
