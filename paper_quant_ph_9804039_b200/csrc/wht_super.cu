// wht_super.cu -- host side of the supertile pass (parameter packing, launch)
// and the ideal-stage instantiation; kernels in wht_super.cuh.
#include <cuda_runtime.h>

#include "wht_super.cuh"

namespace sv {

template void launch_super_uab<0>(int, int, const SuperParamsT<0> &, int, cudaStream_t);
extern template void launch_super_uab<1>(int, int, const SuperParamsT<1> &, int, cudaStream_t);
extern template void launch_super_uab<2>(int, int, const SuperParamsT<2> &, int, cudaStream_t);

int super_grid() {
    static int grid = 0;
    if (grid == 0) {
        int dev = 0, sms = 0, per = 0;
        SV_CUDA(cudaGetDevice(&dev));
        SV_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const int smem = (1 << kTileBitsC64) * (int)sizeof(float2);
        SV_CUDA(cudaFuncSetAttribute(wht_super_kernel<2, 5, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        SV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, wht_super_kernel<2, 5, 0>, 256, smem));
        grid = sms * (per > 0 ? per : 1);
    }
    return grid;
}

template <int NOISY>
static void fill(SuperParamsT<NOISY> &P, const KParams (&kp)[3], const KParamsT<1> (&kc)[3], const KParamsT<2> (&ka)[3]) {
    for (int j = 0; j < 3; ++j) {
        if constexpr (NOISY == 0) static_cast<KParams &>(P.sp[j]) = kp[j];
        else if constexpr (NOISY == 1) P.sp[j] = kc[j];
        else P.sp[j] = ka[j];
    }
}

void launch_wht_super_pass(sv_dtype dt, const SuperArgs &a, cudaStream_t s, TileVariant *describe) {
    SV_CHECK(dt == SV_C64, SV_EINVAL, "internal: supertile passes are complex64 only");
    SV_CHECK(super_pair_supported(a.ua, a.ub), SV_EINVAL, "internal: unsupported supertile level split");
    KParams kp[3];
    KParamsT<1> kc[3];
    KParamsT<2> ka[3];
    int fl[3], u[3];
    const int total_bits = a.sub[0].total_bits;
    for (int j = 0; j < 3; ++j) {
        const PassArgs &pa = a.sub[j];
        SV_CHECK(pa.scale_in == nullptr && pa.sumsq == nullptr && pa.xchg_nl == 0 && pa.mid != MID_ORACLE,
                 SV_EINVAL, "internal: the supertile pass carries F0 only");
        SV_CHECK((pa.tile_mask & ~a.st_mask) == 0, SV_EINVAL, "internal: sub-pass tile outside the supertile");
        unsigned long long nt = 0;
        fl[j] = pack_tile_params(dt, pa, true, kp[j], kc[j], ka[j], &u[j], &nt);
        // tile id within the supertile -> the supertile's slots outside this tile
        for (KParams *k : {&kp[j], static_cast<KParams *>(&kc[j]), static_cast<KParams *>(&ka[j])}) {
            k->free_mask = a.st_mask & ~pa.tile_mask;
            kp_set_free_runs(*k);
            SV_CHECK(k->nruns > 0 || k->free_mask == 0, SV_EINVAL, "internal: in-supertile slots in > 8 runs");
        }
    }
    SV_CHECK(u[0] == a.ua && u[2] == a.ua && u[1] == a.ub, SV_EINVAL, "internal: sub-pass tiles do not match the split");
    // one flavour for the whole pass: tan form only if every sub-pass qualifies
    const int flavour = (fl[0] == 0) ? 0 : ((fl[0] == 2 && fl[1] == 2 && fl[2] == 2) ? 2 : 1);
    if (describe) {
        for (int j = 0; j < 3; ++j) {
            describe[j].family = 3;
            describe[j].u = u[j];
            describe[j].pre = a.sub[j].pre;
            describe[j].mid = a.sub[j].mid;
            describe[j].post = a.sub[j].post;
            describe[j].noisy = flavour;
            describe[j].xchg = 0;
        }
        return;
    }
    // supertile index -> the slots outside the supertile (runs)
    KParams tmp{};
    tmp.free_mask = (total_bits >= 64 ? ~0ull : ((1ull << total_bits) - 1ull)) & ~a.st_mask;
    kp_set_free_runs(tmp);
    SV_CHECK(tmp.nruns > 0 || tmp.free_mask == 0, SV_EINVAL, "internal: supertile index slots in > 8 runs");
    const int stb = __builtin_popcountll(a.st_mask);
    const uint64_t nst = 1ull << (total_bits - stb);
    SV_CHECK(a.nseg == 3 * nst, SV_EINVAL, "internal: supertile segment table size");
    SV_CUDA(cudaMemsetAsync(a.ctr, 0, (size_t)(3 * nst + 1) * sizeof(unsigned int), s));
    auto common = [&](auto &P) {
        P.st_nruns = tmp.nruns;
        for (int r = 0; r < 8; ++r) {
            P.st_start[r] = tmp.run_start[r];
            P.st_len[r] = tmp.run_len[r];
        }
        P.seg = a.seg;
        P.tps_log2 = (unsigned int)(stb - kTileBitsC64);
        P.nitems = a.nseg << P.tps_log2;
        P.ticket = a.ctr;
        P.done = a.ctr + 1;
    };
    if (flavour == 0) {
        SuperParamsT<0> P{};
        fill(P, kp, kc, ka);
        common(P);
        launch_super_uab<0>(a.ua, a.ub, P, a.grid, s);
    } else if (flavour == 1) {
        SuperParamsT<1> P{};
        fill(P, kp, kc, ka);
        common(P);
        launch_super_uab<1>(a.ua, a.ub, P, a.grid, s);
    } else {
        SuperParamsT<2> P{};
        fill(P, kp, kc, ka);
        common(P);
        launch_super_uab<2>(a.ua, a.ub, P, a.grid, s);
    }
}

}  // namespace sv

#ifdef SV_SUPER_STATS
// measurement builds only (build.py -DSV_SUPER_STATS=1 --out=...): read and
// reset the supertile kernel's counters (ideal flavour).
extern "C" int sv_debug_super_stats(unsigned long long *out) {
    if (cudaMemcpyFromSymbol(out, sv::g_super_stats, sizeof(sv::g_super_stats)) != cudaSuccess) return -1;
    const unsigned long long z[8] = {};
    return cudaMemcpyToSymbol(sv::g_super_stats, z, sizeof(z)) == cudaSuccess ? 0 : -1;
}
#endif
