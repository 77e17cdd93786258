// 3D instantiations of the fused operator kernels (see op_kernels.cuh).
#include "op_launch.cuh"

namespace pffmg {

constexpr int TY3D = 8;

template <int MODE, int EPI, bool ISO>
static void set_smem(size_t smem) {
    static size_t done = 0;
    if (done < smem) {
        cudaFuncSetAttribute(op3d_kernel<MODE, EPI, TY3D, ISO>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        done = smem;
    }
}

template <int MODE, int EPI>
int launch3d(const OpArgs& A0, bool iso, cudaStream_t s) {
    OpArgs A = A0;
    const Lat& L = A.L;
    const int sms = sm_count();
    using MI = ModeInfo<3, MODE>;
    constexpr int TV = 33 * (TY3D + 1);
    const size_t smem = sizeof(double) * (2 * MI::NF * TV + TY3D * 2 * MI::NCO * 32) + 2 * TV;
    const int gx = (L.nx + 1 + 30) / 31;
    const int gy = (L.ny + 1 + TY3D - 2) / (TY3D - 1);
    const int planes = L.nz + 1;
    int per = (int)(((int64_t)planes * gx * gy + 2LL * sms - 1) / (2LL * sms));
    per = per < 4 ? 4 : (per > 32 ? 32 : per);
    A.planes_per_cta = per;
    dim3 grid(gx, gy, (planes + per - 1) / per);
    if (iso) {
        set_smem<MODE, EPI, true>(smem);
        op3d_kernel<MODE, EPI, TY3D, true><<<grid, 32 * TY3D, smem, s>>>(A);
    } else {
        set_smem<MODE, EPI, false>(smem);
        op3d_kernel<MODE, EPI, TY3D, false><<<grid, 32 * TY3D, smem, s>>>(A);
    }
    return PFFMG_OK;
}

PFFMG_INSTANTIATE_LAUNCH(launch3d)

}  // namespace pffmg
