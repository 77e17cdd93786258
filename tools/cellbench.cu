// Compute-only throughput of the per-cell kernels (no global memory in the
// loop): separates the FP64/issue cost of cell_kernel_iso from staging and
// memory latency.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I../paper_1902_08112_b200/csrc -o cellbench cellbench.cu ../paper_1902_08112_b200/csrc/capi.cu
#include <cstdio>

#include "cell3_iso.cuh"

using namespace pffmg;

template <int D, int MODE>
__global__ void __launch_bounds__(128) bench(Consts K, IsoK I, int iters, double* out) {
    using MI = ModeInfo<D, MODE>;
    constexpr int NP = 1 << D;
    double cv[MI::NF][NP];
#pragma unroll
    for (int i = 0; i < MI::NF; ++i)
#pragma unroll
        for (int n = 0; n < NP; ++n) cv[i][n] = 1e-3 * (threadIdx.x + 3 * i + n) + (i == MI::F_PT ? 0.5 : 0.0);
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
        double o[MI::NCO][NP];
        cell_kernel_iso<D, MODE, false>(cv, nullptr, K, I, o);
#pragma unroll
        for (int k = 0; k < MI::NCO; ++k)
#pragma unroll
            for (int n = 0; n < NP; ++n) acc += o[k][n];
        const double eps = 1e-30 * acc;   // loop-carried dependency on every input
#pragma unroll
        for (int i = 0; i < MI::NF; ++i)
#pragma unroll
            for (int n = 0; n < NP; ++n) cv[i][n] += eps;
    }
    if (acc == 1234.5) out[0] = acc;
}

template <int MODE>
__global__ void __launch_bounds__(64) bench3(Consts K, IsoK I, int iters, double* out) {
    using MI = ModeInfo<3, MODE>;
    __shared__ double sm[MI::NF][8][64];
    for (int i = 0; i < MI::NF; ++i)
        for (int n = 0; n < 8; ++n) sm[i][n][threadIdx.x] = 1e-3 * (threadIdx.x + 3 * i + n) + (i == MI::F_PT ? 0.5 : 0.0);
    struct Cn {
        double (*sm)[8][64];
        double eps;
        __device__ void load(int f, double (&c)[8]) const {
            for (int n = 0; n < 8; ++n) c[n] = sm[f][n][threadIdx.x] + eps;
        }
    };
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
        Cn C{sm, 1e-30 * acc};
        cell3_iso<MODE, false>(C, nullptr, K, I, [&](int k, double (&o)[8]) {
#pragma unroll
            for (int n = 0; n < 8; ++n) acc += o[n];
        });
    }
    if (acc == 1234.5) out[0] = acc;
}

template <int MODE>
void run3(const char* name, Consts K, IsoK I, double* d) {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int blocks = sms * 8, iters = 100;
    bench3<MODE><<<blocks, 64>>>(K, I, 2, d);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    bench3<MODE><<<blocks, 64>>>(K, I, iters, d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double cells = (double)blocks * 64 * iters;
    printf("%s: %.1f Gcell/s  -> 1.08M cells in %.1f us\n", name, cells / ms * 1e-6, 1.08e6 / (cells / ms * 1e-3));
}

template <int D, int MODE>
void run(const char* name, Consts K, IsoK I, double* d) {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int blocks = sms * 6, iters = 200;
    bench<D, MODE><<<blocks, 128>>>(K, I, 2, d);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    bench<D, MODE><<<blocks, 128>>>(K, I, iters, d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double cells = (double)blocks * 128 * iters;
    printf("%s: %.1f Gcell/s  -> 1.08M cells in %.1f us\n", name, cells / ms * 1e-6, 1.08e6 / (cells / ms * 1e-3));
}

int main() {
    pffmg_lattice lat{};
    lat.dim = 2; lat.nx = 1024; lat.ny = 1024; lat.hx = lat.hy = 1.0 / 1024; lat.n_vertices = 1025 * 1025;
    pffmg_state st{};
    st.mu = 80.77; st.lam = 121.15; st.g_c = 2.7e-3; st.kappa = 1e-8; st.eps = 2.0 / 1024;
    Consts K;
    make_consts(&lat, &st, &K);
    IsoK I = make_iso_host(K);
    double* d;
    cudaMalloc(&d, 8);
    run<2, M_FULL>("2D full", K, I, d);
    run<2, M_UBLK>("2D ublk", K, I, d);
    run<2, M_PBLK>("2D pblk", K, I, d);
    lat.dim = 3; lat.nz = 384; lat.hz = lat.hx;
    make_consts(&lat, &st, &K);
    I = make_iso_host(K);
    run<3, M_FULL>("3D full", K, I, d);
    run<3, M_UBLK>("3D ublk", K, I, d);
    run<3, M_PBLK>("3D pblk", K, I, d);
    run3<M_FULL>("3D stream full", K, I, d);
    run3<M_UBLK>("3D stream ublk", K, I, d);
    run3<M_PBLK>("3D stream pblk", K, I, d);
    return 0;
}
