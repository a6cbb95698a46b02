// Single-image super-resolution with MCI:
// "Our SISR algorithm is based on Example 2 [channels f, f', f''].  We first compute
// interpolation result for each row of image, and then apply interpolation for each
// column by using the same operations.  The derivatives of image are computed by
// three-point centered-difference formula."
//
// Per chunk of images (all kernels here are elementwise / transposes; the two MCI
// passes run on the 1D kernels through launch_axis):
//   1. fd_rows: LR [n][H][W] -> row channels [n H][3][W]: f, f', f'' along x on the periodic
//      grid t = 2 pi x / W, f' = (f[x+1] - f[x-1]) / (2 d), f'' = (f[x+1] - 2 f[x] + f[x-1]) / d^2,
//      d = 2 pi / W;
//   2. MCI along x (M = 3, N = W, L = s W, bank (1, ik, -k^2)) -> I [n][H][sW] (real part);
//   3. fd_cols: I -> column channels [n][3][H][sW] (the same differences along y, d = 2 pi / H);
//   4. MCI along y, reading the strided columns (RowAddr) -> O^T [n][sW][sH];
//   5. transpose -> HR [n][sH][sW].
#include <cstdint>

#include "mci_internal.h"

namespace mci {

namespace sisrk {
constexpr double TWO_PI = 6.283185307179586476925286766559;
}

// x [lines][n] (contiguous lines) -> ch [lines][3][n]
template <typename T>
__global__ void mci_sisr_fd_rows(const T *__restrict__ x, T *__restrict__ ch, int64_t lines, int n, T c1, T c2) {
    const int64_t total = lines * n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t l = i / n;
        const int k = (int)(i - l * n);
        const T *row = x + l * n;
        const T fm = row[k == 0 ? n - 1 : k - 1], f0 = row[k], fp = row[k == n - 1 ? 0 : k + 1];
        T *o = ch + l * 3 * (int64_t)n + k;
        o[0] = f0;
        o[n] = (fp - fm) * c1;                 // 1 / (2 d)
        o[2 * (int64_t)n] = (fp - f0 - f0 + fm) * c2;  // 1 / d^2
    }
}

// I [img][H][C] -> ch [img][3][H][C]: differences along y (periodic in H)
template <typename T>
__global__ void mci_sisr_fd_cols(const T *__restrict__ I, T *__restrict__ ch, int64_t imgs, int H, int C, T c1, T c2) {
    const int64_t plane = (int64_t)H * C, total = imgs * plane;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t img = i / plane;
        const int64_t rem = i - img * plane;
        const int y = (int)(rem / C), c = (int)(rem - (int64_t)y * C);
        const T *p = I + img * plane;
        const T fm = p[(int64_t)(y == 0 ? H - 1 : y - 1) * C + c], f0 = p[rem],
                fp = p[(int64_t)(y == H - 1 ? 0 : y + 1) * C + c];
        T *o = ch + img * 3 * plane + rem;
        o[0] = f0;
        o[plane] = (fp - fm) * c1;
        o[2 * plane] = (fp - f0 - f0 + fm) * c2;
    }
}

// a [img][R][C] -> b [img][C][R] through 32 x 32 shared tiles
template <typename T>
__global__ void mci_sisr_transpose(const T *__restrict__ a, T *__restrict__ b, int R, int C) {
    __shared__ T tile[32][33];
    const int64_t img = blockIdx.z;
    const T *ai = a + img * (int64_t)R * C;
    T *bi = b + img * (int64_t)R * C;
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int r = r0 + dy, c = c0 + threadIdx.x;
        if (r < R && c < C) tile[dy][threadIdx.x] = ai[(int64_t)r * C + c];
    }
    __syncthreads();
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int c = c0 + dy, r = r0 + threadIdx.x;
        if (r < R && c < C) bi[(int64_t)c * R + r] = tile[threadIdx.x][dy];
    }
}

template <typename T>
static cudaError_t sisr_chunk_t(const Axis1D &ax, const Axis1D &ay, int64_t ni, int H, int W, int s, const T *lr, T *hr,
                                T *ws, cudaStream_t st, int *nl) {
    using namespace sisrk;
    const int sW = s * W, sH = s * H;
    T *chr = ws;                                  // [ni H][3][W]
    T *inter = chr + ni * (int64_t)H * 3 * W;     // [ni][H][sW]
    T *chc = inter + ni * (int64_t)H * sW;        // [ni][3][H][sW]
    T *outT = chc + ni * 3 * (int64_t)H * sW;     // [ni][sW][sH]
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const unsigned eg = (unsigned)(nsm * 8);
    const T dx = (T)(TWO_PI / W), dy = (T)(TWO_PI / H);
    mci_sisr_fd_rows<T><<<eg, 256, 0, st>>>(lr, chr, ni * H, W, (T)0.5 / dx, (T)1 / (dx * dx));
    RowAddr rr;  // row pass: contiguous lines [ni H][3][W]
    rr.s2 = 3 * (int64_t)W;
    rr.cs = W;
    rr.ss = 1;
    cudaError_t e = launch_axis(ax, rr, ni * H, chr, inter, nullptr, st, nl);
    if (e != cudaSuccess) return e;
    mci_sisr_fd_cols<T><<<eg, 256, 0, st>>>(inter, chc, ni, H, sW, (T)0.5 / dy, (T)1 / (dy * dy));
    RowAddr rc;  // column pass: line (img, col), samples strided by sW, channels by H sW
    rc.D0 = sW;
    rc.D1 = 1;
    rc.s0 = 1;
    rc.s2 = 3 * (int64_t)H * sW;
    rc.cs = (int64_t)H * sW;
    rc.ss = sW;
    e = launch_axis(ay, rc, ni * sW, chc, outT, nullptr, st, nl);
    if (e != cudaSuccess) return e;
    dim3 tg((sH + 31) / 32, (sW + 31) / 32, (unsigned)ni);
    mci_sisr_transpose<T><<<tg, dim3(32, 8), 0, st>>>(outT, hr, sW, sH);
    if (nl) *nl += 3;
    return cudaGetLastError();
}

size_t sisr_ws_per_image(int H, int W, int s, int dtype) {
    const size_t es = dtype == MCI_F64 ? 8 : 4;
    return ((size_t)H * 3 * W + (size_t)H * s * W + 3 * (size_t)H * s * W + (size_t)s * W * s * H) * es;
}

cudaError_t launch_sisr_chunk(const Axis1D &ax, const Axis1D &ay, int64_t ni, int H, int W, int s, const void *lr,
                              void *hr, void *ws, cudaStream_t st, int *nl) {
    if (ni <= 0) return cudaSuccess;
    return ax.dtype == MCI_F64
               ? sisr_chunk_t<double>(ax, ay, ni, H, W, s, (const double *)lr, (double *)hr, (double *)ws, st, nl)
               : sisr_chunk_t<float>(ax, ay, ni, H, W, s, (const float *)lr, (float *)hr, (float *)ws, st, nl);
}

}  // namespace mci
