// Internal structures shared by the plan builder (mci_plan.cpp) and the CUDA
// launchers (*.cu).  Not part of the ABI.
#pragma once

#include <cstdint>
#include <cstddef>
#include <cuda_runtime.h>

#include "../../include/mci.h"

namespace mci {

// A built-in channel system for device-side multiplier evaluation (error analysis).
struct SysDev {
    int kind = 0, order = 0;
    double tau = 0.0;
};

// Radix plan of a mixed-radix transform (arbitrary-length path): n passes, radices r[].
struct AnyRadix {
    int n = 0;
    int r[24] = {0};
    int bp = 0, bM = 0;  // Bluestein radix (a prime > 16, 0 if none) and its power-of-two length M >= 2 bp - 1
    // device tables of the Bluestein pass: chirp c_j = e^{s pi i (j^2 mod 2p)/p} [bp],
    // H^ = FFT(conj c)/M [bM], roots e^{-2 pi i m/M} and e^{+2 pi i m/M} [bM each]
    const void *bc = nullptr, *bH = nullptr, *bwm = nullptr, *bwp = nullptr;
};

// Per-plan device tables for one 1D axis (fused or four-step path).
struct Axis1D {
    int M = 0;
    int64_t N = 0, L = 0, K = 0;  // K = M*N/2, band {-K .. K-1}
    int64_t S = 0, R = 0;         // inverse FFT length and decimation: L = R*S
    int analytic = 0;             // 1: produce f + i Hf (one-sided spectrum)
    int dtype = MCI_F32;
    // Device tables (element type = plan dtype, complex = 2 scalars):
    void *Qt = nullptr;   // [(N/2+1)][M][M] complex: Q_q[m][l] / N for class q (j_q = q - N*ceil)
    void *twF = nullptr;  // [TW] complex e^{-2 pi i m / TW}, TW = max(N, S, 1024)
    int64_t TW = 0;
    void *twLhi = nullptr;  // [L/LO] complex e^{+2 pi i (h*LO) / L}
    void *twLlo = nullptr;  // [LO]   complex e^{+2 pi i l / L}
    int64_t LO = 0;
    const void *rowtab = nullptr;  // tables of the specialised row kernel (mci_row.cu), or null
    int bank_deriv012 = 0;         // bank is exactly (1, ik, -k^2): closed-form inverse available
    int bank_deriv01 = 0;          // bank is exactly (1, ik): closed-form inverse available
    int bank_derivM = 0;           // bank is exactly (ik)^m, m = 0..M-1: Vandermonde closed form (mci_rowg.cu)
    int rowg = 0;                  // special == 1 served by the row-kernel family (mci_rowg.cu)
    int bank_delay_ti = 0;         // bank is e^{ik 2 pi m/(MN)}, m < M in {2, 4, 8}: time-interleaved sampling
                                   // (closed-form solve in mci_rowg.cu)
    int bank_delay_uniform = 0;    // bank is e^{ik 2 pi m/(MN)}, m < M = 4: H = W diag(e^{ij tau_m}) (closed form)
    int bank_unimodular = 0;       // every |b_m(k)| = 1 (identity / delay channels): equal channel energies,
                                   // the four-step path skips the channel-magnitude pre-pass (reading R14)
    int row_variant = 0;  // row kernel: 0 = 3 groups (default), 2 = 2 groups, 1 = 2 groups + 2-warp forward (MCI_ROW_VARIANT)
    int special = 0;  // 0 generic fused, 1 row kernel (mci_row.cu), 2 line kernel (mci_line.cu), 3 Hilbert (mci_hilbert.cu),
                      // 4 arbitrary lengths (mci_anylen.cu: Qt has all N classes, twF = e^{-2 pi i m/N} [N],
                      //   twLhi = e^{+2 pi i m/L} [L], band K1 = -floor(MN/2))
    int64_t K1 = 0;   // lowest band frequency (arbitrary-length path)
    int cplx = 0;     // complex f: complex channels in, T_N f out (arbitrary-length path, MCI_COMPLEX)
    SysDev sys[8];        // the bank (built-in kinds), for device-side b_m(k) (MCI_ANALYSIS)
    double omega_sum = 0;  // sum_m Omega_m, Omega_m = sup_{band} |r_m|^2 (Eq. errorestimate)
    AnyRadix radN, radL;
};

// Vector accesses of the specialised kernels (128-bit loads / TMA bulk copies / float2 and
// float4 stores) need 16-byte aligned row bases; misaligned buffers (an offset view of a
// tensor, a C caller's odd pointer) are routed to kernels that access elements one by one.
__host__ __device__ inline bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

enum Path { PATH_FUSED = 0, PATH_FOURSTEP = 1, PATH_2D = 2, PATH_SISR = 3 };

// Row addressing of the fused kernel: row r starts at
//   (r / (D0*D1)) * s2 + ((r / D0) % D1) * s1 + (r % D0) * s0
// channel m adds m*cs, sample n adds n*ss; output row r is at r*L.
struct RowAddr {
    int64_t D0 = 1, D1 = 1, s0 = 0, s1 = 0, s2 = 0, cs = 0, ss = 1;
};

// Launchers (mci_fused.cu / mci_fourstep.cu).  All async on `st`.
cudaError_t launch_fused(const Axis1D &ax, const RowAddr &ra, int64_t rows, const void *g, void *f,
                         void *hf, cudaStream_t st, int *n_launches);
size_t fused_smem_bytes(const Axis1D &ax);
bool fused_supported(const Axis1D &ax);

bool row_supported(const Axis1D &ax);
void *tensor_map_encoder();  // PFN_cuTensorMapEncodeTiled_v12000, or nullptr (mci_line.cu)
bool rowg_supported(const Axis1D &ax);
cudaError_t launch_rowg(const Axis1D &ax, int64_t rows, const void *g, void *f, cudaStream_t st, int *n_launches);
bool line_supported(const Axis1D &ax);
bool hilbert_supported(const Axis1D &ax);
cudaError_t launch_hilbert(const Axis1D &ax, int64_t rows, const void *g, void *f, void *hf, cudaStream_t st,
                           int *n_launches);
// tstore: 2D column pass whose output leaves transposed ([D1-block][L][D0] rows), see mci_line.cu
bool line_tstore_ok(const Axis1D &ax, const RowAddr &ra, int64_t lines, const void *g, const void *f);
cudaError_t launch_line(const Axis1D &ax, const RowAddr &ra, int64_t lines, const void *g, void *f, cudaStream_t st,
                        int *n_launches, bool tstore = false);
// dispatch a fused-path axis to its kernel (specialised when available)
cudaError_t launch_axis(const Axis1D &ax, const RowAddr &ra, int64_t rows, const void *g, void *f, void *hf,
                        cudaStream_t st, int *n_launches);
cudaError_t launch_row(const Axis1D &ax, const void *rowtab, int64_t rows, const void *g, void *f, cudaStream_t st,
                       int *n_launches);

bool anylen_supported(const Axis1D &ax);
size_t anylen_smem_bytes(const Axis1D &ax);
cudaError_t launch_anylen(const Axis1D &ax, const RowAddr &ra, int64_t rows, const void *g, void *f, void *hf,
                          cudaStream_t st, int *n_launches);
cudaError_t launch_anylen_residual(const Axis1D &ax, const RowAddr &ra, int64_t rows, const void *g, void *out,
                                   cudaStream_t st);
cudaError_t launch_averaged_error(const Axis1D &ax, int64_t batch, const void *spec, int64_t k_lo, int64_t n_freq,
                                  void *out, cudaStream_t st);
cudaError_t launch_anylen_offgrid(const Axis1D &ax, const RowAddr &ra, int64_t rows, const void *g, int64_t n_pts,
                                  const void *t, void *f, void *hf, cudaStream_t st);

size_t sisr_ws_per_image(int H, int W, int s, int dtype);
cudaError_t launch_sisr_chunk(const Axis1D &ax, const Axis1D &ay, int64_t ni, int H, int W, int s, const void *lr,
                              void *hr, void *ws, cudaStream_t st, int *nl);

cudaError_t launch_fourstep(const Axis1D &ax, int64_t batch, const void *g, void *f, void *ws,
                            int64_t ws_signals, cudaStream_t st, int *n_launches);
size_t fourstep_ws_bytes_per_signal(const Axis1D &ax);
bool fourstep_supported(const Axis1D &ax);

}  // namespace mci
