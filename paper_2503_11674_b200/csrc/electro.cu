// electro.cu — optional electrostatic density (ePlace-style, north_star (2)):
// the bin occupancy rho (the same B-spline rasterisation as the reference density) is treated as charge
// and the potential psi solves the grid's Neumann Poisson problem  L psi = rho - mean(rho),  L the
// 5-point Laplacian with spacings (bw, bh), in the cosine basis that diagonalises it:
//     psi = DCT-III_2D( DCT-II_2D(rho) / lambda ) / (nx ny),
//     lambda_uv = (2 - 2 cos(pi u / nx)) / bw^2 + (2 - 2 cos(pi v / ny)) / bh^2,   lambda_00 term dropped.
// The density energy is D = 1/2 sum_b rho_b psi_b, whose exact gradient is the footprint gather of psi
// (dD/dx_i = sum_b psi_b d rho_b / dx_i: L^+ is symmetric and sum_b psi_b = 0), so the existing
// density-gradient kernel is reused with field psi, scale 1.  Not in the reference (it replaced this
// with the bin-overflow penalty), hence no oracle: tests check the Poisson residual with an
// independent stencil, the gradient by finite differences and that placement spreads cells.
//
// The transforms are hand-written, one grid row per CTA, the row resident in shared memory:
//  * power-of-two lengths: DCT-II as Makhoul's (1980) FFT of the even/odd-reordered row plus a
//    quarter-wave twiddle, the real length-L FFT done as a half-length complex FFT and an untangling step;
//    DCT-III as the pre-twiddled Hermitian spectrum through the inverse; the FFT is a Stockham autosort
//    (natural order in and out) in shared memory, radix-4 stages then one radix-2 stage when needed,
//    twiddles from a per-length table;
//  * other lengths: the direct O(L^2) sums from a cosine table cos(pi j / 2L), j < 4L.
// Five launches per solve: DCT-II along y (rows of rho); tiled shared-memory transpose; one fused x pass
// per row (DCT-II, divide by lambda_uv, DCT-III — the whole x spectrum of a y frequency stays on chip);
// transpose back; DCT-III along y.  Stream-ordered and capturable into the iteration graph.  No
// FFT library (tensor cores would need the transform as a dense FP64 GEMM, 2 L^3 flops per pass —
// ~4 GFLOP at 1024^2 — far more than the FFT's ~50 MFLOP, so they do not pay here).
#include <algorithm>
#include <cmath>

#include "gp_kernels.cuh"

namespace tdpg {

namespace {

constexpr int kDctThreads = 256;

__device__ __forceinline__ double2 cmul(double2 a, double2 b)
{
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// W(m) = exp(-2 pi i m / L) from the half table tw[0 .. L/2) (W(m + L/2) = -W(m)); conj for the inverse
__device__ __forceinline__ double2 twiddle(const double2* tw, int m, int L, bool inverse)
{
    const int h = L >> 1;
    double2 w = m < h ? tw[m] : tw[m - h];
    if (m >= h) w.x = -w.x, w.y = -w.y;
    if (inverse) w.y = -w.y;
    return w;
}

// Stockham autosort FFT (natural order in and out) over shared memory, radix-4 stages then one radix-2
// stage when log2 L is odd; ping-pongs between x and y, returns the buffer holding the result.
// tw: the half twiddle table in shared memory.
__device__ double2* fft_stockham(double2* x, double2* y, int L, const double2* tw, bool inverse)
{
    int Ns = 1;
    for (; Ns * 4 <= L; Ns *= 4) {
        const int q = L >> 2;
        for (int j = threadIdx.x; j < q; j += blockDim.x) {
            const int k = j & (Ns - 1), m = k * (L / (Ns * 4));
            double2 a0 = x[j], a1 = x[j + q], a2 = x[j + 2 * q], a3 = x[j + 3 * q];
            if (Ns > 1) {
                a1 = cmul(a1, twiddle(tw, m, L, inverse));
                a2 = cmul(a2, twiddle(tw, 2 * m, L, inverse));
                a3 = cmul(a3, twiddle(tw, 3 * m, L, inverse));
            }
            const double2 s02 = make_double2(a0.x + a2.x, a0.y + a2.y), d02 = make_double2(a0.x - a2.x, a0.y - a2.y);
            const double2 s13 = make_double2(a1.x + a3.x, a1.y + a3.y), d13 = make_double2(a1.x - a3.x, a1.y - a3.y);
            // -i d13 (forward) or +i d13 (inverse)
            const double2 r13 = inverse ? make_double2(-d13.y, d13.x) : make_double2(d13.y, -d13.x);
            const int base = (j - k) * 4 + k;
            y[base] = make_double2(s02.x + s13.x, s02.y + s13.y);
            y[base + Ns] = make_double2(d02.x + r13.x, d02.y + r13.y);
            y[base + 2 * Ns] = make_double2(s02.x - s13.x, s02.y - s13.y);
            y[base + 3 * Ns] = make_double2(d02.x - r13.x, d02.y - r13.y);
        }
        __syncthreads();
        double2* t = x;
        x = y, y = t;
    }
    if (Ns * 2 == L) { // last radix-2 stage
        const int q = L >> 1;
        for (int j = threadIdx.x; j < q; j += blockDim.x) {
            const int k = j & (Ns - 1), m = k * (L / (Ns * 2));
            const double2 a0 = x[j], a1 = Ns > 1 ? cmul(x[j + q], twiddle(tw, m, L, inverse)) : x[j + q];
            const int base = (j - k) * 2 + k;
            y[base] = make_double2(a0.x + a1.x, a0.y + a1.y);
            y[base + Ns] = make_double2(a0.x - a1.x, a0.y - a1.y);
        }
        __syncthreads();
        x = y;
    }
    return x;
}

// row position m of the Makhoul reordering that element n of the row goes to (v[m] = x[src(m)])
__device__ __forceinline__ int makhoul_pos(int n, int L) { return (n & 1) ? L - 1 - (n >> 1) : (n >> 1); }

struct DctTables {
    const double2* tw; // [L/2] exp(-2 pi i j / L)          (power of two)
    const double2* qt; // [L]   exp(-i pi k / 2L)
    const double* c4;  // [4L]  cos(pi j / 2L)              (direct path)
    const double* lam; // [L]   2 - 2 cos(pi u / L)          (this axis' Laplacian eigenvalues / pitch^-2)
    const double* lam_y; //      the other axis' (x pass only)
};

// Power-of-two rows use the half-length real-FFT form: the reordered real row v (length L) is read as M
// = L/2 complex values z[m] = v[2m] + i v[2m+1] (the same doubles), one M-point FFT, then the split
//   V[k] = (Z[k] + conj Z[M-k]) / 2 - i W_L^k (Z[k] - conj Z[M-k]) / 2,   k = 0..M   (W_L = e^{-2 pi i / L});
// the inverse builds Z[k] = (V[k] + conj V[M-k]) + i W_L^-k (V[k] - conj V[M-k]) and one inverse M-point FFT
// gives v[2m] + i v[2m+1].  Shared memory: two complex rows of M and the M-point twiddles (M/2).
struct RowSmem {
    double2 *z0, *z1, *tw;
    int M;
};

__device__ __forceinline__ double2 wl(const double2* __restrict__ twL, int k, int M)
{   // W_L^k for k in [0, M], from the global half table (W_L^M = -1)
    return k < M ? __ldg(twL + k) : make_double2(-1.0, 0.0);
}

// X[k] = sum_n x[n] cos(pi k (2n + 1) / 2L) for the row `src` (global) into X (shared, L doubles, aliasing
// the work row that is free after the FFT — returned)
__device__ double* dct2_row(const double* __restrict__ src, int L, const DctTables& T, RowSmem& S, bool pow2,
                            double* rowbuf, double* Xdirect)
{
    if (pow2) {
        const int M = S.M;
        double* v = reinterpret_cast<double*>(S.z0);
        for (int n = threadIdx.x; n < L; n += blockDim.x) v[makhoul_pos(n, L)] = src[n];
        __syncthreads();
        const double2* Z = fft_stockham(S.z0, S.z1, M, S.tw, false);
        double* X = reinterpret_cast<double*>(Z == S.z0 ? S.z1 : S.z0);
        for (int k = threadIdx.x; k <= M; k += blockDim.x) {
            const double2 a = Z[k < M ? k : 0], bc = Z[k > 0 ? M - k : 0];
            const double2 b = make_double2(bc.x, -bc.y); // conj Z[M-k]
            const double2 s = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y + b.y));
            const double2 d = make_double2(0.5 * (a.x - b.x), 0.5 * (a.y - b.y));
            const double2 wd = cmul(wl(T.tw, k, M), d);
            const double2 V = make_double2(s.x + wd.y, s.y - wd.x); // s - i w d
            const double2 q = __ldg(T.qt + k);
            X[k] = V.x * q.x - V.y * q.y; // Re(q_k V)
            if (k > 0 && k < M) {
                const double2 q2 = __ldg(T.qt + (L - k));
                X[L - k] = V.x * q2.x + V.y * q2.y; // Re(q_{L-k} conj V)
            }
        }
        __syncthreads();
        return X;
    }
    for (int n = threadIdx.x; n < L; n += blockDim.x) rowbuf[n] = src[n];
    __syncthreads();
    for (int k = threadIdx.x; k < L; k += blockDim.x) {
        double acc = 0.0;
        const long long L4 = 4LL * L;
        long long j = k; // (2n + 1) k mod 4L, advanced by 2k per n
        for (int n = 0; n < L; ++n) {
            acc += rowbuf[n] * __ldg(T.c4 + j);
            j += 2LL * k;
            if (j >= L4) j -= L4;
        }
        Xdirect[k] = acc;
    }
    __syncthreads();
    return Xdirect;
}

// y[n] = X[0] + 2 sum_{k>=1} X[k] cos(pi k (2n + 1) / 2L) (= L x when X = DCT-II(x)); X (shared, real) is
// one of the work rows (power of two), result written to dst (global)
__device__ void dct3_row(double* X, int L, const DctTables& T, RowSmem& S, double* __restrict__ dst, bool pow2)
{
    if (pow2) {
        const int M = S.M;
        double2* zin = reinterpret_cast<double2*>(X) == S.z0 ? S.z1 : S.z0;
        double2* zout = reinterpret_cast<double2*>(X) == S.z0 ? S.z0 : S.z1;
        auto Vk = [&](int k) { // V[k] = e^{+i pi k / 2L} (X[k] - i X[L-k]), X[L] := 0
            const double2 q = __ldg(T.qt + k);
            const double a = X[k], b = k > 0 ? X[L - k] : 0.0;
            return make_double2(q.x * a - q.y * b, -q.y * a - q.x * b); // conj(q)(a - i b)
        };
        for (int k = threadIdx.x; k < M; k += blockDim.x) {
            const double2 a = Vk(k), bb = Vk(M - k);
            const double2 b = make_double2(bb.x, -bb.y); // conj V[M-k]
            const double2 s = make_double2(a.x + b.x, a.y + b.y), d = make_double2(a.x - b.x, a.y - b.y);
            double2 w = wl(T.tw, k, M);
            w.y = -w.y; // W_L^-k
            const double2 wd = cmul(w, d);
            zin[k] = make_double2(s.x - wd.y, s.y + wd.x); // s + i w d
        }
        __syncthreads();
        const double2* z = fft_stockham(zin, zout, M, S.tw, true);
        const double* v = reinterpret_cast<const double*>(z);
        for (int n = threadIdx.x; n < L; n += blockDim.x) dst[n] = v[makhoul_pos(n, L)];
        return;
    }
    for (int n = threadIdx.x; n < L; n += blockDim.x) {
        double acc = 0.0;
        const long long L4 = 4LL * L, step = 2LL * n + 1;
        long long j = step; // (2n + 1) k mod 4L for k = 1, 2, ...
        for (int k = 1; k < L; ++k) {
            acc += X[k] * __ldg(T.c4 + j);
            j += step;
            if (j >= L4) j -= L4;
        }
        dst[n] = X[0] + 2.0 * acc;
    }
}

// MODE 0: out = DCT-II(row); MODE 1: out = DCT-III(row); MODE 2 (x pass, rows are y frequencies v):
// out = DCT-III(DCT-II(row) / lambda_uv / (nx ny)), the (0, 0) term dropped.
template <int MODE>
__global__ void __launch_bounds__(kDctThreads) k_dct_rows(int L, bool pow2, const double* __restrict__ in,
                                                          double* __restrict__ out, DctTables T, int nx, int ny,
                                                          double ibw2, double ibh2)
{
    extern __shared__ double2 dsm[];
    RowSmem S;
    S.M = L / 2;
    S.z0 = dsm, S.z1 = dsm + S.M, S.tw = dsm + 2 * S.M; // (power of two: 2 M + M/2 complex)
    double* ra = reinterpret_cast<double*>(dsm);       // (direct path: two real rows)
    double* rb = ra + L;
    if (pow2) {
        for (int j = threadIdx.x; j < S.M / 2; j += blockDim.x) S.tw[j] = __ldg(T.tw + 2 * j); // W_M^j = W_L^2j
        __syncthreads();
    }
    const long long row = blockIdx.x;
    const double* src = in + row * L;
    double* dst = out + row * L;
    if (MODE == 0) {
        const double* X = dct2_row(src, L, T, S, pow2, ra, rb);
        for (int k = threadIdx.x; k < L; k += blockDim.x) dst[k] = X[k];
    } else if (MODE == 1) {
        double* X = pow2 ? reinterpret_cast<double*>(S.z1) : rb;
        for (int k = threadIdx.x; k < L; k += blockDim.x) X[k] = src[k];
        __syncthreads();
        dct3_row(X, L, T, S, dst, pow2);
    } else {
        double* X = dct2_row(src, L, T, S, pow2, ra, rb);
        const int v = static_cast<int>(row);
        const double lv = __ldg(T.lam_y + v) * ibh2, inv_b = 1.0 / (static_cast<double>(nx) * ny);
        for (int u = threadIdx.x; u < L; u += blockDim.x) {
            const double lam = __ldg(T.lam + u) * ibw2 + lv;
            X[u] = (u == 0 && v == 0) ? 0.0 : X[u] / lam * inv_b;
        }
        __syncthreads();
        dct3_row(X, L, T, S, dst, pow2);
    }
}

// out[c][r] = in[r][c], in is rows x cols; 32x32 tiles through shared memory (padded)
__global__ void k_transpose(int rows, int cols, const double* __restrict__ in, double* __restrict__ out)
{
    __shared__ double t[32][33];
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int j = threadIdx.y; j < 32; j += 8) {
        const int r = r0 + j, c = c0 + threadIdx.x;
        if (r < rows && c < cols) t[j][threadIdx.x] = in[static_cast<long long>(r) * cols + c];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += 8) {
        const int c = c0 + j, r = r0 + threadIdx.x;
        if (r < rows && c < cols) out[static_cast<long long>(c) * rows + r] = t[threadIdx.x][j];
    }
}

__global__ void k_dct_tables(int L, double2* __restrict__ tw, double2* __restrict__ qt, double* __restrict__ c4,
                             double* __restrict__ lam)
{
    for (int j = blockIdx.x * kBlock + threadIdx.x; j < 4 * L; j += gridDim.x * kBlock) {
        double s, c;
        if (j < L) lam[j] = 2.0 - 2.0 * cospi(static_cast<double>(j) / L);
        if (tw && j < L / 2) {
            sincospi(2.0 * j / L, &s, &c);
            tw[j] = make_double2(c, -s);
        }
        if (j < L) {
            sincospi(static_cast<double>(j) / (2.0 * L), &s, &c);
            qt[j] = make_double2(c, -s);
        }
        if (c4) c4[j] = cospi(static_cast<double>(j) / (2.0 * L));
    }
}

// D = 1/2 sum_b rho_b psi_b, per-block partial into part_d[2 b] (same grid as k_density_bins)
__global__ void __launch_bounds__(kBlock) k_electro_energy(long long B, const double* __restrict__ rho,
                                                           const double* __restrict__ psi, double* __restrict__ part_d,
                                                           const Ctrl* __restrict__ ctrl)
{
    __shared__ double sh[kBlock / 32];
    if (ctrl && ctrl->stopped) return;
    double e = 0.0;
    for (long long b = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x; b < B;
         b += static_cast<long long>(gridDim.x) * kBlock)
        e += rho[b] * psi[b];
    e = block_sum<kBlock>(e, sh);
    if (threadIdx.x == 0) part_d[2 * blockIdx.x] = 0.5 * e;
}

bool is_pow2(int L) { return L >= 4 && (L & (L - 1)) == 0; }

// ---------------------------------------------------------------------------------------------------
// Batched line transforms (power-of-two lengths 32 .. 4096): 128 threads carry 1024 / M lines of M = L/2
// complex points (8 per thread), the FFT in registers by radix-8 Stockham stages (one shared-memory round
// trip per stage, then one radix-2 or radix-4 stage when log2 M is not a multiple of 3), the M-point
// twiddles in shared memory.  Lines are rows (contiguous, the y passes) or columns (stride ny, the x pass
// reads 4..64 adjacent columns per CTA), so the 2-D solve needs no transposes.
// ---------------------------------------------------------------------------------------------------
constexpr int kLineThreads = 128;
constexpr double kRsqrt2 = 0.70710678118654752440;

template <bool INV>
__device__ __forceinline__ void dft4(double2& x0, double2& x1, double2& x2, double2& x3)
{
    const double2 s02 = make_double2(x0.x + x2.x, x0.y + x2.y), d02 = make_double2(x0.x - x2.x, x0.y - x2.y);
    const double2 s13 = make_double2(x1.x + x3.x, x1.y + x3.y), d13 = make_double2(x1.x - x3.x, x1.y - x3.y);
    const double2 r13 = INV ? make_double2(-d13.y, d13.x) : make_double2(d13.y, -d13.x); // -/+ i d13
    x0 = make_double2(s02.x + s13.x, s02.y + s13.y);
    x2 = make_double2(s02.x - s13.x, s02.y - s13.y);
    x1 = make_double2(d02.x + r13.x, d02.y + r13.y);
    x3 = make_double2(d02.x - r13.x, d02.y - r13.y);
}

// a[r] -> sum_n a[n] W8^{n r} (W8 = e^{-/+ 2 pi i / 8}): b = a_r + a_{r+4} (even outputs), c = (a_r - a_{r+4}) W8^r
// (odd outputs), two 4-point DFTs
template <bool INV>
__device__ __forceinline__ void dft8(double2 (&a)[8])
{
    double2 b[4], c[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        b[r] = make_double2(a[r].x + a[r + 4].x, a[r].y + a[r + 4].y);
        c[r] = make_double2(a[r].x - a[r + 4].x, a[r].y - a[r + 4].y);
    }
    const double sg = INV ? 1.0 : -1.0; // W8^1 = (1 + sg i) / sqrt2, W8^2 = sg i, W8^3 = (-1 + sg i) / sqrt2
    c[1] = make_double2((c[1].x - sg * c[1].y) * kRsqrt2, (c[1].y + sg * c[1].x) * kRsqrt2);
    c[2] = make_double2(-sg * c[2].y, sg * c[2].x);
    c[3] = make_double2((-c[3].x - sg * c[3].y) * kRsqrt2, (-c[3].y + sg * c[3].x) * kRsqrt2);
    dft4<INV>(b[0], b[1], b[2], b[3]);
    dft4<INV>(c[0], c[1], c[2], c[3]);
#pragma unroll
    for (int m = 0; m < 4; ++m) a[2 * m] = b[m], a[2 * m + 1] = c[m];
}

__device__ __forceinline__ double2 tw_at(const double2* twM, int m, bool inv)
{
    const double2 w = twM[m];
    return inv ? make_double2(w.x, -w.y) : w;
}

// In-place Stockham FFT of the M-point line z (natural order in and out), thread t of T = M/8 per line.
// Every thread of the block takes part in every barrier.
template <bool INV>
__device__ void fft_line8(double2* z, int M, int t, const double2* twM)
{
    const int q8 = M >> 3;
    int Ns = 1;
    for (; Ns * 8 <= M; Ns *= 8) {
        const int j = t, k = j & (Ns - 1);
        double2 a[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) a[r] = z[j + r * q8];
        if (Ns > 1) {
            const int step = k * (M / (8 * Ns));
#pragma unroll
            for (int r = 1; r < 8; ++r) a[r] = cmul(a[r], tw_at(twM, r * step, INV));
        }
        dft8<INV>(a);
        __syncthreads(); // (in place: every read of the stage before any write)
        const int base = (j - k) * 8 + k;
#pragma unroll
        for (int r = 0; r < 8; ++r) z[base + r * Ns] = a[r];
        __syncthreads();
    }
    if (Ns == M) return;
    if (Ns * 4 == M) { // radix 4: two butterflies per thread
        const int q = M >> 2;
        double2 a[2][4];
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const int j = t + b * q8, k = j & (Ns - 1), step = k * (M / (4 * Ns));
#pragma unroll
            for (int r = 0; r < 4; ++r) a[b][r] = z[j + r * q];
#pragma unroll
            for (int r = 1; r < 4; ++r) a[b][r] = cmul(a[b][r], tw_at(twM, r * step, INV));
            dft4<INV>(a[b][0], a[b][1], a[b][2], a[b][3]);
        }
        __syncthreads();
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const int j = t + b * q8, k = j & (Ns - 1), base = (j - k) * 4 + k;
#pragma unroll
            for (int r = 0; r < 4; ++r) z[base + r * Ns] = a[b][r];
        }
        __syncthreads();
    } else { // radix 2: four butterflies per thread
        const int q = M >> 1;
        double2 a[4][2];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int j = t + b * q8, k = j & (Ns - 1), step = k * (M / (2 * Ns));
            const double2 x0 = z[j], x1 = cmul(z[j + q], tw_at(twM, step, INV));
            a[b][0] = make_double2(x0.x + x1.x, x0.y + x1.y);
            a[b][1] = make_double2(x0.x - x1.x, x0.y - x1.y);
        }
        __syncthreads();
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int j = t + b * q8, k = j & (Ns - 1), base = (j - k) * 2 + k;
            z[base] = a[b][0], z[base + Ns] = a[b][1];
        }
        __syncthreads();
    }
}

// DCT-II of the line held (Makhoul-reordered, as M complex) in z, FFT'd in place: the untangling split
// (dct2_row) pair-wise (k, M - k), so every thread reads its pairs before any X is written over z.
// X (L reals) overwrites z.  ti: this thread's index within its line, T threads per line.
__device__ void dct2_post(double2* z, int L, int M, int ti, int T, const double2* __restrict__ wL,
                          const double2* __restrict__ qt)
{
    double* X = reinterpret_cast<double*>(z);
    constexpr int kP = 5; // pairs per thread: ceil((M/2 + 1) / (M/8)) <= 5
    double out[kP][4];
    const int npair = M / 2 + 1; // k = 0 .. M/2 (k and M - k together)
#pragma unroll
    for (int nb = 0; nb < kP; ++nb) {
        const int k = ti + nb * T;
        if (k >= npair) break;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int kh = h ? M - k : k;
            const double2 a = z[kh < M ? kh : 0], bc = z[kh > 0 ? M - kh : 0];
            const double2 b = make_double2(bc.x, -bc.y);
            const double2 sm = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y + b.y));
            const double2 d = make_double2(0.5 * (a.x - b.x), 0.5 * (a.y - b.y));
            const double2 wd = cmul(wl(wL, kh, M), d);
            const double2 V = make_double2(sm.x + wd.y, sm.y - wd.x);
            const double2 q = __ldg(qt + kh);
            out[nb][2 * h] = V.x * q.x - V.y * q.y;
            if (kh > 0 && kh < M) {
                const double2 q2 = __ldg(qt + (L - kh));
                out[nb][2 * h + 1] = V.x * q2.x + V.y * q2.y;
            } else {
                out[nb][2 * h + 1] = 0.0;
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < kP; ++b) {
        const int k = ti + b * T;
        if (k >= npair) break;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int kh = h ? M - k : k;
            if (h && kh == k) continue; // (k = M/2 pairs with itself)
            X[kh] = out[b][2 * h];
            if (kh > 0 && kh < M) X[L - kh] = out[b][2 * h + 1];
        }
    }
    __syncthreads();
}

// DCT-III pre-twiddle (dct3_row) of X (L reals aliasing z) into the M-point spectrum in place, pair-wise.
__device__ void dct3_pre(double2* z, int L, int M, int ti, int T, const double2* __restrict__ wL,
                         const double2* __restrict__ qt)
{
    const double* X = reinterpret_cast<const double*>(z);
    auto Vk = [&](int k) {
        const double2 q = __ldg(qt + k);
        const double a = X[k], b = k > 0 ? X[L - k] : 0.0;
        return make_double2(q.x * a - q.y * b, -q.y * a - q.x * b);
    };
    constexpr int kP = 5;
    double2 out[kP][2];
    const int npair = M / 2 + 1;
#pragma unroll
    for (int nb = 0; nb < kP; ++nb) {
        const int k = ti + nb * T;
        if (k >= npair) break;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int kh = h ? M - k : k;
            if (kh >= M) { out[nb][h] = make_double2(0.0, 0.0); continue; }
            const double2 a = Vk(kh), bb = Vk(M - kh);
            const double2 b = make_double2(bb.x, -bb.y);
            const double2 sm = make_double2(a.x + b.x, a.y + b.y), d = make_double2(a.x - b.x, a.y - b.y);
            double2 w = wl(wL, kh, M);
            w.y = -w.y;
            const double2 wd = cmul(w, d);
            out[nb][h] = make_double2(sm.x - wd.y, sm.y + wd.x);
        }
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < kP; ++b) {
        const int k = ti + b * T;
        if (k >= npair) break;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int kh = h ? M - k : k;
            if (kh >= M || (h && kh == k)) continue;
            z[kh] = out[b][h];
        }
    }
    __syncthreads();
}

// MODE 0: DCT-II, 1: DCT-III, 2: the x pass DCT-III(DCT-II(line) / lambda_uv / (nx ny)), (0, 0) dropped.
// Line l of the launch: element n at in[l * line_step + n * elem_stride]; a CTA takes LPC = 1024 / M
// consecutive lines (2 at L = 1024: 512 CTAs for a 1024-line pass, ~3.5 per SM).
template <int MODE>
__global__ void __launch_bounds__(kLineThreads) k_dct_lines(int L, int nlines, long long line_step,
                                                            long long elem_stride, const double* __restrict__ in,
                                                            double* __restrict__ out, DctTables T, int nx, int ny,
                                                            double ibw2, double ibh2)
{
    extern __shared__ double2 lsm[];
    const int M = L >> 1, TPL = M >> 3, LPC = kLineThreads / TPL;
    const int lgL = __ffs(L) - 1, lgP = __ffs(LPC) - 1; // (powers of two: index math by shifts)
    double2* twM = lsm;                 // [M] W_M^m
    double2* lines = lsm + M;           // [LPC][M]
    for (int m = threadIdx.x; m < M; m += kLineThreads) {
        const int j = 2 * m; // W_M^m = W_L^{2m}, from the half table W_L^j (j < M), W_L^{j + M} = -W_L^j
        const double2 w = __ldg(T.tw + (j < M ? j : j - M));
        twM[m] = j < M ? w : make_double2(-w.x, -w.y);
    }
    const int l0 = blockIdx.x * LPC;
    const int nl = min(LPC, nlines - l0);
    // load, Makhoul-reordered (MODE 1 loads X as is)
    const bool cols = elem_stride != 1;
    for (int idx = threadIdx.x; idx < LPC * L; idx += kLineThreads) {
        int l, n;
        if (cols) l = idx & (LPC - 1), n = idx >> lgP; // (adjacent lines are adjacent in memory)
        else l = idx >> lgL, n = idx & (L - 1);
        double* v = reinterpret_cast<double*>(lines + l * M);
        const double x = l < nl ? in[(l0 + l) * line_step + n * elem_stride] : 0.0;
        v[MODE == 1 ? n : makhoul_pos(n, L)] = x;
    }
    __syncthreads();
    const int li = threadIdx.x / TPL, ti = threadIdx.x & (TPL - 1);
    double2* z = lines + li * M;
    if (MODE != 1) {
        fft_line8<false>(z, M, ti, twM);
        dct2_post(z, L, M, ti, TPL, T.tw, T.qt);
    }
    if (MODE == 2) {
        double* X = reinterpret_cast<double*>(z);
        const int v = l0 + li;
        const double lv = v < nlines ? __ldg(T.lam_y + v) * ibh2 : 1.0, inv_b = 1.0 / (static_cast<double>(nx) * ny);
        for (int u = ti; u < L; u += TPL) {
            const double lam = __ldg(T.lam + u) * ibw2 + lv;
            X[u] = (u == 0 && v == 0) ? 0.0 : X[u] / lam * inv_b;
        }
        __syncthreads();
    }
    if (MODE != 0) {
        dct3_pre(z, L, M, ti, TPL, T.tw, T.qt);
        fft_line8<true>(z, M, ti, twM);
    }
    for (int idx = threadIdx.x; idx < LPC * L; idx += kLineThreads) {
        int l, n;
        if (cols) l = idx & (LPC - 1), n = idx >> lgP;
        else l = idx >> lgL, n = idx & (L - 1);
        if (l >= nl) continue;
        const double* v = reinterpret_cast<const double*>(lines + l * M);
        out[(l0 + l) * line_step + n * elem_stride] = v[MODE == 0 ? n : makhoul_pos(n, L)];
    }
}

bool lines_path(int L) { return L >= 32 && L <= 2048 && (L & (L - 1)) == 0; } // (M / 8 <= 128 threads)

template <int MODE>
void launch_lines(int nlines, int L, long long line_step, long long elem_stride, const ElectroPlan::Axis& ax,
                  const ElectroPlan::Axis& other, const double* in, double* out, int nx, int ny, double ibw2,
                  double ibh2, cudaStream_t st)
{
    const int M = L / 2, LPC = kLineThreads / (M / 8);
    const size_t sm = sizeof(double2) * static_cast<size_t>(M) * (LPC + 1);
    if (sm > 48 * 1024) CK(cudaFuncSetAttribute(k_dct_lines<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                static_cast<int>(sm)));
    const DctTables T{ax.tw.p, ax.qt.p, ax.c4.p, ax.lam.p, other.lam.p};
    k_dct_lines<MODE><<<(nlines + LPC - 1) / LPC, kLineThreads, sm, st>>>(L, nlines, line_step, elem_stride, in, out, T,
                                                                          nx, ny, ibw2, ibh2);
    CK_LAUNCH();
}

size_t dct_smem(int L) { return is_pow2(L) ? 20 * static_cast<size_t>(L) + 16 : 16 * static_cast<size_t>(L); }

template <int MODE>
void launch_rows(int rows, int L, const ElectroPlan::Axis& ax, const ElectroPlan::Axis& other, const double* in,
                 double* out, int nx, int ny, double ibw2, double ibh2, cudaStream_t st)
{
    const size_t sm = dct_smem(L);
    if (sm > 48 * 1024) CK(cudaFuncSetAttribute(k_dct_rows<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                static_cast<int>(sm)));
    const DctTables T{ax.tw.p, ax.qt.p, ax.c4.p, ax.lam.p, other.lam.p};
    // power of two: one thread per radix-4 butterfly of the M = L/2-point FFT (M/4), so a 1024 grid's rows
    // fit one wave at 11 rows per SM; the direct path keeps a full block for its O(L) inner loops
    const int threads = is_pow2(L) ? std::max(32, std::min(kDctThreads, L / 8)) : kDctThreads;
    k_dct_rows<MODE><<<rows, threads, sm, st>>>(L, is_pow2(L), in, out, T, nx, ny, ibw2, ibh2);
    CK_LAUNCH();
}

} // namespace

void ElectroPlan::Axis::make(int len, cudaStream_t st)
{
    L = len;
    if (is_pow2(L)) {
        tw.alloc(L / 2), c4.release();
    } else {
        tw.release(), c4.alloc(4 * static_cast<size_t>(L));
    }
    qt.alloc(L), lam.alloc(L);
    k_dct_tables<<<blocks_for(4LL * L, kBlock), kBlock, 0, st>>>(L, tw.p, qt.p, c4.p, lam.p);
    CK_LAUNCH();
}

ElectroPlan::~ElectroPlan() { release(); }

void ElectroPlan::release() { nx = ny = 0; }

void ElectroPlan::ensure(int gx, int gy)
{
    if (gx == nx && gy == ny) return;
    if (dct_smem(std::max(gx, gy)) > 227 * 1024) // (one grid row per CTA in shared memory)
        throw Error(TDPG_ERR_VALIDATION, "validation error: electrostatic density supports up to 8192 bins per axis "
                                         "for power-of-two grids and 14528 otherwise");
    nx = gx, ny = gy;
    const long long B = static_cast<long long>(nx) * ny;
    rho.alloc(B), psi.alloc(B), r1.alloc(B), r2.alloc(B);
    ax.make(nx, 0), ay.make(ny, 0);
    CK(cudaStreamSynchronize(0));
}

// TDPG_DCT_LINES=0: the one-row-per-CTA kernels with transposes (A/B switch).
bool lines_fast()
{
    static const bool on = [] {
        const char* e = std::getenv("TDPG_DCT_LINES");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}

// psi = L^+ (rho - mean rho) on the session's grid (rho in plan.rho), stream-ordered on `st`.
void electro_solve(tdpg_session* s, cudaStream_t st)
{
    Grid& g = s->grid;
    ElectroPlan& E = g.electro;
    const int nx = g.nx, ny = g.ny;
    const double ibw2 = 1.0 / (g.bw * g.bw), ibh2 = 1.0 / (g.bh * g.bh);
    if (lines_path(nx) && lines_path(ny) && lines_fast()) { // batched lines, no transposes (layout: bin (x, y) at x ny + y)
        launch_lines<0>(nx, ny, ny, 1, E.ay, E.ax, E.rho, E.r1, nx, ny, ibw2, ibh2, st);   // DCT-II along y (rows)
        launch_lines<2>(ny, nx, 1, ny, E.ax, E.ay, E.r1, E.r2, nx, ny, ibw2, ibh2, st);    // x: II, /lambda, III (columns)
        launch_lines<1>(nx, ny, ny, 1, E.ay, E.ax, E.r2, E.psi, nx, ny, ibw2, ibh2, st);   // DCT-III along y
        return;
    }
    const dim3 tb(32, 8);
    launch_rows<0>(nx, ny, E.ay, E.ax, E.rho, E.r1, nx, ny, ibw2, ibh2, st);                        // DCT-II along y
    k_transpose<<<dim3((ny + 31) / 32, (nx + 31) / 32), tb, 0, st>>>(nx, ny, E.r1, E.r2);     // -> [ny][nx]
    launch_rows<2>(ny, nx, E.ax, E.ay, E.r2, E.r1, nx, ny, ibw2, ibh2, st);                         // x: II, /lambda, III
    k_transpose<<<dim3((nx + 31) / 32, (ny + 31) / 32), tb, 0, st>>>(ny, nx, E.r1, E.r2);     // -> [nx][ny]
    launch_rows<1>(nx, ny, E.ay, E.ax, E.r2, E.psi, nx, ny, ibw2, ibh2, st);                        // DCT-III along y
    CK_LAUNCH();
}

void electro_energy(tdpg_session* s, double* part_d, int nblk, const Ctrl* ctrl, cudaStream_t st)
{
    Grid& g = s->grid;
    k_electro_energy<<<nblk, kBlock, 0, st>>>(g.bins(), g.electro.rho, g.electro.psi, part_d, ctrl);
    CK_LAUNCH();
}

} // namespace tdpg
