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
// Each 1D DCT is an N-point real FFT of the even/odd-reordered sequence plus a twiddle (Makhoul 1980),
// run as batched cuFFT D2Z / Z2D along the contiguous axis; the other axis is reached by a tiled
// shared-memory transpose.  All steps are stream-ordered and capturable into the iteration graph.
#include <cufft.h>

#include <cmath>

#include "gp_kernels.cuh"

namespace tdpg {

namespace {

void cufft_check(cufftResult r, const char* what)
{
    if (r != CUFFT_SUCCESS) throw Error(TDPG_ERR_CUDA, std::string("cufft error ") + std::to_string(r) + " (" + what + ")");
}

// v[m] = x[2m] for m < ceil(L/2), else x[2(L-1-m)+1]  (rows of length L)
__global__ void k_dct_pre(long long total, int L, const double* __restrict__ in, double* __restrict__ out)
{
    const long long i = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x;
    if (i >= total) return;
    const long long row = i / L;
    const int m = static_cast<int>(i - row * L);
    const int src = m < (L + 1) / 2 ? 2 * m : 2 * (L - 1 - m) + 1;
    out[i] = in[row * L + src];
}

// X[k] = Re(exp(-i pi k / 2L) V[k]), V[k > L/2] = conj(V[L - k])
__global__ void k_dct_post(long long total, int L, const double2* __restrict__ z, double* __restrict__ out)
{
    const long long i = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x;
    if (i >= total) return;
    const long long row = i / L;
    const int k = static_cast<int>(i - row * L), H = L / 2 + 1;
    double s, c;
    sincospi(static_cast<double>(k) / (2.0 * L), &s, &c);
    if (k < H) {
        const double2 v = z[row * H + k];
        out[i] = v.x * c + v.y * s;
    } else {
        const double2 v = z[row * H + (L - k)];
        out[i] = v.x * c - v.y * s;
    }
}

// DCT-III pre-twiddle: V[k] = exp(+i pi k / 2L) (X[k] - i X[L-k]), k = 0..L/2 (X[L] := 0)
__global__ void k_dct3_pre(long long total_h, int L, const double* __restrict__ X, double2* __restrict__ z)
{
    const int H = L / 2 + 1;
    const long long i = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x;
    if (i >= total_h) return;
    const long long row = i / H;
    const int k = static_cast<int>(i - row * H);
    const double a = X[row * L + k], b = k > 0 ? X[row * L + (L - k)] : 0.0;
    double s, c;
    sincospi(static_cast<double>(k) / (2.0 * L), &s, &c);
    z[i] = make_double2(c * a + s * b, s * a - c * b); // (c + i s)(a - i b)
}

// x[2m] = v[m] (m < ceil(L/2)), x[2(L-1-m)+1] = v[m]
__global__ void k_dct3_post(long long total, int L, const double* __restrict__ v, double* __restrict__ out)
{
    const long long i = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x;
    if (i >= total) return;
    const long long row = i / L;
    const int m = static_cast<int>(i - row * L);
    const int dst = m < (L + 1) / 2 ? 2 * m : 2 * (L - 1 - m) + 1;
    out[row * L + dst] = v[i];
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

// coefficients in the transposed layout A^T[v][u] (ny rows of nx): divide by lambda_uv, drop (0,0),
// fold in the inverse transform's 1 / (nx ny)
__global__ void k_poisson_scale(int nx, int ny, double ibw2, double ibh2, double* __restrict__ a)
{
    const long long i = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x;
    if (i >= static_cast<long long>(nx) * ny) return;
    const int v = static_cast<int>(i / nx), u = static_cast<int>(i - static_cast<long long>(v) * nx);
    if (u == 0 && v == 0) {
        a[i] = 0.0;
        return;
    }
    const double lam = (2.0 - 2.0 * cospi(static_cast<double>(u) / nx)) * ibw2 +
                       (2.0 - 2.0 * cospi(static_cast<double>(v) / ny)) * ibh2;
    a[i] = a[i] / lam / (static_cast<double>(nx) * ny);
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

} // namespace

ElectroPlan::~ElectroPlan() { release(); }

void ElectroPlan::release()
{
    for (auto& p : plan)
        if (p) cufftDestroy(p), p = 0;
    nx = ny = 0;
}

void ElectroPlan::ensure(int gx, int gy)
{
    if (gx == nx && gy == ny) return;
    release();
    nx = gx, ny = gy;
    const long long B = static_cast<long long>(nx) * ny;
    rho.alloc(B), psi.alloc(B), r1.alloc(B), r2.alloc(B);
    z.alloc(std::max(static_cast<long long>(nx) * (ny / 2 + 1), static_cast<long long>(ny) * (nx / 2 + 1)));
    int n_y[1] = {ny}, n_x[1] = {nx};
    cufft_check(cufftPlanMany(&plan[0], 1, n_y, nullptr, 1, ny, nullptr, 1, ny / 2 + 1, CUFFT_D2Z, nx), "plan y D2Z");
    cufft_check(cufftPlanMany(&plan[1], 1, n_x, nullptr, 1, nx, nullptr, 1, nx / 2 + 1, CUFFT_D2Z, ny), "plan x D2Z");
    cufft_check(cufftPlanMany(&plan[2], 1, n_x, nullptr, 1, nx / 2 + 1, nullptr, 1, nx, CUFFT_Z2D, ny), "plan x Z2D");
    cufft_check(cufftPlanMany(&plan[3], 1, n_y, nullptr, 1, ny / 2 + 1, nullptr, 1, ny, CUFFT_Z2D, nx), "plan y Z2D");
}

// psi = L^+ (rho - mean rho) on the session's grid (rho in plan.rho), stream-ordered on `st`.
void electro_solve(tdpg_session* s, cudaStream_t st)
{
    Grid& g = s->grid;
    ElectroPlan& E = g.electro;
    const int nx = g.nx, ny = g.ny;
    const long long B = g.bins();
    const unsigned nb = blocks_for(B, kBlock);
    auto hz = [&](int L, int batch) { return static_cast<long long>(batch) * (L / 2 + 1); };
    auto d2z = [&](cufftHandle p, double* in, double2* out) {
        cufft_check(cufftSetStream(p, st), "set stream");
        cufft_check(cufftExecD2Z(p, in, reinterpret_cast<cufftDoubleComplex*>(out)), "exec D2Z");
    };
    auto z2d = [&](cufftHandle p, double2* in, double* out) {
        cufft_check(cufftSetStream(p, st), "set stream");
        cufft_check(cufftExecZ2D(p, reinterpret_cast<cufftDoubleComplex*>(in), out), "exec Z2D");
    };
    const dim3 tb(32, 8);
    // forward DCT-II along y (rows of length ny), then along x (after a transpose)
    k_dct_pre<<<nb, kBlock, 0, st>>>(B, ny, E.rho, E.r1);
    d2z(E.plan[0], E.r1, E.z);
    k_dct_post<<<nb, kBlock, 0, st>>>(B, ny, E.z, E.r2);
    k_transpose<<<dim3((ny + 31) / 32, (nx + 31) / 32), tb, 0, st>>>(nx, ny, E.r2, E.r1); // -> [ny][nx]
    k_dct_pre<<<nb, kBlock, 0, st>>>(B, nx, E.r1, E.r2);
    d2z(E.plan[1], E.r2, E.z);
    k_dct_post<<<nb, kBlock, 0, st>>>(B, nx, E.z, E.r1); // A^T [ny][nx]
    k_poisson_scale<<<nb, kBlock, 0, st>>>(nx, ny, 1.0 / (g.bw * g.bw), 1.0 / (g.bh * g.bh), E.r1);
    // inverse DCT-III along x, transpose back, along y
    k_dct3_pre<<<blocks_for(hz(nx, ny), kBlock), kBlock, 0, st>>>(hz(nx, ny), nx, E.r1, E.z);
    z2d(E.plan[2], E.z, E.r2);
    k_dct3_post<<<nb, kBlock, 0, st>>>(B, nx, E.r2, E.r1);
    k_transpose<<<dim3((nx + 31) / 32, (ny + 31) / 32), tb, 0, st>>>(ny, nx, E.r1, E.r2); // -> [nx][ny]
    k_dct3_pre<<<blocks_for(hz(ny, nx), kBlock), kBlock, 0, st>>>(hz(ny, nx), ny, E.r2, E.z);
    z2d(E.plan[3], E.z, E.r1);
    k_dct3_post<<<nb, kBlock, 0, st>>>(B, ny, E.r1, E.psi);
    CK_LAUNCH();
}

void electro_energy(tdpg_session* s, double* part_d, int nblk, const Ctrl* ctrl, cudaStream_t st)
{
    Grid& g = s->grid;
    k_electro_energy<<<nblk, kBlock, 0, st>>>(g.bins(), g.electro.rho, g.electro.psi, part_d, ctrl);
    CK_LAUNCH();
}

} // namespace tdpg
