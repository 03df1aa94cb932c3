// step_scalars.cu — the SBCI1 step's small-matrix algebra on the device (one thread), so the commit
// pass can follow the subspace pass without a host round trip (SURVEY §7 hard part 6).
//
// It restates, operation for operation, what the host does between the two passes
// (sbci1.hpp:193-246 via host_math.hpp): symmetrise the 2x2 / 3x3 subspace matrix
// V_ij = (h_ij + h_ji) / 2, diagonalise it with the reference's cyclic Jacobi (small_eig.hpp:46-106:
// rotation formula, sweep order, stopping rule, stable ascending sort), and form k, b, c and the
// second-Ritz coefficients (sbci1.hpp:230-254, 287-311). This file is compiled with --fmad=false
// and uses only +, -, *, / and sqrt, which CUDA rounds exactly like the host's IEEE double
// arithmetic (x86-64 without -march emits no FMA), so every scalar — and therefore every branch the
// host takes after reading them back — is bit-identical to the host path (kept as the fallback).
#include <cmath>

#include "common.cuh"
#include "kernels.cuh"

namespace sbg {

namespace {

__device__ void jacobi_small(int n, double m[3][3], double ev[3], double vec[3][3]) {
    double v[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) v[i][j] = (i == j) ? 1.0 : 0.0;
    double fro = 0.0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) fro += m[i][j] * m[i][j];
    const double stop = 1e-30 * fmax(fro, 1e-300);
    auto offdiag = [&]() {
        double s = 0.0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                if (i != j) s += m[i][j] * m[i][j];
        return s;
    };
    for (int sweep = 0; sweep < 100 && offdiag() > stop; ++sweep)
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                const double apq = m[p][q];
                if (apq == 0.0) continue;
                const double tau = (m[q][q] - m[p][p]) / (2.0 * apq);
                const double t = (tau >= 0.0) ? 1.0 / (tau + sqrt(1.0 + tau * tau)) : 1.0 / (tau - sqrt(1.0 + tau * tau));
                const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
                for (int k = 0; k < n; ++k) {
                    const double a = m[k][p], b = m[k][q];
                    m[k][p] = c * a - s * b;
                    m[k][q] = s * a + c * b;
                }
                for (int k = 0; k < n; ++k) {
                    const double a = m[p][k], b = m[q][k];
                    m[p][k] = c * a - s * b;
                    m[q][k] = s * a + c * b;
                }
                for (int k = 0; k < n; ++k) {
                    const double a = v[k][p], b = v[k][q];
                    v[k][p] = c * a - s * b;
                    v[k][q] = s * a + c * b;
                }
            }
    // stable ascending sort of the diagonal (std::stable_sort on indices)
    int order[3] = {0, 1, 2};
    for (int i = 1; i < n; ++i) {
        const int key = order[i];
        int j = i - 1;
        while (j >= 0 && m[key][key] < m[order[j]][order[j]]) {
            order[j + 1] = order[j];
            --j;
        }
        order[j + 1] = key;
    }
    for (int k = 0; k < n; ++k) {
        ev[k] = m[order[k]][order[k]];
        for (int i = 0; i < n; ++i) vec[i][k] = v[i][order[k]];
    }
}

__global__ void k_step_scalars(const double* __restrict__ dots, const StepScalarArgs a, double* __restrict__ coef,
                               double* __restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int m = a.three ? 3 : 2;
    double v[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int i = 0; i < m; ++i)
        for (int j = i; j < m; ++j) v[i][j] = v[j][i] = 0.5 * (dots[i * m + j] + dots[j * m + i]);
    double ev[3], vec[3][3];
    jacobi_small(m, v, ev, vec);
    const double vx = vec[0][0], vy = a.three ? vec[1][0] : 0.0, vz = vec[m - 1][0];
    const double wx = vec[0][1], wy = a.three ? vec[1][1] : 0.0, wz = vec[m - 1][1];
    const double e_new = ev[0];
    const double k_den = vx * a.Ax + vy * a.Bx + vz * a.Cx;
    double flag = 0.0, k = 0.0, b = 0.0, c = 0.0;
    if (fabs(k_den) < 1e-14) {
        flag = 1.0;  // restart (StallSmallB), no commit
    } else {
        k = 1.0 / k_den;
        if (a.three) {
            const double b_den = vy * a.By + vz * a.Cy;
            if (fabs(b_den) < 1e-14) {
                flag = 1.0;
            } else {
                b = k * b_den;
                c = -vz * a.Cz / b_den;
            }
        } else {
            b = 1.0;
            c = -k * vz * a.Cz;
        }
    }
    out[0] = flag;
    out[1] = k;
    out[2] = b;
    out[3] = c;
    out[4] = e_new;
    out[5] = ev[1];
    out[6] = wx * a.Ax + wy * a.Bx + wz * a.Cx;  // second Ritz vector (sbci1.hpp:287-311)
    out[7] = wy * a.By + wz * a.Cy;
    out[8] = wz * a.Cz;
    // coefficients of the merged guard + commit pass (solver.cu, slot layout: inputs x, y, z, Hx, Hy, Hz
    // = 0..5; outputs y', Hy', x', Hx', z' = kMaxIn + 0..4)
    constexpr int W = kMaxIn + kMaxOut;
    for (int i = 0; i < kMaxOut * W; ++i) coef[i] = 0.0;
    if (flag != 0.0) return;  // never read: the host restarts without committing
    if (a.three) {
        coef[0 * W + 1] = 1.0;
        coef[1 * W + 4] = 1.0;
    }
    coef[0 * W + 2] = -c;
    coef[1 * W + 5] = -c;
    coef[2 * W + 0] = 1.0;
    coef[2 * W + kMaxIn + 0] = b;
    coef[3 * W + 3] = 1.0;
    coef[3 * W + kMaxIn + 1] = b;
    coef[4 * W + kMaxIn + 3] = 1.0 / k;
    coef[4 * W + kMaxIn + 2] = -e_new / k;
}

}  // namespace

void launch_step_scalars(const double* dots, const StepScalarArgs& a, double* coef, double* out, cudaStream_t st) {
    k_step_scalars<<<1, 32, 0, st>>>(dots, a, coef, out);
    SBG_LAUNCH_CHECK();
}

}  // namespace sbg
