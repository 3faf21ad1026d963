// libfks host side: the C ABI of include/fks.h, the fp64 table generator (written from the
// paper independently of the oracle), the shift tables and the launch orchestration.
// Compiled with -fmad=false / -ffp-contract=off for the host so the shift formula rounds
// exactly as stated in DESIGN.md reading #16.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: NCCL is dlopen'ed by fks_set_comm (no link-time dependency)

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <thread>
#include <vector>

#include "../../include/fks.h"
#include "common.cuh"
#include "kernels.cuh"

namespace {

constexpr double kPi = 3.14159265358979323846;
const double kLambda = 2.0 / (3.0 + std::sqrt(2.0));

struct Dirs {
  std::vector<double> e;  // [A][dv]
  std::vector<double> w;  // [A]
};

// ------------------------------------------------------------------ radial functions
double sinc(double x) { return x == 0.0 ? 1.0 : std::sin(x) / x; }
// phi_R^2(s) = 2 R sinc(R s)
double phi2(double s, double R) { return 2.0 * R * sinc(R * s); }
// phi_R^3(s) = R^2 [2 sinc(R s) - sinc^2(R s / 2)]
double phi3(double s, double R) {
  const double h = sinc(0.5 * R * s);
  return R * R * (2.0 * sinc(R * s) - h * h);
}
// Reading #2 (P:501-506 derivation): psi(s) = 2 pi R J1(R s) / s, psi(0) = pi R^2
double psi3(double s, double R) { return s == 0.0 ? kPi * R * R : 2.0 * kPi * R * ::j1(R * s) / s; }

// NEXT-3 (reading #25): phi_{R,a}(s) = int_{-R}^{R} |rho|^gamma e^{i rho s} d rho
// = 2 R^{gamma+1} int_0^1 t^gamma cos(R s t) dt, by an n-point Gauss-Jacobi
// rule for the weight t^gamma.  Nodes: eigenvalues of the Jacobi matrix of P^(0,gamma) found by
// Sturm-sequence bisection, polished by Newton on the orthonormal recurrence; weights from the
// Christoffel sum 1 / sum_k q_k(x)^2.
struct GaussJacobi {
  std::vector<double> t, w;  // nodes in (0, 1), weights for int_0^1 t^gamma g(t) dt
};

GaussJacobi gauss_jacobi01(int n, double gamma) {
  const double a = 0.0, b = gamma, ab = a + b;
  std::vector<double> al(n), sb(n);  // diagonal alpha_k, off-diagonal sqrt(beta_{k+1})
  for (int k = 0; k < n; ++k) {
    al[k] = k == 0 ? (b - a) / (ab + 2.0) : (b * b - a * a) / ((2.0 * k + ab) * (2.0 * k + ab + 2.0));
    const double j = k + 1.0;
    sb[k] = std::sqrt(4.0 * j * (j + a) * (j + b) * (j + ab) /
                      ((2.0 * j + ab) * (2.0 * j + ab) * (2.0 * j + ab + 1.0) * (2.0 * j + ab - 1.0)));
  }
  const double mu0 = std::exp((ab + 1.0) * std::log(2.0) + std::lgamma(a + 1.0) + std::lgamma(b + 1.0) -
                              std::lgamma(ab + 2.0));
  auto below = [&](double x) {  // number of eigenvalues < x (Sturm sequence of J - x)
    int cnt = 0;
    double d = 1.0;
    for (int k = 0; k < n; ++k) {
      d = (al[k] - x) - (k ? sb[k - 1] * sb[k - 1] / d : 0.0);
      if (d == 0.0) d = -1e-300;
      if (d < 0.0) ++cnt;
    }
    return cnt;
  };
  // q_n(x), q_n'(x) and sum_{k<n} q_k(x)^2 by the orthonormal three-term recurrence
  auto recur = [&](double x, double* qn, double* dqn, double* ssum) {
    double qm = 0.0, q = 1.0 / std::sqrt(mu0), dm = 0.0, dq = 0.0, s = q * q;
    for (int k = 0; k < n; ++k) {
      const double prev = k ? sb[k - 1] : 0.0;
      const double q1 = ((x - al[k]) * q - prev * qm) / sb[k];
      const double d1 = (q + (x - al[k]) * dq - prev * dm) / sb[k];
      qm = q; q = q1; dm = dq; dq = d1;
      if (k < n - 1) s += q * q;
    }
    *qn = q; *dqn = dq; *ssum = s;
  };
  GaussJacobi g;
  g.t.resize(n);
  g.w.resize(n);
  for (int i = 0; i < n; ++i) {
    double lo = -1.0, hi = 1.0;
    for (int it = 0; it < 200 && hi - lo > 1e-17; ++it) {
      const double mid = 0.5 * (lo + hi);
      if (below(mid) > i) hi = mid; else lo = mid;
    }
    double x = 0.5 * (lo + hi), qn, dqn, ss;
    for (int it = 0; it < 3; ++it) {
      recur(x, &qn, &dqn, &ss);
      x -= qn / dqn;
    }
    recur(x, &qn, &dqn, &ss);
    g.t[i] = 0.5 * (1.0 + x);
    g.w[i] = std::exp2(-b - 1.0) / ss;
  }
  return g;
}

constexpr int kJacobiNodes = 160;  // exact for cos(z t) to rounding up to z ~ 300 (N = 64: z <= 160)

double phi_a(double s, double R, double gamma, const GaussJacobi& g) {
  double acc = 0.0;
  for (size_t i = 0; i < g.t.size(); ++i) acc += g.w[i] * std::cos(R * s * g.t[i]);
  return 2.0 * std::pow(R, gamma + 1.0) * acc;
}

// ------------------------------------------------------------------ direction sets
Dirs dirs_2d(int A) {  // P:490 theta_p = pi p / A, weight pi / A (reading #5)
  Dirs d;
  for (int p = 1; p <= A; ++p) {
    const double th = kPi * p / A;
    d.e.push_back(std::cos(th));
    d.e.push_back(std::sin(th));
    d.w.push_back(kPi / A);
  }
  return d;
}

double cubic(double t) { return ((105.0 * t - 105.0) * t + 21.0) * t - 1.0; }

// Reading #17: 24-point 7-design = O-orbit of (sqrt a, sqrt b, sqrt c), a<b<c the roots of
// 105 t^3 - 105 t^2 + 21 t - 1 (bracketed by sign changes on [0,.1], [.1,.3], [.3,1]).
Dirs dirs_design24() {
  const double br[4] = {0.0, 0.1, 0.3, 1.0};
  double r[3];
  for (int i = 0; i < 3; ++i) {
    double lo = br[i], hi = br[i + 1];
    const bool up = cubic(lo) < 0.0;
    for (int it = 0; it < 200; ++it) {
      const double mid = 0.5 * (lo + hi);
      if ((cubic(mid) < 0.0) == up) lo = mid; else hi = mid;
    }
    double t = 0.5 * (lo + hi);
    for (int it = 0; it < 3; ++it) t -= cubic(t) / ((315.0 * t - 210.0) * t + 21.0);
    r[i] = std::sqrt(t);
  }
  Dirs d;
  int perm[3] = {0, 1, 2};
  do {
    const int inv = (perm[0] > perm[1]) + (perm[0] > perm[2]) + (perm[1] > perm[2]);
    for (int sg = 0; sg < 8; ++sg) {
      const double s0 = (sg & 4) ? -1.0 : 1.0, s1 = (sg & 2) ? -1.0 : 1.0, s2 = (sg & 1) ? -1.0 : 1.0;
      const double det = ((inv & 1) ? -1.0 : 1.0) * s0 * s1 * s2;
      if (det < 0) continue;
      d.e.push_back(s0 * r[perm[0]]);
      d.e.push_back(s1 * r[perm[1]]);
      d.e.push_back(s2 * r[perm[2]]);
      d.w.push_back(2.0 * kPi / 24.0);
    }
  } while (std::next_permutation(perm, perm + 3));
  return d;
}

// P:527-540 with the sin(theta) Jacobian and midpoint theta (reading #6), sum w = 2 pi.
Dirs dirs_product(int A1) {
  Dirs d;
  double tot = 0.0;
  for (int p = 0; p < A1; ++p)
    for (int q = 0; q < A1; ++q) {
      const double th = (p + 0.5) * kPi / A1, ph = q * kPi / A1;
      d.e.push_back(std::sin(th) * std::cos(ph));
      d.e.push_back(std::sin(th) * std::sin(ph));
      d.e.push_back(std::cos(th));
      const double w = kPi * kPi * std::sin(th) / (A1 * A1);
      d.w.push_back(w);
      tot += w;
    }
  for (double& w : d.w) w *= 2.0 * kPi / tot;
  return d;
}

bool default_dirs(int dv, int M, Dirs* out) {
  if (M <= 0) return false;
  if (dv == 2) { *out = dirs_2d(M); return true; }
  if (M == 24) { *out = dirs_design24(); return true; }
  const int a = (int)std::lround(std::sqrt((double)M));
  if (a * a == M) { *out = dirs_product(a); return true; }
  return false;
}

int mu(int j, int N) { return j < N / 2 ? j : j - N; }

// The Carleman kernel is constant -- closed-form radial functions -- exactly when gamma = d - 2
// (2D Maxwell molecules, 3D hard spheres); otherwise the decoupled model of reading #25.
bool exact_gamma(int dv, double gamma) { return gamma == (double)(dv - 2); }

// Unfolded tables: alpha, alphap [A][n] in FFT mode order, symmetrised over
// l -> -l (reading #10), and D = sum_p w_p alpha_p alpha'_p.  Directions are built in parallel
// host threads (the general-gamma radial function is a 160-point quadrature per entry).
void build_tables(int dv, int N, double R, double gamma, const Dirs& dirs, std::vector<double>& alpha,
                  std::vector<double>& alphap, std::vector<double>& D) {
  const int A = (int)dirs.w.size();
  const int n = dv == 3 ? N * N * N : N * N;
  alpha.assign((size_t)A * n, 0.0);
  alphap.assign((size_t)A * n, 0.0);
  const bool exact = exact_gamma(dv, gamma);
  GaussJacobi gj;
  if (!exact) gj = gauss_jacobi01(kJacobiNodes, gamma);
  auto one_dir = [&](int p) {
    std::vector<double> ra(n), rb(n);
    const double* e = &dirs.e[(size_t)p * dv];
    for (int k = 0; k < n; ++k) {
      const double lx = mu(k % N, N), ly = mu((k / N) % N, N), lz = dv == 3 ? mu(k / (N * N), N) : 0.0;
      if (dv == 2) {
        const double dot = lx * e[0] + ly * e[1];
        ra[k] = exact ? phi2(dot, R) : phi_a(dot, R, gamma, gj);
        rb[k] = phi2(-lx * e[1] + ly * e[0], R);  // e_perp = e_{theta + pi/2}
      } else {
        const double dot = lx * e[0] + ly * e[1] + lz * e[2];
        const double cx = ly * e[2] - lz * e[1], cy = lz * e[0] - lx * e[2], cz = lx * e[1] - ly * e[0];
        ra[k] = exact ? phi3(dot, R) : phi_a(dot, R, gamma, gj);
        rb[k] = psi3(std::sqrt(cx * cx + cy * cy + cz * cz), R);
      }
    }
    for (int k = 0; k < n; ++k) {
      const int x = k % N, y = (k / N) % N, z = dv == 3 ? k / (N * N) : 0;
      const int mx = (N - x) % N, my = (N - y) % N, mz = (N - z) % N;
      const int km = dv == 3 ? mx + N * (my + N * mz) : mx + N * my;
      alpha[(size_t)p * n + k] = 0.5 * (ra[k] + ra[km]);
      alphap[(size_t)p * n + k] = 0.5 * (rb[k] + rb[km]);
    }
  };
  const int nth = std::max(1, std::min<int>(A, (int)std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (int t = 0; t < nth; ++t)
    pool.emplace_back([&, t]() {
      for (int p = t; p < A; p += nth) one_dir(p);
    });
  for (auto& th : pool) th.join();
  D.assign(n, 0.0);
  for (int p = 0; p < A; ++p)
    for (int k = 0; k < n; ++k) D[k] += dirs.w[p] * alpha[(size_t)p * n + k] * alphap[(size_t)p * n + k];
}

// s = Btilde kappa^-(d+gamma), Btilde = 2^{d-1} C (reading #3): 2D Maxwell 2 b0 (L/pi)^2, 3D hard
// spheres 4 C1 (L/pi)^4; any gamma (reading #25): 2^{d-1} C (L/pi)^{d+gamma}.
double node_scale(int dv, double L, double kconst, double gamma) {
  const double k = L / kPi;
  if (exact_gamma(dv, gamma)) return dv == 2 ? 2.0 * kconst * k * k : 4.0 * kconst * k * k * k * k;
  return (dv == 2 ? 2.0 : 4.0) * kconst * std::pow(k, dv + gamma);
}

bool valid_gamma(double g) { return g > -1.0 && g <= 2.0; }

double default_kconst(int dv) { return dv == 2 ? 1.0 / (2.0 * kPi) : 1.0 / (4.0 * kPi); }

// delta for one axis (a1, reading #16): s^n = floor(0.5 - n * ((v dt) / h)); no contraction.
void shift_delta(int64_t n, int N, double L, double dt, double h, int8_t* out) {
  const double dv = 2.0 * L / N;
  for (int k = 0; k < N; ++k) {
    volatile double v = -L + (k + 0.5) * dv;
    volatile double vdt = v * dt;
    volatile double c = vdt / h;
    volatile double t0 = (double)n * c;
    volatile double t1 = (double)(n + 1) * c;
    volatile double a0 = 0.5 - t0;
    volatile double a1 = 0.5 - t1;
    out[k] = (int8_t)((int64_t)std::floor(a1) - (int64_t)std::floor(a0));
  }
}

// NEXT-4 (Strang, reading #26): delta between the half-step positions p and p + 1 (time p dt / 2):
// s = floor(0.5 - (p * c) * 0.5); for even p this is bitwise the full-step s^{p/2} above.
void shift_delta_half(int64_t p, int N, double L, double dt, double h, int8_t* out) {
  const double dv = 2.0 * L / N;
  for (int k = 0; k < N; ++k) {
    volatile double v = -L + (k + 0.5) * dv;
    volatile double vdt = v * dt;
    volatile double c = vdt / h;
    volatile double t0 = (double)p * c;
    volatile double t1 = (double)(p + 1) * c;
    volatile double h0 = t0 * 0.5;
    volatile double h1 = t1 * 0.5;
    volatile double a0 = 0.5 - h0;
    volatile double a1 = 0.5 - h1;
    out[k] = (int8_t)((int64_t)std::floor(a1) - (int64_t)std::floor(a0));
  }
}

bool invert(std::vector<double> a, int m, double* out) {  // Gauss-Jordan with partial pivoting
  std::vector<double> b((size_t)m * m, 0.0);
  for (int i = 0; i < m; ++i) b[(size_t)i * m + i] = 1.0;
  for (int c = 0; c < m; ++c) {
    int piv = c;
    for (int r = c + 1; r < m; ++r)
      if (std::fabs(a[(size_t)r * m + c]) > std::fabs(a[(size_t)piv * m + c])) piv = r;
    if (a[(size_t)piv * m + c] == 0.0) return false;
    for (int k = 0; k < m; ++k) {
      std::swap(a[(size_t)c * m + k], a[(size_t)piv * m + k]);
      std::swap(b[(size_t)c * m + k], b[(size_t)piv * m + k]);
    }
    const double d = a[(size_t)c * m + c];
    for (int k = 0; k < m; ++k) { a[(size_t)c * m + k] /= d; b[(size_t)c * m + k] /= d; }
    for (int r = 0; r < m; ++r) {
      if (r == c) continue;
      const double f = a[(size_t)r * m + c];
      for (int k = 0; k < m; ++k) { a[(size_t)r * m + k] -= f * a[(size_t)c * m + k]; b[(size_t)r * m + k] -= f * b[(size_t)c * m + k]; }
    }
  }
  std::memcpy(out, b.data(), sizeof(double) * m * m);
  return true;
}

}  // namespace

struct fks_ctx {
  fks_grid grid;
  int dv = 0, N = 0, n = 0, A = 0;
  double L = 0, h = 0, gamma = 0;
  double tau = 1.0, kconst = 0.0, R = 0.0;
  int project = 1;
  Dirs dirs;
  int64_t ncells = 0;      // local cells
  int64_t step_n = 0;      // FKS step counter n
  double dt = 0.0;
  cudaStream_t stream = 0;
  int sm_count = 0;
  int nclusters = 0;       // 3D persistent clusters
  double Ginv[25];
  double2* d_tables = nullptr;
  int64_t table_elems = 0;
  double2* d_scratch = nullptr;
  unsigned* d_sync = nullptr;  // 3D group counters
  int* d_flag = nullptr;
  int* d_fluid = nullptr;
  int nfluid = 0;
  int* d_solid_list = nullptr;
  int nsolid = 0;
  uint8_t* d_solid = nullptr;
  int reflect = 0;  // NEXT-1: specular reflection at solid cells
  double* d_ghost[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  const double* halo[2] = {nullptr, nullptr};  // caller-owned neighbour planes (FKS_BC_HALO)
  int split = FKS_SPLIT_LIE;       // NEXT-4 time scheme (fks_set_scheme)
  int integ = FKS_TIME_EULER;
  double* d_tmp = nullptr;         // one state-sized scratch for the Heun / Strang sequences
  double* d_inplace = nullptr;     // in-place calls (f_out == f_in): the result lands here first
  double* d_host_in = nullptr;
  double* d_host_out = nullptr;
  // fks_step_host pipeline (0D, no solids): copy streams and per-chunk events
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_out;
  int64_t launches = 0;
  // a2 inside the library (fks_set_comm / fks_set_comm_loopback): per HALO face f (0 = lo, 1 = hi of
  // the slab axis) a library-owned neighbour plane [pc][n], packed send / receive buffers holding only
  // the velocity slices whose shift crosses that face this step, a communication stream and events.
  int comm_kind = 0;               // 0 none, 1 NCCL, 2 loopback
  ncclComm_t nccl = nullptr;
  fks_loopback* loop = nullptr;
  int rank = 0, nranks = 1;
  int peer[2] = {-1, -1};          // neighbour rank across the lo / hi face (-1: not a HALO face)
  cudaStream_t s_comm = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_halo = nullptr, ev_packed = nullptr;
  double* d_halo[2] = {nullptr, nullptr};
  double* d_send[2] = {nullptr, nullptr};
  double* d_recv[2] = {nullptr, nullptr};
  fks::SliceList send_sl[2], recv_sl[2];
  int64_t pc = 0;                  // cells per plane of the slab axis
  int64_t posted = -1;             // step whose exchange has been posted
  int64_t bytes_sent = 0;          // payload sent by the last exchange (both faces)
  int* d_interior = nullptr;       // fluid cells that never read a halo plane
  int ninterior = 0;
  int* d_boundary = nullptr;       // fluid cells on a HALO-face plane
  int nboundary = 0;
  std::vector<uint8_t> h_solid;    // host copy of the solid mask (empty: none)
  uint8_t* d_halo_solid[2] = {nullptr, nullptr};  // neighbour planes' solid flags (specular + comm)
  uint8_t* d_zero_mask = nullptr;  // all-fluid mask / plane for contexts without solids (specular)
  // fks_step_host on a spatial grid: per plane-chunk fluid / solid cell lists (built on first use)
  std::vector<int64_t> chunk_first;  // first plane of each chunk (+ the end)
  std::vector<int*> d_chunk_fluid, d_chunk_solid;
  std::vector<int> n_chunk_fluid, n_chunk_solid;
};

// Loopback communicator: contexts of one process (one device) exchange through device copies,
// so a partitioned run can be checked on one GPU (fks_comm_loopback_create).
struct fks_loopback {
  int nranks = 0;
  std::vector<fks_ctx*> ctx;
};

namespace {

fks_status cuda_fail(cudaError_t e) { return e == cudaSuccess ? FKS_OK : FKS_E_CUDA; }

fks_status upload_tables(fks_ctx* c) {
  std::vector<double> al, alp, D;
  build_tables(c->dv, c->N, c->R, c->gamma, c->dirs, al, alp, D);
  const int n = c->n, N = c->N, A = c->A;
  const double s = node_scale(c->dv, c->L, c->kconst, c->gamma);
  // Fold s, w_p and 1/n (the kernels use the unnormalised forward DFT) into the tables.
  auto folded = [&](int p, int k) {
    return p < A ? make_double2(s * c->dirs.w[p] * al[(size_t)p * n + k] / n, alp[(size_t)p * n + k] / n)
                 : make_double2(s * D[k] / n, 0.0);
  };
  std::vector<double2> T;
  if (c->dv == 2 || N == 64 || N == 4) {  // T[p][k], k = l_x + N l_y (+ N^2 l_z)
    T.resize((size_t)(A + 1) * n);
    for (int p = 0; p <= A; ++p)
      for (int k = 0; k < n; ++k) T[(size_t)p * n + k] = folded(p, k);
  } else {
    // T3[p][rank][row][l_x]: rank r owns the l_y planes at positions r*NP .. r*NP+NP-1 of the
    // order 0, N/2, 1, N-1, 2, N-2, ...; it stores the first plane of each mirror pair (N rows
    // l_z) and the rows l_z <= N/2 of the self-mirror planes 0 and N/2 (kernels3d.cu Cfg3).
    int P = 0, NP = 0, slabr = 0;
    if (fks::table_layout3d(N, &P, &NP, &slabr) != 0) return FKS_E_INVAL;
    auto plane_of = [&](int q) { return q == 0 ? 0 : q == 1 ? N / 2 : (q & 1) ? N - q / 2 : q / 2; };
    T.assign((size_t)(A + 1) * P * slabr * N, make_double2(0.0, 0.0));
    for (int p = 0; p <= A; ++p)
      for (int r = 0; r < P; ++r) {
        int row = 0;
        for (int e = 0; e < NP; ++e) {
          const int ly = plane_of(r * NP + e);
          int nrows = 0;
          if (ly == 0 || ly == N / 2) nrows = N / 2 + 1;
          else if ((e & 1) == 0) nrows = N;
          for (int lz = 0; lz < nrows; ++lz, ++row)
            for (int lx = 0; lx < N; ++lx)
              T[(((size_t)p * P + r) * slabr + row) * N + lx] = folded(p, lx + N * (ly + N * lz));
        }
      }
  }
  if (c->d_tables) cudaFree(c->d_tables);
  c->d_tables = nullptr;
  if (cudaMalloc(&c->d_tables, T.size() * sizeof(double2)) != cudaSuccess) return FKS_E_NOMEM;
  c->table_elems = (int64_t)T.size();
  return cuda_fail(cudaMemcpy(c->d_tables, T.data(), T.size() * sizeof(double2), cudaMemcpyHostToDevice));
}

void build_gram(fks_ctx* c) {
  const int m = c->dv + 2;
  std::vector<double> g((size_t)m * m, 0.0);
  const double dv = 2.0 * c->L / c->N;
  for (int k = 0; k < c->n; ++k) {
    double v[3] = {-c->L + (k % c->N + 0.5) * dv, -c->L + ((k / c->N) % c->N + 0.5) * dv,
                   c->dv == 3 ? -c->L + (k / (c->N * c->N) + 0.5) * dv : 0.0};
    double phi[5];
    phi[0] = 1.0;
    double v2 = 0.0;
    for (int a = 0; a < c->dv; ++a) { phi[1 + a] = v[a]; v2 += v[a] * v[a]; }
    phi[m - 1] = v2;
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) g[(size_t)i * m + j] += phi[i] * phi[j];
  }
  std::memset(c->Ginv, 0, sizeof(c->Ginv));
  invert(g, m, c->Ginv);
}

fks_status update_comm_lists(fks_ctx* c);

void free_chunk_lists(fks_ctx* c) {
  for (int* p : c->d_chunk_fluid) cudaFree(p);
  for (int* p : c->d_chunk_solid) cudaFree(p);
  c->d_chunk_fluid.clear();
  c->d_chunk_solid.clear();
  c->n_chunk_fluid.clear();
  c->n_chunk_solid.clear();
  c->chunk_first.clear();
}

fks_status set_cell_lists(fks_ctx* c, const uint8_t* solid_host) {
  free_chunk_lists(c);
  if (solid_host) c->h_solid.assign(solid_host, solid_host + c->ncells);
  else c->h_solid.clear();
  std::vector<int> fluid, solid;
  for (int64_t i = 0; i < c->ncells; ++i) {
    if (solid_host && solid_host[i]) solid.push_back((int)i); else fluid.push_back((int)i);
  }
  cudaFree(c->d_fluid); cudaFree(c->d_solid_list); cudaFree(c->d_solid);
  c->d_fluid = nullptr; c->d_solid_list = nullptr; c->d_solid = nullptr;
  c->nfluid = (int)fluid.size();
  c->nsolid = (int)solid.size();
  if (!fluid.empty()) {
    if (cudaMalloc(&c->d_fluid, fluid.size() * sizeof(int)) != cudaSuccess) return FKS_E_NOMEM;
    cudaMemcpy(c->d_fluid, fluid.data(), fluid.size() * sizeof(int), cudaMemcpyHostToDevice);
  }
  if (!solid.empty()) {
    if (cudaMalloc(&c->d_solid_list, solid.size() * sizeof(int)) != cudaSuccess) return FKS_E_NOMEM;
    cudaMemcpy(c->d_solid_list, solid.data(), solid.size() * sizeof(int), cudaMemcpyHostToDevice);
    if (cudaMalloc(&c->d_solid, c->ncells) != cudaSuccess) return FKS_E_NOMEM;
    cudaMemcpy(c->d_solid, solid_host, c->ncells, cudaMemcpyHostToDevice);
  }
  fks_status st = update_comm_lists(c);
  if (st != FKS_OK) return st;
  return cuda_fail(cudaGetLastError());
}

// a2: fluid cells split into those on a HALO-face plane of the slab axis (they may read a neighbour
// plane, CFL <= 1) and the interior, so the interior runs while the exchange is in flight.
fks_status update_comm_lists(fks_ctx* c) {
  cudaFree(c->d_interior); cudaFree(c->d_boundary);
  c->d_interior = c->d_boundary = nullptr;
  c->ninterior = c->nboundary = 0;
  if (c->comm_kind == 0) return FKS_OK;
  const int a = c->grid.dx - 1;
  const int64_t Ma = c->grid.M[a];
  std::vector<int> in, bd;
  for (int64_t i = 0; i < c->ncells; ++i) {
    if (!c->h_solid.empty() && c->h_solid[i]) continue;
    const int64_t ja = i / c->pc;  // slab axis = slowest axis
    const bool edge = (c->peer[0] >= 0 && ja == 0) || (c->peer[1] >= 0 && ja == Ma - 1);
    (edge ? bd : in).push_back((int)i);
  }
  c->ninterior = (int)in.size();
  c->nboundary = (int)bd.size();
  if (!in.empty()) {
    if (cudaMalloc(&c->d_interior, in.size() * sizeof(int)) != cudaSuccess) return FKS_E_NOMEM;
    cudaMemcpy(c->d_interior, in.data(), in.size() * sizeof(int), cudaMemcpyHostToDevice);
  }
  if (!bd.empty()) {
    if (cudaMalloc(&c->d_boundary, bd.size() * sizeof(int)) != cudaSuccess) return FKS_E_NOMEM;
    cudaMemcpy(c->d_boundary, bd.data(), bd.size() * sizeof(int), cudaMemcpyHostToDevice);
  }
  return FKS_OK;
}

// Returns FKS_E_UNSUPPORTED when a shift along the slab axis exceeds one cell while that axis has a
// HALO face: the neighbour rank sends exactly one plane (halo width 1 at CFL <= 1, reading #15), so a
// source two planes away would silently read the wrong plane.
fks_status fill_transport(const fks_ctx* c, fks::TransportParams* tp, bool with_shift, int64_t half = -1) {
  std::memset(tp, 0, sizeof(*tp));
  tp->dx = with_shift ? c->grid.dx : 0;
  for (int a = 0; a < 3; ++a) tp->M[a] = (int)c->grid.M[a];
  for (int f = 0; f < 6; ++f) { tp->bc[f] = c->grid.bc[f]; tp->ghost[f] = c->d_ghost[f]; }
  tp->halo[0] = c->comm_kind ? c->d_halo[0] : c->halo[0];  // library-owned planes when a comm is set
  tp->halo[1] = c->comm_kind ? c->d_halo[1] : c->halo[1];
  if (with_shift)
    for (int a = 0; a < c->grid.dx; ++a) {
      if (half >= 0) shift_delta_half(half, c->N, c->L, c->dt, c->grid.h, tp->delta[a]);
      else shift_delta(c->step_n, c->N, c->L, c->dt, c->grid.h, tp->delta[a]);
    }
  tp->solid = c->d_solid ? c->d_solid : c->d_zero_mask;
  // specular reflection needs solid cells somewhere: local ones, or (partitioned) the neighbours'
  tp->reflect = (c->reflect && with_shift && (c->d_solid || (c->comm_kind && c->d_zero_mask))) ? 1 : 0;
  tp->halo_solid[0] = c->comm_kind && c->reflect ? c->d_halo_solid[0] : nullptr;
  tp->halo_solid[1] = c->comm_kind && c->reflect ? c->d_halo_solid[1] : nullptr;
  tp->Nv = c->N;
  tp->ncells_total = c->ncells;
  tp->plane_cells = 1;
  for (int b = 0; b + 1 < c->grid.dx; ++b) tp->plane_cells *= c->grid.M[b];
  tp->cfl1 = 1;
  for (int a = 0; a < 3; ++a)
    for (int k = 0; k < fks::kMaxN; ++k) tp->cfl1 &= tp->delta[a][k] >= -1 && tp->delta[a][k] <= 1;
  if (with_shift && c->grid.dx > 0) {
    const int a = c->grid.dx - 1;  // HALO faces exist only on the slowest axis
    if (c->grid.bc[2 * a] == FKS_BC_HALO || c->grid.bc[2 * a + 1] == FKS_BC_HALO)
      for (int k = 0; k < c->N; ++k)
        if (tp->delta[a][k] < -1 || tp->delta[a][k] > 1) return FKS_E_UNSUPPORTED;
  }
  return FKS_OK;
}

fks::StepParams base_params(fks_ctx* c, const double* f_in, double* f_out, int mode) {
  fks::StepParams p;
  std::memset(&p, 0, sizeof(p));
  p.f_in = f_in;
  p.f_out = f_out;
  p.tables = c->d_tables;
  p.table_elems = c->table_elems;
  p.scratch = c->d_scratch;
  p.sync = c->d_sync;
  p.nonfinite = c->d_flag;
  p.A = c->A;
  p.mode = mode;
  p.project = c->project;
  p.dt_tau = c->dt / c->tau;
  p.L = c->L;
  p.dv = 2.0 * c->L / c->N;
  std::memcpy(p.Ginv, c->Ginv, sizeof(p.Ginv));
  return p;
}

fks_status run_collision(fks_ctx* c, fks::StepParams& p) {
  if (p.ncells == 0) return FKS_OK;
  cudaError_t e;
  if (c->N == 4) {
    e = fks::launch_step_small(c->N, c->dv, p, c->sm_count, c->stream);
  } else if (c->dv == 3 && c->N == 64) {
    const int ncl = std::min<int64_t>(p.ncells, c->nclusters);
    e = cudaMemsetAsync(c->d_sync, 0, (size_t)ncl * fks::sync_bytes3d64(), c->stream);
    if (e == cudaSuccess) e = fks::launch_step3d64(p, ncl, c->stream);
  } else if (c->dv == 3) {
    const int ncl = std::min<int64_t>(p.ncells, c->nclusters);
    e = cudaMemsetAsync(c->d_sync, 0, (size_t)ncl * fks::sync_bytes3d(), c->stream);
    if (e == cudaSuccess) e = fks::launch_step3d(c->N, p, ncl, c->stream);
  } else {
    const bool pair = fks::use_pair2d(c->N, c->A);
    const int per = pair ? fks::cells_per_block2d_pair(c->N) : fks::cells_per_block2d(c->N);
    const int64_t need = (p.ncells + per - 1) / per;
    const int nb = (int)std::min<int64_t>(need, (int64_t)c->sm_count);
    e = pair ? fks::launch_step2d_pair(c->N, p, nb, c->stream) : fks::launch_step2d(c->N, p, nb, c->stream);
  }
  c->launches++;
  return cuda_fail(e);
}

// Velocity nodes per axis: 4, 8, 16, 32, 64 in 2D and 3D (4 <= N <= 64; the paper
// quotes 8-64 per axis; 3D N = 64 runs kernels3d64.cu, N = 4 kernels_small.cu).
bool valid_N(int N, int dv) { (void)dv; return N == 4 || N == 8 || N == 16 || N == 32 || N == 64; }

}  // namespace

// ------------------------------------------------------------------ a2: slab halo exchange
// NCCL is resolved at run time (the copy torch already loaded, else the system libnccl.so.2), so
// libfks has no link-time NCCL dependency and builds without a GPU.
namespace {
struct NcclApi {
  decltype(&ncclGetUniqueId) getUniqueId;
  decltype(&ncclCommInitRank) commInitRank;
  decltype(&ncclCommDestroy) commDestroy;
  decltype(&ncclGroupStart) groupStart;
  decltype(&ncclGroupEnd) groupEnd;
  decltype(&ncclSend) send;
  decltype(&ncclRecv) recv;
};

const NcclApi* nccl_api() {
  static NcclApi api;
  static int state = 0;  // 0 untried, 1 ok, -1 unavailable
  if (state == 0) {
    state = -1;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
      api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
      api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
      api.groupStart = (decltype(api.groupStart))dlsym(h, "ncclGroupStart");
      api.groupEnd = (decltype(api.groupEnd))dlsym(h, "ncclGroupEnd");
      api.send = (decltype(api.send))dlsym(h, "ncclSend");
      api.recv = (decltype(api.recv))dlsym(h, "ncclRecv");
      if (api.getUniqueId && api.commInitRank && api.commDestroy && api.groupStart && api.groupEnd && api.send &&
          api.recv)
        state = 1;
    }
  }
  return state == 1 ? &api : nullptr;
}

// The velocity slices k_a a step moves across the slab faces: `down` (delta = +1: the lower rank's
// cells read one plane up, i.e. my first plane) and `up` (delta = -1).  false if |delta| > 1.
bool halo_plan(int64_t n, int N, double L, double dt, double h, fks::SliceList* down, fks::SliceList* up) {
  int8_t d[fks::kMaxN];
  shift_delta(n, N, L, dt, h, d);
  down->n = up->n = 0;
  for (int k = 0; k < N; ++k) {
    if (d[k] < -1 || d[k] > 1) return false;  // halo width 1 (reading #15)
    if (d[k] > 0) down->k[down->n++] = (int8_t)k;
    if (d[k] < 0) up->k[up->n++] = (int8_t)k;
  }
  return true;
}

bool comm_active(const fks_ctx* c) { return c->comm_kind != 0 && (c->peer[0] >= 0 || c->peer[1] >= 0); }

// Neighbours, plane size and buffers for the slab axis a = dx - 1 (each rank keeps all
// velocities of its slab, ghost planes are exchanged every step).
fks_status comm_setup(fks_ctx* c, int rank, int nranks) {
  const int a = c->grid.dx - 1;
  c->rank = rank;
  c->nranks = nranks;
  c->pc = 1;
  for (int b = 0; b < a; ++b) c->pc *= c->grid.M[b];
  c->peer[0] = c->grid.bc[2 * a] == FKS_BC_HALO ? (rank - 1 + nranks) % nranks : -1;
  c->peer[1] = c->grid.bc[2 * a + 1] == FKS_BC_HALO ? (rank + 1) % nranks : -1;
  if (!c->s_comm && cudaStreamCreateWithFlags(&c->s_comm, cudaStreamNonBlocking) != cudaSuccess) return FKS_E_CUDA;
  for (cudaEvent_t* e : {&c->ev_ready, &c->ev_halo, &c->ev_packed})
    if (!*e && cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) return FKS_E_CUDA;
  const size_t bytes = (size_t)c->pc * c->n * sizeof(double);
  for (int f = 0; f < 2; ++f) {
    if (c->peer[f] < 0) continue;
    for (double** b : {&c->d_halo[f], &c->d_send[f], &c->d_recv[f]})
      if (!*b && cudaMalloc(b, bytes) != cudaSuccess) return FKS_E_NOMEM;
    if (!c->d_halo_solid[f]) {
      if (cudaMalloc(&c->d_halo_solid[f], (size_t)c->pc) != cudaSuccess) return FKS_E_NOMEM;
      cudaMemset(c->d_halo_solid[f], 0, (size_t)c->pc);
    }
  }
  if (!c->d_zero_mask) {  // a local all-fluid mask (also a zero plane to send) for contexts without solids
    if (cudaMalloc(&c->d_zero_mask, (size_t)c->ncells) != cudaSuccess) return FKS_E_NOMEM;
    cudaMemset(c->d_zero_mask, 0, (size_t)c->ncells);
  }
  c->posted = -1;
  return update_comm_lists(c);
}

size_t slice_elems(const fks_ctx* c, const fks::SliceList& sl) {
  return (size_t)c->pc * sl.n * (c->dv == 3 ? c->N * c->N : c->N);
}

// Pack and send this step's boundary planes: to the lower neighbour the slices k_a with delta > 0
// (its cells read one plane up), to the upper one those with delta < 0 -- only the velocities whose
// FKS shift crosses the face; receive the mirror sets into the halo planes.
fks_status halo_post_impl(fks_ctx* c, const double* f_in) {
  if (!comm_active(c) || c->posted == c->step_n) return FKS_OK;
  const int a = c->grid.dx - 1;
  fks::SliceList down{}, up{};
  if (!halo_plan(c->step_n, c->N, c->L, c->dt, c->grid.h, &down, &up)) return FKS_E_UNSUPPORTED;
  c->send_sl[0] = down;  // my first plane -> lower neighbour's hi halo
  c->send_sl[1] = up;    // my last plane  -> upper neighbour's lo halo
  c->recv_sl[0] = up;    // my lo halo <- lower neighbour's last plane
  c->recv_sl[1] = down;  // my hi halo <- upper neighbour's first plane
  if (cudaEventRecord(c->ev_ready, c->stream) != cudaSuccess ||
      cudaStreamWaitEvent(c->s_comm, c->ev_ready, 0) != cudaSuccess)
    return FKS_E_CUDA;
  const int64_t first[2] = {0, (c->grid.M[a] - 1) * c->pc};
  c->bytes_sent = 0;
  for (int f = 0; f < 2; ++f) {
    if (c->peer[f] < 0) continue;
    if (fks::launch_halo_pack(f_in, first[f], (int)c->pc, c->n, c->N, c->dv, a, c->send_sl[f], c->d_send[f], false,
                              c->s_comm) != cudaSuccess)
      return FKS_E_CUDA;
    c->launches++;
    c->bytes_sent += (int64_t)slice_elems(c, c->send_sl[f]) * 8;
  }
  if (c->comm_kind == 1) {
    const NcclApi* nc = nccl_api();
    if (!nc) return FKS_E_NCCL;
    // fixed issue order (data moving up before data moving down, sends before receives): with two
    // ranks on a periodic axis both neighbours are the same peer and NCCL matches in issue order
    bool ok = nc->groupStart() == ncclSuccess;
    if (c->peer[1] >= 0 && ok)
      ok = nc->send(c->d_send[1], slice_elems(c, c->send_sl[1]), ncclFloat64, c->peer[1], c->nccl, c->s_comm) == ncclSuccess;
    if (c->peer[0] >= 0 && ok)
      ok = nc->send(c->d_send[0], slice_elems(c, c->send_sl[0]), ncclFloat64, c->peer[0], c->nccl, c->s_comm) == ncclSuccess;
    if (c->peer[0] >= 0 && ok)
      ok = nc->recv(c->d_recv[0], slice_elems(c, c->recv_sl[0]), ncclFloat64, c->peer[0], c->nccl, c->s_comm) == ncclSuccess;
    if (c->peer[1] >= 0 && ok)
      ok = nc->recv(c->d_recv[1], slice_elems(c, c->recv_sl[1]), ncclFloat64, c->peer[1], c->nccl, c->s_comm) == ncclSuccess;
    if (c->reflect) {  // specular walls: the boundary planes' solid flags travel with the planes
      const uint8_t* mask = c->d_solid ? c->d_solid : c->d_zero_mask;
      if (c->peer[1] >= 0 && ok)
        ok = nc->send(mask + first[1], (size_t)c->pc, ncclUint8, c->peer[1], c->nccl, c->s_comm) == ncclSuccess;
      if (c->peer[0] >= 0 && ok)
        ok = nc->send(mask + first[0], (size_t)c->pc, ncclUint8, c->peer[0], c->nccl, c->s_comm) == ncclSuccess;
      if (c->peer[0] >= 0 && ok)
        ok = nc->recv(c->d_halo_solid[0], (size_t)c->pc, ncclUint8, c->peer[0], c->nccl, c->s_comm) == ncclSuccess;
      if (c->peer[1] >= 0 && ok)
        ok = nc->recv(c->d_halo_solid[1], (size_t)c->pc, ncclUint8, c->peer[1], c->nccl, c->s_comm) == ncclSuccess;
    }
    if (nc->groupEnd() != ncclSuccess || !ok) return FKS_E_NCCL;
    for (int f = 0; f < 2; ++f) {
      if (c->peer[f] < 0) continue;
      if (fks::launch_halo_pack(c->d_halo[f], 0, (int)c->pc, c->n, c->N, c->dv, a, c->recv_sl[f], c->d_recv[f], true,
                                c->s_comm) != cudaSuccess)
        return FKS_E_CUDA;
      c->launches++;
    }
    if (cudaEventRecord(c->ev_halo, c->s_comm) != cudaSuccess) return FKS_E_CUDA;
  } else if (cudaEventRecord(c->ev_packed, c->s_comm) != cudaSuccess) {
    return FKS_E_CUDA;
  }
  c->posted = c->step_n;
  return FKS_OK;
}

// Make the halo planes of this step visible to the context stream.  Loopback: pull the neighbours'
// packed planes (they must have posted this step) with device copies, unpack, and finish before
// returning so a neighbour's next post cannot overwrite its send buffer under the copy.
fks_status halo_wait_impl(fks_ctx* c) {
  if (!comm_active(c)) return FKS_OK;
  if (c->posted != c->step_n) return FKS_E_STATE;
  if (c->comm_kind == 2) {
    const int a = c->grid.dx - 1;
    for (int f = 0; f < 2; ++f) {
      if (c->peer[f] < 0) continue;
      fks_ctx* q = c->loop->ctx[c->peer[f]];
      if (!q || q->posted != c->step_n) return FKS_E_STATE;
      if (cudaStreamWaitEvent(c->s_comm, q->ev_packed, 0) != cudaSuccess ||
          cudaMemcpyAsync(c->d_recv[f], q->d_send[1 - f], slice_elems(c, c->recv_sl[f]) * sizeof(double),
                          cudaMemcpyDeviceToDevice, c->s_comm) != cudaSuccess)
        return FKS_E_CUDA;
      if (fks::launch_halo_pack(c->d_halo[f], 0, (int)c->pc, c->n, c->N, c->dv, a, c->recv_sl[f], c->d_recv[f], true,
                                c->s_comm) != cudaSuccess)
        return FKS_E_CUDA;
      c->launches++;
      if (c->reflect) {  // the neighbour's boundary-plane solid flags (lo halo <- its last plane)
        const int64_t qfirst = f == 0 ? (q->grid.M[a] - 1) * q->pc : 0;
        const uint8_t* qmask = q->d_solid ? q->d_solid : q->d_zero_mask;
        cudaError_t e = qmask ? cudaMemcpyAsync(c->d_halo_solid[f], qmask + qfirst, (size_t)c->pc,
                                                cudaMemcpyDeviceToDevice, c->s_comm)
                              : cudaMemsetAsync(c->d_halo_solid[f], 0, (size_t)c->pc, c->s_comm);
        if (e != cudaSuccess) return FKS_E_CUDA;
      }
    }
    if (cudaEventRecord(c->ev_halo, c->s_comm) != cudaSuccess || cudaStreamSynchronize(c->s_comm) != cudaSuccess)
      return FKS_E_CUDA;
  }
  return cuda_fail(cudaStreamWaitEvent(c->stream, c->ev_halo, 0));
}

// Loopback: every neighbour must have posted this step before anything is enqueued here.
fks_status loop_peers_posted(const fks_ctx* c) {
  if (c->comm_kind != 2) return FKS_OK;
  for (int f = 0; f < 2; ++f) {
    if (c->peer[f] < 0) continue;
    const fks_ctx* q = c->loop->ctx[c->peer[f]];
    if (!q || q->posted != c->step_n) return FKS_E_STATE;
  }
  return FKS_OK;
}

fks_status halo_sync(fks_ctx* c, const double* f_in) {
  fks_status st = halo_post_impl(c, f_in);
  if (st == FKS_OK) st = loop_peers_posted(c);
  return st != FKS_OK ? st : halo_wait_impl(c);
}
}  // namespace

extern "C" {

const char* fks_strerror(fks_status s) {
  switch (s) {
    case FKS_OK: return "ok";
    case FKS_E_INVAL: return "invalid argument";
    case FKS_E_UNSUPPORTED: return "unsupported configuration";
    case FKS_E_NOMEM: return "out of device memory";
    case FKS_E_CUDA: return "CUDA error (no sm_100 device, launch failure or asynchronous fault)";
    case FKS_E_NCCL: return "NCCL error";
    case FKS_E_NONFINITE: return "non-finite value produced by a step";
    case FKS_E_STATE: return "invalid state (dt changed mid-run or call out of order)";
  }
  return "unknown status";
}

fks_status fks_host_tables(int dv, int Nv, double L, int M_dirs, double R, double kernel_const, double kernel_gamma,
                           double* alpha_host, double* alphap_host, double* D_host, double* w_host, double* e_host,
                           double* scale) {
  if ((dv != 2 && dv != 3) || !valid_N(Nv, dv) || !(L > 0)) return FKS_E_INVAL;
  if (!valid_gamma(kernel_gamma)) return FKS_E_UNSUPPORTED;
  Dirs d;
  if (!default_dirs(dv, M_dirs, &d)) return FKS_E_UNSUPPORTED;
  if (!(R > 0)) R = 2.0 * kLambda * kPi;
  if (!(kernel_const > 0)) kernel_const = default_kconst(dv);
  std::vector<double> al, alp, D;
  build_tables(dv, Nv, R, kernel_gamma, d, al, alp, D);
  if (alpha_host) std::memcpy(alpha_host, al.data(), al.size() * sizeof(double));
  if (alphap_host) std::memcpy(alphap_host, alp.data(), alp.size() * sizeof(double));
  if (D_host) std::memcpy(D_host, D.data(), D.size() * sizeof(double));
  if (w_host) std::memcpy(w_host, d.w.data(), d.w.size() * sizeof(double));
  if (e_host) std::memcpy(e_host, d.e.data(), d.e.size() * sizeof(double));
  if (scale) *scale = node_scale(dv, L, kernel_const, kernel_gamma);
  return FKS_OK;
}

fks_status fks_host_halo_slices(int64_t n, int Nv, double L, double dt, double h, int8_t* to_lower, int* n_lower,
                                int8_t* to_upper, int* n_upper) {
  if (Nv <= 0 || Nv > fks::kMaxN || !(L > 0) || !(h > 0) || n < 0 || !to_lower || !to_upper || !n_lower || !n_upper)
    return FKS_E_INVAL;
  fks::SliceList down{}, up{};
  if (!halo_plan(n, Nv, L, dt, h, &down, &up)) return FKS_E_UNSUPPORTED;
  for (int i = 0; i < down.n; ++i) to_lower[i] = down.k[i];
  for (int i = 0; i < up.n; ++i) to_upper[i] = up.k[i];
  *n_lower = down.n;
  *n_upper = up.n;
  return FKS_OK;
}

fks_status fks_host_shift(int64_t n, int Nv, double L, double dt, double h, int8_t* delta_host) {
  if (Nv <= 0 || Nv > fks::kMaxN || !(L > 0) || !(h > 0) || !delta_host || n < 0) return FKS_E_INVAL;
  shift_delta(n, Nv, L, dt, h, delta_host);
  return FKS_OK;
}

fks_status fks_init(const fks_grid* grid, int Nv, double L, int M_dirs, double kernel_gamma, fks_ctx** out) {
  if (!grid || !out) return FKS_E_INVAL;
  *out = nullptr;
  const int dv = grid->dv;
  if ((dv != 2 && dv != 3) || !valid_N(Nv, dv) || !(L > 0) || grid->dx < 0 || grid->dx > 3 || grid->dx > dv)
    return FKS_E_INVAL;
  if (!valid_gamma(kernel_gamma)) return FKS_E_UNSUPPORTED;  // NEXT-3: -1 < gamma <= 2 (reading #25)
  int64_t ncells = 1;
  const int axes = grid->dx == 0 ? 1 : grid->dx;
  for (int a = 0; a < axes; ++a) {
    if (grid->M[a] <= 0) return FKS_E_INVAL;
    ncells *= grid->M[a];
  }
  if (ncells > INT32_MAX) return FKS_E_INVAL;
  if (grid->dx > 0 && !(grid->h > 0)) return FKS_E_INVAL;
  for (int f = 0; f < 2 * grid->dx; ++f) {
    if (grid->bc[f] < 0 || grid->bc[f] > 3) return FKS_E_INVAL;
    if (grid->bc[f] == 3 && f / 2 != grid->dx - 1) return FKS_E_INVAL;  // HALO: slowest axis only
  }
  Dirs dirs;
  if (!default_dirs(dv, M_dirs, &dirs)) return FKS_E_UNSUPPORTED;

  int dev = 0;
  cudaDeviceProp prop;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return FKS_E_CUDA;
  if (prop.major != 10) return FKS_E_CUDA;  // built for sm_100a only

  fks_ctx* c = new (std::nothrow) fks_ctx();
  if (!c) return FKS_E_NOMEM;
  c->grid = *grid;
  if (grid->dx == 0) {
    c->grid.M[1] = c->grid.M[2] = 1;
  } else {
    for (int a = grid->dx; a < 3; ++a) c->grid.M[a] = 1;
  }
  c->dv = dv;
  c->N = Nv;
  c->n = dv == 3 ? Nv * Nv * Nv : Nv * Nv;
  c->L = L;
  c->h = grid->h;
  c->gamma = kernel_gamma;
  c->kconst = default_kconst(dv);
  c->R = 2.0 * kLambda * kPi;
  c->dirs = dirs;
  c->A = (int)dirs.w.size();
  c->ncells = ncells;
  c->sm_count = prop.multiProcessorCount;
  fks_status st = upload_tables(c);
  if (st == FKS_OK) {
    build_gram(c);
    if (cudaMalloc(&c->d_flag, sizeof(int)) != cudaSuccess) st = FKS_E_NOMEM;
    else cudaMemset(c->d_flag, 0, sizeof(int));
  }
  if (st == FKS_OK && Nv == 4) {
    c->nclusters = c->sm_count * 8;  // kernels_small.cu: no groups; the round size of fks_step_host
  } else if (st == FKS_OK && dv == 3) {
    c->nclusters = Nv == 64 ? fks::max_groups3d64() : fks::max_active_clusters3d(Nv);
    if (const char* e = getenv("FKS_MAX_CLUSTERS")) {  // development: scaling with the cluster count
      const int m = atoi(e);
      if (m > 0 && m < c->nclusters) c->nclusters = m;
    }
    if (getenv("FKS_VERBOSE")) fprintf(stderr, "fks: N=%d, %d resident CTA groups\n", Nv, c->nclusters);
    if (c->nclusters <= 0) st = FKS_E_CUDA;
    else if (cudaMalloc(&c->d_scratch, (size_t)c->nclusters * (Nv == 64 ? fks::scratch_elems3d64() : fks::scratch_elems3d(Nv)) *
                                           sizeof(double2)) != cudaSuccess ||
             cudaMalloc(&c->d_sync, (size_t)c->nclusters * (Nv == 64 ? fks::sync_bytes3d64() : fks::sync_bytes3d())) !=
                 cudaSuccess)
      st = FKS_E_NOMEM;
  }
  if (st == FKS_OK) st = set_cell_lists(c, nullptr);
  if (st != FKS_OK) { fks_finalize(c); return st; }
  *out = c;
  return FKS_OK;
}

fks_status fks_set_params(fks_ctx* c, double tau, double kernel_const, double R, int project) {
  if (!c || !(tau > 0)) return FKS_E_INVAL;
  c->tau = tau;
  if (kernel_const > 0) c->kconst = kernel_const;
  if (R > 0) c->R = R;
  c->project = project ? 1 : 0;
  return upload_tables(c);
}

fks_status fks_set_dirs(fks_ctx* c, const double* e_host, const double* w_host, int M) {
  if (!c || !e_host || !w_host || M <= 0) return FKS_E_INVAL;
  Dirs d;
  d.e.assign(e_host, e_host + (size_t)M * c->dv);
  d.w.assign(w_host, w_host + M);
  c->dirs = d;
  c->A = M;
  return upload_tables(c);
}

fks_status fks_set_ghost(fks_ctx* c, int face, const double* ghost_f) {
  if (!c || face < 0 || face >= 6 || !ghost_f) return FKS_E_INVAL;
  if (!c->d_ghost[face] && cudaMalloc(&c->d_ghost[face], (size_t)c->n * sizeof(double)) != cudaSuccess)
    return FKS_E_NOMEM;
  return cuda_fail(cudaMemcpyAsync(c->d_ghost[face], ghost_f, (size_t)c->n * sizeof(double), cudaMemcpyDeviceToDevice,
                                   c->stream));
}

fks_status fks_set_halo(fks_ctx* c, const double* lo_plane, const double* hi_plane) {
  if (!c) return FKS_E_INVAL;
  c->halo[0] = lo_plane;
  c->halo[1] = hi_plane;
  return FKS_OK;
}

fks_status fks_set_specular(fks_ctx* c, int on) {
  if (!c) return FKS_E_INVAL;
  c->reflect = on ? 1 : 0;  // on a partitioned grid the library comm carries the neighbours' solid flags
  return FKS_OK;
}

fks_status fks_set_solid(fks_ctx* c, const uint8_t* solid_host) {
  if (!c) return FKS_E_INVAL;
  return set_cell_lists(c, solid_host);
}

fks_status fks_set_scheme(fks_ctx* c, int splitting, int integrator) {
  if (!c || (splitting != FKS_SPLIT_LIE && splitting != FKS_SPLIT_STRANG) ||
      (integrator != FKS_TIME_EULER && integrator != FKS_TIME_HEUN))
    return FKS_E_INVAL;
  if (splitting == FKS_SPLIT_STRANG)
    for (int f = 0; f < 2 * c->grid.dx; ++f)
      if (c->grid.bc[f] == FKS_BC_HALO) return FKS_E_UNSUPPORTED;
  c->split = splitting;
  c->integ = integrator;
  return FKS_OK;
}

// ---- peer memory (a2 fused into the gather) ----------------------------------
fks_status fks_ipc_get_handle(const void* dptr, void* handle_out, int64_t* offset_out) {
  if (!dptr || !handle_out || !offset_out) return FKS_E_INVAL;
  // the allocation containing dptr (a caching allocator hands out interior pointers): driver API,
  // dlopen'ed like NCCL so that libfks links the runtime only
  using GetRange = int (*)(unsigned long long*, size_t*, unsigned long long);
  static const GetRange get_range = []() -> GetRange {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    return h ? reinterpret_cast<GetRange>(dlsym(h, "cuMemGetAddressRange_v2")) : nullptr;
  }();
  if (!get_range) return FKS_E_CUDA;
  unsigned long long base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<unsigned long long>(dptr)) != 0) return FKS_E_INVAL;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)) != cudaSuccess) return FKS_E_CUDA;
  static_assert(sizeof(h) == FKS_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle_out, &h, sizeof(h));
  *offset_out = (int64_t)(reinterpret_cast<unsigned long long>(dptr) - base);
  return FKS_OK;
}

fks_status fks_ipc_open(const void* handle, void** base_out) {
  if (!handle || !base_out) return FKS_E_INVAL;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  return cuda_fail(cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess));
}

fks_status fks_ipc_close(void* base) {
  if (!base) return FKS_E_INVAL;
  return cuda_fail(cudaIpcCloseMemHandle(base));
}

fks_status fks_comm_unique_id(void* id_out) {
  if (!id_out) return FKS_E_INVAL;
  const NcclApi* nc = nccl_api();
  if (!nc) return FKS_E_NCCL;
  ncclUniqueId id;
  if (nc->getUniqueId(&id) != ncclSuccess) return FKS_E_NCCL;
  std::memcpy(id_out, &id, sizeof(id));
  return FKS_OK;
}

fks_status fks_set_comm(fks_ctx* c, const void* nccl_unique_id, int rank, int nranks) {
  if (!c || !nccl_unique_id || nranks < 1 || rank < 0 || rank >= nranks || c->grid.dx < 1 || c->comm_kind)
    return FKS_E_INVAL;
  const NcclApi* nc = nccl_api();
  if (!nc) return FKS_E_NCCL;
  ncclUniqueId id;
  std::memcpy(&id, nccl_unique_id, sizeof(id));
  if (nc->commInitRank(&c->nccl, nranks, id, rank) != ncclSuccess) return FKS_E_NCCL;
  c->comm_kind = 1;
  return comm_setup(c, rank, nranks);
}

fks_status fks_comm_loopback_create(int nranks, fks_loopback** out) {
  if (!out || nranks < 1) return FKS_E_INVAL;
  fks_loopback* l = new (std::nothrow) fks_loopback();
  if (!l) return FKS_E_NOMEM;
  l->nranks = nranks;
  l->ctx.assign(nranks, nullptr);
  *out = l;
  return FKS_OK;
}

fks_status fks_comm_loopback_destroy(fks_loopback* l) {
  if (!l) return FKS_E_INVAL;
  for (fks_ctx* c : l->ctx)
    if (c) c->loop = nullptr, c->comm_kind = 0;
  delete l;
  return FKS_OK;
}

fks_status fks_set_comm_loopback(fks_ctx* c, fks_loopback* l, int rank) {
  if (!c || !l || rank < 0 || rank >= l->nranks || l->ctx[rank] || c->grid.dx < 1 || c->comm_kind)
    return FKS_E_INVAL;
  c->comm_kind = 2;
  c->loop = l;
  l->ctx[rank] = c;
  return comm_setup(c, rank, l->nranks);
}

fks_status fks_halo_post(fks_ctx* c, const double* f_in) {
  if (!c || !f_in) return FKS_E_INVAL;
  if (!comm_active(c)) return FKS_OK;
  if (!(c->dt > 0)) return FKS_E_STATE;  // dt is fixed by the first step / fks_set_state
  return halo_post_impl(c, f_in);
}

fks_status fks_get_comm_stats(const fks_ctx* c, int64_t* bytes_sent_last, int* interior_cells, int* boundary_cells) {
  if (!c) return FKS_E_INVAL;
  if (bytes_sent_last) *bytes_sent_last = c->bytes_sent;
  if (interior_cells) *interior_cells = c->ninterior;
  if (boundary_cells) *boundary_cells = c->nboundary;
  return FKS_OK;
}

fks_status fks_set_stream(fks_ctx* c, void* s) {
  if (!c) return FKS_E_INVAL;
  c->stream = (cudaStream_t)s;
  return FKS_OK;
}

// §8(b) in-place calls: with f_out == f_in the call writes a library-owned state-sized buffer
// (allocated on first use), then one device-to-device copy on the context stream moves it back.
static fks_status ensure_inplace(fks_ctx* c) {
  if (c->d_inplace) return FKS_OK;
  return cudaMalloc(&c->d_inplace, (size_t)c->ncells * c->n * sizeof(double)) == cudaSuccess ? FKS_OK
                                                                                                  : FKS_E_NOMEM;
}

extern "C++" {
template <typename Call>
static fks_status maybe_inplace(fks_ctx* c, const double* in, double* out, Call&& call) {
  if (in != out) return call(out);
  fks_status st = ensure_inplace(c);
  if (st != FKS_OK) return st;
  if ((st = call(c->d_inplace)) != FKS_OK) return st;
  return cuda_fail(cudaMemcpyAsync(out, c->d_inplace, (size_t)c->ncells * c->n * sizeof(double),
                                   cudaMemcpyDeviceToDevice, c->stream));
}
}

static fks_status collide_impl(fks_ctx* c, const double* f, double* Q) {
  fks::StepParams p = base_params(c, f, Q, 0);
  fill_transport(c, &p.tp, false);  // no shifts: cannot fail
  p.cell_list = nullptr;
  p.ncells = (int)c->ncells;
  return run_collision(c, p);
}

fks_status fks_collide(fks_ctx* c, const double* f, double* Q) {
  if (!c || !f || !Q) return FKS_E_INVAL;
  return maybe_inplace(c, f, Q, [&](double* out) { return collide_impl(c, f, out); });
}

static fks_status check_dt(fks_ctx* c, double dt) {
  if (!(dt > 0)) return FKS_E_INVAL;
  if ((c->reflect && !c->comm_kind) || (c->split == FKS_SPLIT_STRANG && c->grid.dx > 0))
    // caller-owned halo planes (fks_set_halo) carry no solid flags; Strang's second half transport
    // would need a second exchange of the collided state
    for (int f = 0; f < 2 * c->grid.dx; ++f)
      if (c->grid.bc[f] == FKS_BC_HALO) return FKS_E_UNSUPPORTED;
  for (int f = 0; f < 2 * c->grid.dx; ++f) {
    if (c->grid.bc[f] == FKS_BC_GHOST && !c->d_ghost[f]) return FKS_E_STATE;
    if (c->grid.bc[f] == FKS_BC_HALO && !(c->comm_kind ? c->d_halo[f & 1] : c->halo[f & 1])) return FKS_E_STATE;
  }
  if (c->dt == 0.0) c->dt = dt;
  else if (c->dt != dt) return FKS_E_STATE;
  return FKS_OK;
}

static fks_status transport_impl(fks_ctx* c, const double* f_in, double* f_out, double dt) {
  fks_status st = check_dt(c, dt);
  if (st != FKS_OK) return st;
  fks::TransportParams tp;
  st = fill_transport(c, &tp, true);
  if (st != FKS_OK) return st;
  if ((st = halo_sync(c, f_in)) != FKS_OK) return st;
  cudaError_t e = fks::launch_transport(f_in, f_out, tp, c->d_solid, c->ncells, c->n, c->N, c->dv, c->stream);
  c->launches++;
  if (e != cudaSuccess) return FKS_E_CUDA;
  c->step_n++;
  return FKS_OK;
}


static fks_status ensure_tmp(fks_ctx* c) {
  if (c->d_tmp) return FKS_OK;
  return cudaMalloc(&c->d_tmp, (size_t)c->ncells * c->n * sizeof(double)) == cudaSuccess ? FKS_OK : FKS_E_NOMEM;
}

// One collision pass over the fluid cells: mode 1 (f_out = f + dt/tau Pi Q(f)) or mode 2 (Heun stage,
// f_out = (base + f + dt/tau Pi Q(f)) / 2) with the given transport (shifted or none).
static fks_status collision_pass(fks_ctx* c, const double* in, double* out, int mode, const double* base,
                                 const fks::TransportParams& tp) {
  fks::StepParams p = base_params(c, in, out, mode);
  p.tp = tp;
  p.f_base = base;
  p.cell_list = c->nsolid ? c->d_fluid : nullptr;
  p.ncells = c->nfluid;
  return run_collision(c, p);
}

static fks_status transport_pass(fks_ctx* c, const double* in, double* out, const fks::TransportParams& tp) {
  cudaError_t e = fks::launch_transport(in, out, tp, c->d_solid, c->ncells, c->n, c->N, c->dv, c->stream);
  c->launches++;
  return cuda_fail(e);
}

static fks_status copy_solids(fks_ctx* c, const double* in, double* out) {
  if (!c->nsolid) return FKS_OK;
  cudaError_t e = fks::launch_copy_cells(in, out, c->d_solid_list, c->nsolid, c->n, c->stream);
  c->launches++;
  return cuda_fail(e);
}

// NEXT-4 step sequences (reading #26); all buffers distinct from f_in, the in-place passes are
// collision passes without transport (each cell reads only its own vector before writing it).
static fks_status step_scheme(fks_ctx* c, const double* f_in, double* f_out) {
  fks_status st = ensure_tmp(c);
  if (st != FKS_OK) return st;
  double* tmp = c->d_tmp;
  fks::TransportParams none, full, h1, h2;
  fill_transport(c, &none, false);
  const bool spatial = c->grid.dx > 0;
  const bool strang = c->split == FKS_SPLIT_STRANG && spatial;
  if (!strang) {  // Lie + Heun: f* = T f_in; f1 = E(f*); f_out = (f* + E(f1)) / 2
    const double* fstar = f_in;
    if (spatial) {
      if ((st = fill_transport(c, &full, true)) != FKS_OK) return st;
      if ((st = halo_sync(c, f_in)) != FKS_OK) return st;
      if ((st = transport_pass(c, f_in, tmp, full)) != FKS_OK) return st;
      fstar = tmp;
    }
    if ((st = copy_solids(c, f_in, f_out)) != FKS_OK) return st;
    if ((st = collision_pass(c, fstar, f_out, 1, nullptr, none)) != FKS_OK) return st;
    return collision_pass(c, f_out, f_out, 2, fstar, none);
  }
  if ((st = fill_transport(c, &h1, true, 2 * c->step_n)) != FKS_OK) return st;
  if ((st = fill_transport(c, &h2, true, 2 * c->step_n + 1)) != FKS_OK) return st;
  if (c->integ == FKS_TIME_EULER) {  // Strang + Euler: tmp = E(T_half f_in); f_out = T_half tmp
    if ((st = copy_solids(c, f_in, tmp)) != FKS_OK) return st;
    if ((st = collision_pass(c, f_in, tmp, 1, nullptr, h1)) != FKS_OK) return st;
    return transport_pass(c, tmp, f_out, h2);
  }
  // Strang + Heun: f* = T_half f_in (in f_out); tmp = E(f*); tmp = (f* + E(tmp)) / 2; f_out = T_half tmp
  if ((st = transport_pass(c, f_in, f_out, h1)) != FKS_OK) return st;
  if ((st = copy_solids(c, f_in, tmp)) != FKS_OK) return st;
  if ((st = collision_pass(c, f_out, tmp, 1, nullptr, none)) != FKS_OK) return st;
  if ((st = collision_pass(c, tmp, tmp, 2, f_out, none)) != FKS_OK) return st;
  return transport_pass(c, tmp, f_out, h2);
}

static fks_status step_impl(fks_ctx* c, const double* f_in, double* f_out, double dt) {
  fks_status st = check_dt(c, dt);
  if (st != FKS_OK) return st;
  if (c->integ != FKS_TIME_EULER || (c->split == FKS_SPLIT_STRANG && c->grid.dx > 0)) {
    st = step_scheme(c, f_in, f_out);
    if (st != FKS_OK) return st;
    c->step_n++;
    return FKS_OK;
  }
  fks::StepParams p = base_params(c, f_in, f_out, 1);
  st = fill_transport(c, &p.tp, true);
  if (st != FKS_OK) return st;
  if ((st = halo_post_impl(c, f_in)) != FKS_OK) return st;  // a2 on the communication stream
  if ((st = loop_peers_posted(c)) != FKS_OK) return st;
  if (c->nsolid) {
    if (fks::launch_copy_cells(f_in, f_out, c->d_solid_list, c->nsolid, c->n, c->stream) != cudaSuccess)
      return FKS_E_CUDA;
    c->launches++;
  }
  if (comm_active(c)) {
    // interior cells while the exchange is in flight, then the cells on the HALO-face planes
    p.cell_list = c->d_interior;
    p.ncells = c->ninterior;
    if ((st = run_collision(c, p)) != FKS_OK) return st;
    if ((st = halo_wait_impl(c)) != FKS_OK) return st;
    p.cell_list = c->d_boundary;
    p.ncells = c->nboundary;
    if ((st = run_collision(c, p)) != FKS_OK) return st;
    c->step_n++;
    return FKS_OK;
  }
  p.cell_list = c->nsolid ? c->d_fluid : nullptr;  // identity list: let the kernels prefetch
  p.ncells = c->nfluid;
  st = run_collision(c, p);
  if (st != FKS_OK) return st;
  c->step_n++;
  return FKS_OK;
}

static fks_status step_bgk_impl(fks_ctx* c, const double* f_in, double* f_out, double dt, int nu_rule, double mu) {
  if (nu_rule < FKS_NU_RHO || nu_rule > FKS_NU_EULER || (nu_rule == FKS_NU_CONST && !(mu > 0))) return FKS_E_INVAL;
  if (c->integ != FKS_TIME_EULER) return FKS_E_UNSUPPORTED;  // the BGK step is forward Euler only
  fks_status st = check_dt(c, dt);
  if (st != FKS_OK) return st;
  fks::BgkParams p;
  std::memset(&p, 0, sizeof(p));
  const bool strang = c->split == FKS_SPLIT_STRANG && c->grid.dx > 0;  // NEXT-4: T_half B T_half
  double* out1 = f_out;
  fks::TransportParams h2;
  if (strang) {
    if ((st = ensure_tmp(c)) != FKS_OK) return st;
    out1 = c->d_tmp;
    if ((st = fill_transport(c, &p.tp, true, 2 * c->step_n)) != FKS_OK) return st;
    if ((st = fill_transport(c, &h2, true, 2 * c->step_n + 1)) != FKS_OK) return st;
  } else {
    st = fill_transport(c, &p.tp, true);
    if (st != FKS_OK) return st;
  }
  if ((st = copy_solids(c, f_in, out1)) != FKS_OK) return st;
  p.f_in = f_in;
  p.f_out = out1;
  p.nonfinite = c->d_flag;
  p.cell_list = c->nsolid ? c->d_fluid : nullptr;
  p.ncells = c->nfluid;
  p.nu_rule = nu_rule;
  p.mu = mu;
  p.dt_tau = c->dt / c->tau;
  p.L = c->L;
  p.dv = 2.0 * c->L / c->N;
  std::memcpy(p.Ginv, c->Ginv, sizeof(p.Ginv));
  if ((st = halo_sync(c, f_in)) != FKS_OK) return st;
  cudaError_t e = fks::launch_bgk(c->N, c->dv, p, c->sm_count, c->stream);
  c->launches++;
  if (e != cudaSuccess) return FKS_E_CUDA;
  if (strang && (st = transport_pass(c, out1, f_out, h2)) != FKS_OK) return st;
  c->step_n++;
  return FKS_OK;
}

fks_status fks_transport(fks_ctx* c, const double* f_in, double* f_out, double dt) {
  if (!c || !f_in || !f_out) return FKS_E_INVAL;
  return maybe_inplace(c, f_in, f_out, [&](double* out) { return transport_impl(c, f_in, out, dt); });
}

fks_status fks_step(fks_ctx* c, const double* f_in, double* f_out, double dt) {
  if (!c || !f_in || !f_out) return FKS_E_INVAL;
  return maybe_inplace(c, f_in, f_out, [&](double* out) { return step_impl(c, f_in, out, dt); });
}

fks_status fks_step_bgk(fks_ctx* c, const double* f_in, double* f_out, double dt, int nu_rule, double mu) {
  if (!c || !f_in || !f_out) return FKS_E_INVAL;
  return maybe_inplace(c, f_in, f_out, [&](double* out) { return step_bgk_impl(c, f_in, out, dt, nu_rule, mu); });
}

// fks_step_host for independent cells (dx = 0, no solids): the batch is cut into chunks and
// chunk i's step overlaps the host->device copy of chunk i+1 and the device->host copy of
// chunk i-1 (two copy streams + events; PCIe is full duplex), so the end-to-end time tends to
// the slowest of the three instead of their sum.
static fks_status step_host_pipelined(fks_ctx* c, const double* f_in_host, double* f_out_host, double dt) {
  fks_status st = check_dt(c, dt);
  if (st != FKS_OK) return st;
  const int64_t n = c->n;
  const int64_t per_round = (c->dv == 3 || c->N == 4) ? (int64_t)std::max(1, c->nclusters)
                                       : (int64_t)c->sm_count * (fks::use_pair2d(c->N, c->A) ? fks::cells_per_block2d_pair(c->N)
                                                                                          : fks::cells_per_block2d(c->N));
  // FKS_HOST_CHUNKS: pipeline depth (C2: 12 chunks 25.6 ms, 32: 24.6 ms; PCIe-bound), read once
  static const int64_t nchunks = [] {
    const char* e = getenv("FKS_HOST_CHUNKS");
    return e ? (int64_t)std::max(1, atoi(e)) : (int64_t)32;
  }();
  int64_t chunk = std::max<int64_t>(per_round * 2, (c->ncells + nchunks - 1) / nchunks);
  chunk = (chunk + per_round - 1) / per_round * per_round;  // whole rounds of the persistent grid
  const int nch = (int)((c->ncells + chunk - 1) / chunk);
  if (!c->s_h2d) {
    if (cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking) != cudaSuccess)
      return FKS_E_CUDA;
  }
  while ((int)c->ev_in.size() < nch) {
    cudaEvent_t a, b;
    if (cudaEventCreateWithFlags(&a, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&b, cudaEventDisableTiming) != cudaSuccess)
      return FKS_E_CUDA;
    c->ev_in.push_back(a);
    c->ev_out.push_back(b);
  }
  cudaEvent_t start;  // the copies must not overtake work already queued on the context stream
  if (cudaEventCreateWithFlags(&start, cudaEventDisableTiming) != cudaSuccess) return FKS_E_CUDA;
  cudaEventRecord(start, c->stream);
  cudaStreamWaitEvent(c->s_h2d, start, 0);
  cudaStreamWaitEvent(c->s_d2h, start, 0);
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < nch && e == cudaSuccess; ++i) {
    const int64_t off = (int64_t)i * chunk, cnt = std::min(chunk, c->ncells - off);
    const size_t bytes = (size_t)cnt * n * sizeof(double);
    e = cudaMemcpyAsync(c->d_host_in + off * n, f_in_host + off * n, bytes, cudaMemcpyHostToDevice, c->s_h2d);
    if (e == cudaSuccess) e = cudaEventRecord(c->ev_in[i], c->s_h2d);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->stream, c->ev_in[i], 0);
    if (e != cudaSuccess) break;
    fks::StepParams p = base_params(c, c->d_host_in + off * n, c->d_host_out + off * n, 1);
    fill_transport(c, &p.tp, true);  // dx = 0: no shifts, cannot fail
    p.cell_list = nullptr;
    p.ncells = (int)cnt;
    st = run_collision(c, p);
    if (st != FKS_OK) break;
    e = cudaEventRecord(c->ev_out[i], c->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->s_d2h, c->ev_out[i], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(f_out_host + off * n, c->d_host_out + off * n, bytes, cudaMemcpyDeviceToHost, c->s_d2h);
  }
  cudaEventDestroy(start);
  if (st != FKS_OK) return st;
  if (e != cudaSuccess) return FKS_E_CUDA;
  c->step_n++;
  if (cudaStreamSynchronize(c->s_d2h) != cudaSuccess) return FKS_E_CUDA;
  return cuda_fail(cudaStreamSynchronize(c->stream));
}

// fks_step_host on a spatial grid (dx > 0): the grid is cut into chunks of planes along the slowest
// axis; chunk i's step needs its own planes and the first plane of chunk i+1 (shifts of one cell at
// CFL <= 1), so it starts as soon as those host->device copies landed, and its device->host copy
// overlaps the following chunks' copies and steps.  Bitwise the one-shot path (same kernels per
// cell).  Falls back when the slab axis is periodic or a HALO face (the first chunk would need the
// last), with a comm, with CFL > 1 along the slab axis, or with a non-default time scheme.
static fks_status step_host_spatial(fks_ctx* c, const double* f_in_host, double* f_out_host, double dt, bool* done) {
  *done = false;
  const int a = c->grid.dx - 1;
  const int64_t Ma = c->grid.M[a];
  const int64_t pc = c->ncells / Ma;
  if (c->grid.bc[2 * a] == FKS_BC_PERIODIC || c->grid.bc[2 * a + 1] == FKS_BC_PERIODIC ||
      c->grid.bc[2 * a] == FKS_BC_HALO || c->grid.bc[2 * a + 1] == FKS_BC_HALO || c->comm_kind ||
      c->integ != FKS_TIME_EULER || c->split != FKS_SPLIT_LIE || Ma < 4)
    return FKS_OK;
  fks_status st = check_dt(c, dt);
  if (st != FKS_OK) return st;
  fks::StepParams p = base_params(c, c->d_host_in, c->d_host_out, 1);
  if ((st = fill_transport(c, &p.tp, true)) != FKS_OK) return st;
  for (int k = 0; k < c->N; ++k)
    if (p.tp.delta[a][k] < -1 || p.tp.delta[a][k] > 1) return FKS_OK;  // needs more than one neighbour plane
  if (c->chunk_first.empty()) {  // chunk lists (fluid / solid cells per chunk of planes)
    const int64_t nch = std::min<int64_t>(16, Ma / 2);
    for (int64_t i = 0; i <= nch; ++i) c->chunk_first.push_back(Ma * i / nch);
    for (int64_t i = 0; i < nch; ++i) {
      std::vector<int> fl, so;
      for (int64_t cell = c->chunk_first[i] * pc; cell < c->chunk_first[i + 1] * pc; ++cell)
        ((!c->h_solid.empty() && c->h_solid[cell]) ? so : fl).push_back((int)cell);
      int *dfl = nullptr, *dso = nullptr;
      if (!fl.empty()) {
        if (cudaMalloc(&dfl, fl.size() * sizeof(int)) != cudaSuccess) return FKS_E_NOMEM;
        cudaMemcpy(dfl, fl.data(), fl.size() * sizeof(int), cudaMemcpyHostToDevice);
      }
      if (!so.empty()) {
        if (cudaMalloc(&dso, so.size() * sizeof(int)) != cudaSuccess) return FKS_E_NOMEM;
        cudaMemcpy(dso, so.data(), so.size() * sizeof(int), cudaMemcpyHostToDevice);
      }
      c->d_chunk_fluid.push_back(dfl);
      c->d_chunk_solid.push_back(dso);
      c->n_chunk_fluid.push_back((int)fl.size());
      c->n_chunk_solid.push_back((int)so.size());
    }
  }
  const int nch = (int)c->chunk_first.size() - 1;
  if (!c->s_h2d) {
    if (cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking) != cudaSuccess)
      return FKS_E_CUDA;
  }
  while ((int)c->ev_in.size() < nch) {
    cudaEvent_t e1, e2;
    if (cudaEventCreateWithFlags(&e1, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e2, cudaEventDisableTiming) != cudaSuccess)
      return FKS_E_CUDA;
    c->ev_in.push_back(e1);
    c->ev_out.push_back(e2);
  }
  cudaEvent_t start;
  if (cudaEventCreateWithFlags(&start, cudaEventDisableTiming) != cudaSuccess) return FKS_E_CUDA;
  cudaEventRecord(start, c->stream);
  cudaStreamWaitEvent(c->s_h2d, start, 0);
  cudaStreamWaitEvent(c->s_d2h, start, 0);
  const int64_t n = c->n;
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < nch && e == cudaSuccess; ++i) {  // all copies in, chunk by chunk
    const int64_t off = c->chunk_first[i] * pc * n, cnt = (c->chunk_first[i + 1] - c->chunk_first[i]) * pc * n;
    e = cudaMemcpyAsync(c->d_host_in + off, f_in_host + off, (size_t)cnt * sizeof(double), cudaMemcpyHostToDevice,
                        c->s_h2d);
    if (e == cudaSuccess) e = cudaEventRecord(c->ev_in[i], c->s_h2d);
  }
  for (int i = 0; i < nch && e == cudaSuccess && st == FKS_OK; ++i) {
    // chunk i reads its planes and the first plane of chunk i + 1
    e = cudaStreamWaitEvent(c->stream, c->ev_in[std::min(i + 1, nch - 1)], 0);
    if (e == cudaSuccess && c->n_chunk_solid[i]) {
      e = fks::launch_copy_cells(c->d_host_in, c->d_host_out, c->d_chunk_solid[i], c->n_chunk_solid[i], c->n, c->stream);
      c->launches++;
    }
    if (e != cudaSuccess) break;
    p.cell_list = c->d_chunk_fluid[i];
    p.ncells = c->n_chunk_fluid[i];
    st = run_collision(c, p);
    if (st != FKS_OK) break;
    const int64_t off = c->chunk_first[i] * pc * n, cnt = (c->chunk_first[i + 1] - c->chunk_first[i]) * pc * n;
    e = cudaEventRecord(c->ev_out[i], c->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->s_d2h, c->ev_out[i], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(f_out_host + off, c->d_host_out + off, (size_t)cnt * sizeof(double), cudaMemcpyDeviceToHost,
                          c->s_d2h);
  }
  cudaEventDestroy(start);
  if (st != FKS_OK) return st;
  if (e != cudaSuccess) return FKS_E_CUDA;
  c->step_n++;
  *done = true;
  if (cudaStreamSynchronize(c->s_d2h) != cudaSuccess) return FKS_E_CUDA;
  return cuda_fail(cudaStreamSynchronize(c->stream));
}

fks_status fks_step_host(fks_ctx* c, const double* f_in_host, double* f_out_host, double dt) {
  if (!c || !f_in_host || !f_out_host) return FKS_E_INVAL;
  const size_t bytes = (size_t)c->ncells * c->n * sizeof(double);
  if (!c->d_host_in) {  // both buffers or neither: a half-allocated pair is never stored
    double *in = nullptr, *out = nullptr;
    if (cudaMalloc(&in, bytes) != cudaSuccess) return FKS_E_NOMEM;
    if (cudaMalloc(&out, bytes) != cudaSuccess) {
      cudaFree(in);
      return FKS_E_NOMEM;
    }
    c->d_host_in = in;
    c->d_host_out = out;
  }
  if (c->grid.dx == 0 && c->nsolid == 0 && c->integ == FKS_TIME_EULER)
    return step_host_pipelined(c, f_in_host, f_out_host, dt);
  if (c->grid.dx > 0) {
    bool done = false;
    fks_status st = step_host_spatial(c, f_in_host, f_out_host, dt, &done);
    if (st != FKS_OK || done) return st;
  }
  if (cudaMemcpyAsync(c->d_host_in, f_in_host, bytes, cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
    return FKS_E_CUDA;
  fks_status st = fks_step(c, c->d_host_in, c->d_host_out, dt);
  if (st != FKS_OK) return st;
  if (cudaMemcpyAsync(f_out_host, c->d_host_out, bytes, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess)
    return FKS_E_CUDA;
  return cuda_fail(cudaStreamSynchronize(c->stream));
}

fks_status fks_moments(fks_ctx* c, const double* f, double* rho, double* u, double* T) {
  if (!c || !f || !rho || !u || !T) return FKS_E_INVAL;
  cudaError_t e = fks::launch_moments(f, rho, u, T, c->ncells, c->N, c->dv, c->L, 2.0 * c->L / c->N, c->stream);
  c->launches++;
  return cuda_fail(e);
}

fks_status fks_get_state(fks_ctx* c, int64_t* n, double* dt) {
  if (!c) return FKS_E_INVAL;
  if (n) *n = c->step_n;
  if (dt) *dt = c->dt;
  return FKS_OK;
}

fks_status fks_set_state(fks_ctx* c, int64_t n, double dt) {
  if (!c || n < 0 || dt < 0) return FKS_E_INVAL;
  c->step_n = n;
  c->dt = dt;
  return FKS_OK;
}

fks_status fks_check(fks_ctx* c) {
  if (!c) return FKS_E_INVAL;
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) return FKS_E_CUDA;
  int flag = 0;
  if (cudaMemcpy(&flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return FKS_E_CUDA;
  if (flag) {
    cudaMemset(c->d_flag, 0, sizeof(int));
    return FKS_E_NONFINITE;
  }
  return FKS_OK;
}

int64_t fks_launch_count(const fks_ctx* c) { return c ? c->launches : -1; }

fks_status fks_finalize(fks_ctx* c) {
  if (!c) return FKS_E_INVAL;
  cudaFree(c->d_tables);
  cudaFree(c->d_scratch);
  cudaFree(c->d_sync);
  cudaFree(c->d_flag);
  cudaFree(c->d_fluid);
  cudaFree(c->d_solid_list);
  cudaFree(c->d_solid);
  for (auto& g : c->d_ghost) cudaFree(g);
  for (cudaEvent_t ev : c->ev_in) cudaEventDestroy(ev);
  for (cudaEvent_t ev : c->ev_out) cudaEventDestroy(ev);
  if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
  if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
  cudaFree(c->d_host_in);
  cudaFree(c->d_host_out);
  cudaFree(c->d_tmp);
  cudaFree(c->d_inplace);
  if (c->nccl) {
    if (c->s_comm) cudaStreamSynchronize(c->s_comm);  // no exchange in flight when the comm goes
    if (const NcclApi* nc = nccl_api()) nc->commDestroy(c->nccl);
  }
  if (c->loop)
    for (auto& q : c->loop->ctx)
      if (q == c) q = nullptr;
  for (int f = 0; f < 2; ++f) {
    cudaFree(c->d_halo[f]);
    cudaFree(c->d_send[f]);
    cudaFree(c->d_recv[f]);
  }
  cudaFree(c->d_interior);
  cudaFree(c->d_boundary);
  free_chunk_lists(c);
  cudaFree(c->d_halo_solid[0]);
  cudaFree(c->d_halo_solid[1]);
  cudaFree(c->d_zero_mask);
  for (cudaEvent_t e : {c->ev_ready, c->ev_halo, c->ev_packed})
    if (e) cudaEventDestroy(e);
  if (c->s_comm) cudaStreamDestroy(c->s_comm);
  delete c;
  return FKS_OK;
}

}  // extern "C"
