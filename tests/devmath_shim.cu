// Host build of the CUDA path's per-face / per-cell arithmetic (spark_device.cuh)
// for CPU tests against the oracle (tests/test_devmath.py).  On the host the
// MUFU seeds are replaced by fp32 seeds; the Newton steps, the limiter, the
// reconstruction and the Riemann formulations are the same source as on the GPU.
#include "../paper_2401_03378_b200/csrc/spark_device.cuh"

using namespace spark::dev;

template <int NV, int RS>
static void rs_dispatch(int d, double g, const double* wl, const double* wr, double* f) {
    const double gm1i = 1.0 / (g - 1.0);
    if (d == 0) riemann<NV, RS, 0>(wl, wr, g, gm1i, f);
    else if (d == 1) riemann<NV, RS, 1>(wl, wr, g, gm1i, f);
    else riemann<NV, RS, 2>(wl, wr, g, gm1i, f);
}

extern "C" {
void shim_riemann(int kind, int nv, int d, double gamma, const double* wl, const double* wr, double* f) {
    if (nv == 3) kind ? rs_dispatch<3, 1>(d, gamma, wl, wr, f) : rs_dispatch<3, 0>(d, gamma, wl, wr, f);
    else if (nv == 4) kind ? rs_dispatch<4, 1>(d, gamma, wl, wr, f) : rs_dispatch<4, 0>(d, gamma, wl, wr, f);
    else kind ? rs_dispatch<5, 1>(d, gamma, wl, wr, f) : rs_dispatch<5, 0>(d, gamma, wl, wr, f);
}
double shim_minmod3(double a, double b, double c) { return minmod3(a, b, c); }

void shim_recon(int recon, const double* s, double* lo, double* hi) {
    if (recon == 0) recon_cell<0>(s, *lo, *hi);
    else if (recon == 1) recon_cell<1>(s, *lo, *hi);
    else if (recon == 3) recon_cell<3>(s, *lo, *hi);
    else if (recon == 4) recon_cell<4>(s, *lo, *hi);
    else recon_cell<2>(s, *lo, *hi);
}
double shim_minmod(double a, double b) { return minmod(a, b); }
double shim_rcp(double x) { return rcp(x); }
double shim_sqrt(double x) { return sqrt_fast(x); }
int shim_cons_to_prim(int nv, double gamma, const double* u, double* w) {
    if (nv == 3) return cons_to_prim<3>(u, w, gamma - 1.0);
    if (nv == 4) return cons_to_prim<4>(u, w, gamma - 1.0);
    return cons_to_prim<5>(u, w, gamma - 1.0);
}
}
