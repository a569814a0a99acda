// Library-level C-ABI entry points.
#include "../../include/cdp_b200.h"
#include "host.h"

extern "C" const char *cdp_last_error(void) { return cdp::get_error(); }

extern "C" int cdp_version(void) { return 1; }

extern "C" int cdp_memcpy_d2h(void *dst, const void *src, size_t bytes) {
    return cdp::guarded([&] { CDP_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost)); });
}

extern "C" int cdp_set_device(int device) {
    return cdp::guarded([&] { CDP_CUDA(cudaSetDevice(device)); });
}

extern "C" int cdp_device_sm_count(void) {
    int n = 0;
    if (cdp::guarded([&] { n = cdp::num_sms(); }) != 0) return 0;
    return n;
}


// ---------------------------------------------------------------------------
// Coupled-quadratic fixture (ref training/_kernels.pyx:135-172): fp64, one CTA,
// same summation order as the reference (rows, then samples, then columns).
__global__ void quad_value_grad_kernel(int m, int p, const double *a, const double *theta, int batch,
                                       const double *targets, double *loss, double *grad, double *work) {
    double *z = work, *rsum = work + m;
    for (int r = threadIdx.x; r < m; r += blockDim.x) {
        double acc = 0.0;
        for (int c = 0; c < p; ++c) acc = __dadd_rn(acc, __dmul_rn(a[size_t(r) * p + c], theta[c]));
        z[r] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double l = 0.0;
        for (int r = 0; r < m; ++r) rsum[r] = 0.0;
        for (int s = 0; s < batch; ++s)
            for (int r = 0; r < m; ++r) {
                const double d = __dsub_rn(z[r], targets[size_t(s) * m + r]);
                l = __dadd_rn(l, __dmul_rn(d, d));
                rsum[r] = __dadd_rn(rsum[r], d);
            }
        *loss = l / (2.0 * m * batch);
    }
    __syncthreads();
    const double scale = 1.0 / (double(m) * batch);
    for (int c = threadIdx.x; c < p; c += blockDim.x) {
        double acc = 0.0;
        for (int r = 0; r < m; ++r) acc = __dadd_rn(acc, __dmul_rn(a[size_t(r) * p + c], rsum[r]));
        grad[c] = __dmul_rn(acc, scale);
    }
}

extern "C" int cdp_quad_value_grad(int m, int p, const double *a, const double *theta, int batch,
                                   const double *targets, double *loss_out, double *grad_out) {
    return cdp::guarded([&] {
        CDP_REQUIRE(m >= 1 && p >= 1 && batch >= 1, "empty quadratic problem");
        const size_t na = size_t(m) * p, nt = size_t(batch) * m;
        double *d = nullptr;
        const size_t total = na + p + nt + 1 + p + 2 * size_t(m);
        CDP_CUDA(cudaMalloc(&d, total * 8));
        double *da = d, *dth = da + na, *dt = dth + p, *dl = dt + nt, *dg = dl + 1, *dw = dg + p;
        try {
            CDP_CUDA(cudaMemcpy(da, a, na * 8, cudaMemcpyHostToDevice));
            CDP_CUDA(cudaMemcpy(dth, theta, size_t(p) * 8, cudaMemcpyHostToDevice));
            CDP_CUDA(cudaMemcpy(dt, targets, nt * 8, cudaMemcpyHostToDevice));
            quad_value_grad_kernel<<<1, 256>>>(m, p, da, dth, batch, dt, dl, dg, dw);
            CDP_CUDA(cudaGetLastError());
            CDP_CUDA(cudaMemcpy(loss_out, dl, 8, cudaMemcpyDeviceToHost));
            CDP_CUDA(cudaMemcpy(grad_out, dg, size_t(p) * 8, cudaMemcpyDeviceToHost));
        } catch (...) {
            cudaFree(d);
            throw;
        }
        CDP_CUDA(cudaFree(d));
    });
}
