// Library-level C-ABI entry points.
#include "../../include/cdp_b200.h"
#include "host.h"

extern "C" const char *cdp_last_error(void) { return cdp::get_error(); }

extern "C" int cdp_version(void) { return 1; }

extern "C" int cdp_device_sm_count(void) {
    int n = 0;
    if (cdp::guarded([&] { n = cdp::num_sms(); }) != 0) return 0;
    return n;
}

// Temporary until the operator kernels land.
extern "C" int cdp_mlp_value_grad(int, const int64_t *, const double *, int, const double *, const double *,
                                  const int64_t *, int, int, double *, double *) {
    return cdp::guarded([] { throw cdp::CdpError("cdp_mlp_value_grad: not built yet"); });
}
extern "C" int cdp_quad_value_grad(int, int, const double *, const double *, int, const double *, double *, double *) {
    return cdp::guarded([] { throw cdp::CdpError("cdp_quad_value_grad: not built yet"); });
}
