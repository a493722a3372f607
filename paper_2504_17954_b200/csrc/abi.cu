// C-ABI plumbing: version, thread-local error strings, launch checks.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ivr_common.cuh"

namespace {
thread_local char g_err[512] = "";
}

namespace ivr {
int pdl_level() {
    static const int lvl = [] {
        const char *e = getenv("IVR_PDL");
        return e && e[0] >= '0' && e[0] <= '9' ? e[0] - '0' : 1;
    }();
    return lvl;
}

void set_error(const char *msg) {
    strncpy(g_err, msg, sizeof(g_err) - 1);
    g_err[sizeof(g_err) - 1] = 0;
}

int check_launch(const char *what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
        return IVR_ERR_CUDA;
    }
    return IVR_OK;
}
}  // namespace ivr

extern "C" int ivr_version(void) { return IVR_ABI_VERSION; }
extern "C" const char *ivr_last_error(void) { return g_err; }
