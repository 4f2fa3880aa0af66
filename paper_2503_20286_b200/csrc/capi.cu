// ABI version and error strings of the temo_b200 C interface.
#include "common.cuh"

extern "C" int temo_abi_version(void) { return 1; }

extern "C" const char *temo_strerror(int code) {
    switch (code) {
        case TEMO_OK: return "ok";
        case TEMO_EINVAL: return "invalid argument";
        case TEMO_ENAN: return "objective matrix contains NaN rows";
        case TEMO_ERUNTIME: return "runtime error";
        case TEMO_EWORKSPACE: return "workspace too small";
        case TEMO_ECUDA: return "CUDA error";
        default: return "unknown error";
    }
}
