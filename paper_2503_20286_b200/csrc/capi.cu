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

// ------------------------------------------------------------------ stage timing
// Optional CUDA-event timing of each kernel stage on the stream it runs on
// (bench.py reads it to compute roofline.achieved).  Off by default: zero cost.
#include <mutex>
#include <vector>

namespace temo {
namespace {
struct Slot {
    std::vector<cudaEvent_t> pending;  // begin/end pairs
    double ms = 0.0;
    int64_t calls = 0;
};
std::mutex g_mu;
bool g_on = false;
Slot g_slots[TEMO_STAGE_COUNT];
std::vector<cudaEvent_t> g_pool;

cudaEvent_t grab() {
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
}  // namespace

void stage_begin(int stage, cudaStream_t st) {
    if (!g_on) return;
    std::lock_guard<std::mutex> lk(g_mu);
    cudaEvent_t e = grab();
    cudaEventRecord(e, st);
    g_slots[stage].pending.push_back(e);
}

void stage_end(int stage, cudaStream_t st) {
    if (!g_on) return;
    std::lock_guard<std::mutex> lk(g_mu);
    cudaEvent_t e = grab();
    cudaEventRecord(e, st);
    g_slots[stage].pending.push_back(e);
}
}  // namespace temo

static const char *k_stage_names[TEMO_STAGE_COUNT] = {
    "rank_prep", "dom_bits", "peel", "normalize", "associate", "niche", "offspring",
    "evaluate", "hv_count", "hv_contrib", "hype_select", "moead", "gather", "misc", "offspring_apply", "apply_vec"};

extern "C" void temo_timing_enable(int on) {
    std::lock_guard<std::mutex> lk(temo::g_mu);
    temo::g_on = on != 0;
}

extern "C" const char *temo_timing_name(int stage) {
    return (stage >= 0 && stage < TEMO_STAGE_COUNT) ? k_stage_names[stage] : "";
}

extern "C" int temo_timing_read(double *ms_out, int64_t *calls_out, int reset) {
    std::lock_guard<std::mutex> lk(temo::g_mu);
    for (int s = 0; s < TEMO_STAGE_COUNT; ++s) {
        auto &sl = temo::g_slots[s];
        for (size_t k = 0; k + 1 < sl.pending.size(); k += 2) {
            cudaEventSynchronize(sl.pending[k + 1]);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, sl.pending[k], sl.pending[k + 1]);
            sl.ms += ms;
            sl.calls += 1;
            temo::g_pool.push_back(sl.pending[k]);
            temo::g_pool.push_back(sl.pending[k + 1]);
        }
        sl.pending.clear();
        ms_out[s] = sl.ms;
        calls_out[s] = sl.calls;
        if (reset) {
            sl.ms = 0.0;
            sl.calls = 0;
        }
    }
    return TEMO_STAGE_COUNT;
}
