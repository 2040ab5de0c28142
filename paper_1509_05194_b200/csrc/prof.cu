// Opt-in per-kernel timing with CUDA events on the launching stream.
// bench.py enables it for the timed region and reads back per-kernel totals;
// with profiling off the hooks cost one branch.
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace da {

struct ProfRec {
    const char* name;
    cudaEvent_t a, b;
};

static bool g_prof_on = false;
bool prof_enabled() { return g_prof_on; }
static std::mutex g_prof_mu;
static std::vector<ProfRec> g_recs;
static std::vector<cudaEvent_t> g_free_events;

static cudaEvent_t take_event() {
    if (!g_free_events.empty()) {
        cudaEvent_t e = g_free_events.back();
        g_free_events.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

ProfScope::ProfScope(const char* name, cudaStream_t s) : name_(name), s_(s), a_(nullptr) {
    if (!g_prof_on) return;
    std::lock_guard<std::mutex> g(g_prof_mu);
    a_ = take_event();
    cudaEventRecord((cudaEvent_t)a_, s_);
}

ProfScope::~ProfScope() {
    if (!a_) return;
    std::lock_guard<std::mutex> g(g_prof_mu);
    cudaEvent_t b = take_event();
    cudaEventRecord(b, s_);
    g_recs.push_back({name_, (cudaEvent_t)a_, b});
}

}  // namespace da

extern "C" {

int da_prof_enable(int on) {
    da::g_prof_on = on != 0;
    return 0;
}

// Writes "name count total_ms\n" lines into buf (NUL-terminated) and clears the log.
int da_prof_collect(char* buf, int cap) {
    using namespace da;
    std::lock_guard<std::mutex> g(g_prof_mu);
    std::map<std::string, std::pair<long long, double>> agg;
    for (auto& r : g_recs) {
        cudaEventSynchronize(r.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        auto& x = agg[r.name];
        x.first += 1;
        x.second += ms;
        g_free_events.push_back(r.a);
        g_free_events.push_back(r.b);
    }
    g_recs.clear();
    std::string out;
    for (auto& kv : agg) {
        char line[256];
        snprintf(line, sizeof(line), "%s %lld %.6f\n", kv.first.c_str(), kv.second.first, kv.second.second);
        out += line;
    }
    if ((int)out.size() + 1 > cap) return fail_arg("prof buffer too small (%d bytes needed)", (int)out.size() + 1);
    memcpy(buf, out.c_str(), out.size() + 1);
    return 0;
}

}  // extern "C"
