// Host-side plan queries shared by the C ABI (pass counts, workspace sizes)
// and the field-dispatched pointwise multiply.
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>
#include <vector>
#include "launch.cuh"
namespace nttb200 {

// ---- launch window: may a single-pass launch defer its dependency wait? ----
// Every fast / tile / four-step kernel is launched with programmatic stream
// serialisation.  A fast-kernel launch whose buffers are disjoint from those of
// every launch that may still be running on its stream loads its first rows at
// once, under its predecessor's tail, and waits for the predecessor only at its
// end (fast.cuh k_fast, a.defer), so grids still complete in stream order.
// What may still be running when launch m starts: launch m - 1 and -- when
// m - 1 deferred its wait too -- whatever m - 1 could overlap: the run of
// deferred launches before m back to the waiting launch that started it (a
// waiting launch triggers its dependents after its wait, so nothing older
// overlaps them).  An EXCLUSIVE launch (one CTA per SM by shared memory, on
// every SM) cuts the run short: m starts only after every CTA of m - 1 has
// started, i.e. after every CTA of the launches before m - 1 has left its SM.
// Launches the window does not model (multi-pass, pointwise, distributed
// steps) end the run; the next single-pass launch waits at its start.
namespace {
struct LaunchSpan { const char *in0, *in1, *out0, *out1; bool exclusive; };
std::mutex g_run_mu;
std::map<std::pair<int, cudaStream_t>, std::vector<LaunchSpan>> g_runs;
constexpr size_t kMaxRun = 16;
inline bool overlap(const char* a0, const char* a1, const char* b0, const char* b1) { return a0 < b1 && b0 < a1; }
inline int current_device() { int d = 0; cudaGetDevice(&d); return d; }
}  // namespace

void window_break(cudaStream_t stream) {
    std::lock_guard<std::mutex> lk(g_run_mu);
    auto it = g_runs.find({current_device(), stream});
    if (it != g_runs.end()) it->second.clear();
}

bool window_admit(cudaStream_t stream, const void* in, const void* out, uint64_t bytes, bool exclusive) {
    static const bool on = [] { const char* e = getenv("NTT_PDL_DEFER"); return !e || atoi(e) != 0; }();
    const LaunchSpan me{static_cast<const char*>(in), static_cast<const char*>(in) + bytes,
                        static_cast<const char*>(out), static_cast<const char*>(out) + bytes, exclusive};
    std::lock_guard<std::mutex> lk(g_run_mu);
    std::vector<LaunchSpan>& run = g_runs[{current_device(), stream}];
    if (!run.empty() && run.back().exclusive) run.erase(run.begin(), run.end() - 1);
    bool defer = on && !run.empty() && run.size() < kMaxRun;
    for (const LaunchSpan& o : run)
        if (overlap(me.in0, me.in1, o.out0, o.out1) || overlap(me.out0, me.out1, o.out0, o.out1) ||
            overlap(me.out0, me.out1, o.in0, o.in1))
            defer = false;
    if (!defer) run.clear();            // this launch waits at its start: it begins a new run
    run.push_back(me);
    return defer;
}

cudaError_t pointwise_f32s(uint64_t, const void*, const void*, void*, uint64_t, cudaStream_t, int, int*);
cudaError_t pointwise_f32w(uint64_t, const void*, const void*, void*, uint64_t, cudaStream_t, int, int*);
cudaError_t pointwise_gold(uint64_t, const void*, const void*, void*, uint64_t, cudaStream_t, int, int*);
cudaError_t pointwise_f64(uint64_t, const void*, const void*, void*, uint64_t, cudaStream_t, int, int*);

int mp_num_passes(int L, int word, int variant, uint64_t p) {
    if (variant == V_SIXSTEP) return 2;
    if (fourstep_applies(L, variant, p, word)) return 2;
    if (tile_2p14_applies(L, variant, p, word)) return variant == V_FLAT ? 3 : 2;
    if (variant == V_NAIVE || L <= single_pass_max_log2(word)) return 1;
    int K[8];
    int P = plan_passes(L, word, variant, K);
    return P + (variant == V_FLAT ? 1 : 0);
}

uint64_t mp_workspace_bytes(int L, int word, int variant, uint64_t batch, uint64_t p) {
    const uint64_t row = (1ull << L) * (uint64_t)word;
    if (variant == V_SIXSTEP) return 2 * batch * row;      // column / row passes ping-pong (tiles.cuh)
    if (fourstep_applies(L, variant, p, word)) return batch * row;       // pass A -> workspace -> pass B
    if (tile_2p14_applies(L, variant, p, word)) return 2 * batch * row;
    if (variant == V_NAIVE || L <= single_pass_max_log2(word)) return 0;
    return 2 * batch * row;
}

cudaError_t pointwise_launch(int kind, uint64_t p, const void* a, const void* b, void* c, uint64_t n,
                             cudaStream_t s, int num_sms, int* launches) {
    switch (kind) {
        case 0: return pointwise_f32s(p, a, b, c, n, s, num_sms, launches);
        case 1: return pointwise_f32w(p, a, b, c, n, s, num_sms, launches);
        case 2: return pointwise_gold(p, a, b, c, n, s, num_sms, launches);
        default: return pointwise_f64(p, a, b, c, n, s, num_sms, launches);
    }
}
}  // namespace nttb200
