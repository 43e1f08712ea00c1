// Host-side plan queries shared by the C ABI (pass counts, workspace sizes)
// and the field-dispatched pointwise multiply.
#include "launch.cuh"
namespace nttb200 {
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
