// Multi-pass tile kernels and the six-step split, Goldilocks (canonical).
#include "tiles.cuh"
#include "lazy.cuh"
#include <cstdlib>
namespace nttb200 {
cudaError_t tile_passes_gold(int variant, const MultipassReq& r, bool* ok) {
    using A = GoldPolicy<false>;
    switch (variant) {
        case V_DIT: return ftile::run_tile_passes<A, V_DIT>(r, ok);
        case V_DIF: return ftile::run_tile_passes<GoldPolicy<true>, V_DIF>(r, ok);
        case V_FLAT: return ftile::run_tile_passes<A, V_FLAT>(r, ok);
        case V_PEASE: return ftile::run_tile_passes<A, V_PEASE>(r, ok);
        case V_PEASE_NC: return ftile::run_tile_passes<A, V_PEASE_NC>(r, ok);
        case V_STOCKHAM: return ftile::run_tile_passes<A, V_STOCKHAM>(r, ok);
        default: *ok = false; return cudaSuccess;
    }
}
template <int K1, int K2>
static bool six_match(const MultipassReq& r) {
    return r.n1 == (1ull << K1) && r.n2 == (1ull << K2);
}
cudaError_t tile_sixstep_gold(const MultipassReq& r, bool* ok) {
    using A = GoldPolicy<false>;
    *ok = false;
    if (!r.stw1 || !r.stw2 || !r.cor_lo) return cudaSuccess;
    // long-run column/row passes + explicit transpose (the 2^13 x 2^13 and
    // 2^7 x 2^7 splits); other splits fall to the column-at-a-time kernels
    {
        cudaError_t e = ftile::run_sixstep_cols<A>(r, ok);
        if (e != cudaSuccess || *ok) return e;
    }
    *ok = true;
    if (six_match<13, 13>(r)) return ftile::run_sixstep_tiles_k<A, 13, 13>(r);
    if (six_match<7, 7>(r)) return ftile::run_sixstep_tiles_k<A, 7, 7>(r);
    *ok = false;
    return cudaSuccess;
}
uint64_t sixstep_dist_ws_bytes(uint64_t n, int world, int word) { return 2 * (n / (uint64_t)world) * (uint64_t)word; }

cudaError_t tile_sixstep_dist_gold(const MultipassReq& r, int step, int rank, int world, const void* in, void* out,
                                   bool* ok, void* const* peers) {
    using A = GoldPolicy<false>;
    *ok = false;
    if (!r.stw1 || !r.stw2 || !r.cor_lo) return cudaSuccess;
    // long-run column passes + per-destination transpose
    {
        cudaError_t e = ftile::run_sixstep_cols_dist<A>(r, step, rank, world, in, out, r.ws, ok, peers);
        if (e != cudaSuccess || *ok || peers) return e;      // the peer pack exists on the long-run path only
    }
    *ok = true;
    if (six_match<13, 13>(r))
        return step == 0 ? ftile::sixstep_step_a<A, 13, 13>(r, rank, world, in, out)
                         : ftile::sixstep_step_b<A, 13, 13>(r, world, in, out);
    if (six_match<7, 7>(r))
        return step == 0 ? ftile::sixstep_step_a<A, 7, 7>(r, rank, world, in, out)
                         : ftile::sixstep_step_b<A, 7, 7>(r, world, in, out);
    *ok = false;
    return cudaSuccess;
}
}  // namespace nttb200
