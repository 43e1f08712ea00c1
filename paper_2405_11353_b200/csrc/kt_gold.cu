// Multi-pass tile kernels and the six-step split, Goldilocks (canonical).
#include "tiles.cuh"
#include "lazy.cuh"
namespace nttb200 {
cudaError_t tile_passes_gold(int variant, const MultipassReq& r, bool* ok) {
    using A = Canon<FGold>;
    switch (variant) {
        case V_DIT: return ftile::run_tile_passes<A, V_DIT>(r, ok);
        case V_DIF: return ftile::run_tile_passes<A, V_DIF>(r, ok);
        case V_FLAT: return ftile::run_tile_passes<A, V_FLAT>(r, ok);
        case V_PEASE: return ftile::run_tile_passes<A, V_PEASE>(r, ok);
        case V_PEASE_NC: return ftile::run_tile_passes<A, V_PEASE_NC>(r, ok);
        case V_STOCKHAM: return ftile::run_tile_passes<A, V_STOCKHAM>(r, ok);
        default: *ok = false; return cudaSuccess;
    }
}
cudaError_t tile_sixstep_gold(const MultipassReq& r, bool* ok) {
    *ok = false;
    if (r.n1 == (1ull << 13) && r.n2 == (1ull << 13) && r.stw1 && r.stw2 && r.cor_lo) {
        *ok = true;
        return ftile::run_sixstep_tiles_k<Canon<FGold>, 13, 13>(r);
    }
    return cudaSuccess;
}
}  // namespace nttb200
