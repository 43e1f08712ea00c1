// Multi-pass tile kernels, u32 fields (p < 2^31): LazyF32 (p < 2^30) and canonical.
#include "tiles.cuh"
#include "lazy.cuh"
namespace nttb200 {
template <class A>
static cudaError_t run_v(int variant, const MultipassReq& r, bool* ok) {
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
cudaError_t tile_passes_f32(int variant, bool lazy, const MultipassReq& r, bool* ok) {
    return lazy ? run_v<LazyF32>(variant, r, ok) : run_v<Canon<F32S>>(variant, r, ok);
}
}  // namespace nttb200
