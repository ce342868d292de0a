// attention_ws.cu -- the warp-specialized tensor-core decode-attention kernel
// (attention_ws.cuh) and its dispatch over (D, query rows per pass, Key / Value bits, group
// size). attend_mma (attention_mma.cu) calls attend_ws_launch first and falls back to the
// single-warp kernel when it returns 0.
#include "mma_common.cuh"

namespace kvb {
namespace {

#include "attention_ws.cuh"

template <int D, int KB, int VB, int R>
int ws_gs(MmaParams& p, int BH, Workspace& ws, cudaStream_t st) {
  if constexpr (KB == 3 && D != 128) {
    return 0;
  } else {
    return p.gs == 32 ? launch_ws<D, KB, VB, R, 32>(p, BH, ws, st) : launch_ws<D, KB, VB, R, 0>(p, BH, ws, st);
  }
}

template <int D, int R>
int ws_bits(MmaParams& p, int kb, int vb, int BH, Workspace& ws, cudaStream_t st) {
  switch (kb * 10 + vb) {
    case 22: return ws_gs<D, 2, 2, R>(p, BH, ws, st);
    case 24: return ws_gs<D, 2, 4, R>(p, BH, ws, st);
    case 42: return ws_gs<D, 4, 2, R>(p, BH, ws, st);
    case 44: return ws_gs<D, 4, 4, R>(p, BH, ws, st);
    case 32: return ws_gs<D, 3, 2, R>(p, BH, ws, st);
    case 34: return ws_gs<D, 3, 4, R>(p, BH, ws, st);
    case 23: return ws_gs<D, 2, 3, R>(p, BH, ws, st);
    case 33: return ws_gs<D, 3, 3, R>(p, BH, ws, st);
    case 43: return ws_gs<D, 4, 3, R>(p, BH, ws, st);
    default: return 0;
  }
}

}  // namespace

// Launches the warp-specialized kernel for one pass chunk; returns the unit-range count (0 =
// this combination is not served here).
int attend_ws_launch(MmaParams& p, int D, int rows, int kb, int vb, int BH, Workspace& ws, cudaStream_t st) {
  if (D == 64) return rows == 1 ? ws_bits<64, 1>(p, kb, vb, BH, ws, st) : ws_bits<64, 2>(p, kb, vb, BH, ws, st);
  if (D == 128) return rows == 1 ? ws_bits<128, 1>(p, kb, vb, BH, ws, st) : ws_bits<128, 2>(p, kb, vb, BH, ws, st);
  return 0;
}

}  // namespace kvb
