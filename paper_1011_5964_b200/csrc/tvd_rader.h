// Rader DST-I engine for prime odd-core lengths (tvd_rader.cu).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "tvd_internal.h"

namespace tvd {

// host: plan for the DST odd core L (prime, M = L - 1 a product of 2,3,4,5,7,8,11,13 whose
// stages fit the CTA); false when the engine does not apply
bool build_rader_plan(int L, RaderPlan* P, std::vector<void*>& owned);
bool rader_launchable(const RaderPlan& P, int len, int family);
// DST-I (family DST1 / SINE_HAT) of every row of an nlines x len row-major array, one row
// per CTA, with the LineIO pre / mid (sandwich) / post / dot / finalizer hooks
cudaError_t launch_rader_rows(const RaderPlan& P, int family, int len, int nlines,
                              const LineIO& io, int* nblocks_out, cudaStream_t st);
int rader_threads();
// band projection (preconditioner assembly, k_band's math) of every line with the length-L DFT
// computed by the Rader engine: one line per CTA; *nblocks_out = nlines (min / max partials)
cudaError_t launch_band_rader(const RaderPlan& P, int n, const double2* wfull, const BandLines& b,
                              int* nblocks_out, cudaStream_t st);

}  // namespace tvd
