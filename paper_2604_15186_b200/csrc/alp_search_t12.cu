// k_search instantiations for 12 rows per lane (see alp_search.cuh).
#include "alp_search.cuh"

namespace alp {

cudaError_t launch_search_t12(const SearchArgs &a, int grid, cudaStream_t st) {
#define CALL(T, N, T2) launch_one<T, N, T2>(a, grid, st)
  ALP_DISPATCH_W(CALL, 12);
#undef CALL
}

int occ_search_t12(const SearchArgs &a) {
#define CALL(T, N, T2) occ_one<T, N, T2>(a)
  ALP_DISPATCH_W(CALL, 12);
#undef CALL
}

}  // namespace alp
