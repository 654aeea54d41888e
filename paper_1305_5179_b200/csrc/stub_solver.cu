#include "internal.h"
extern "C" {
rbf_status rbf_precond_create(rbf_ctx*, const rbf_cells*, const rbf_kernel*, const rbf_precond_cfg*, rbf_precond** out) { if (out) *out = nullptr; rbf::set_error("not yet"); return RBF_EUNSUPPORTED; }
void rbf_precond_free(rbf_precond*) {}
rbf_status rbf_precond_apply(rbf_ctx*, const rbf_precond*, const float*, float*) { return RBF_EUNSUPPORTED; }
rbf_status rbf_precond_blocks(const rbf_precond*, int64_t*, int64_t*, int64_t*, int64_t*, int32_t*, int32_t*) { return RBF_EUNSUPPORTED; }
rbf_status rbf_gmres_solve(rbf_ctx*, const rbf_cells*, const rbf_kernel*, const rbf_precond*, const rbf_precond_cfg*, const rbf_gmres_cfg*, const float*, double*, rbf_solve_report*) { return RBF_EUNSUPPORTED; }
rbf_status rbf_reconstruct_host(rbf_ctx*, const float*, const float*, int64_t, const rbf_kernel*, const rbf_cell_cfg*, const rbf_precond_cfg*, const rbf_gmres_cfg*, const rbf_grid*, double*, float*, rbf_solve_report*) { return RBF_EUNSUPPORTED; }
}
