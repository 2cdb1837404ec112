// TEMPORARY: replaced by generate.cu / convert.cu.
#include "common.cuh"
using namespace spmvb;
#define NI(name) return fail(SPMVB_ERR_INVALID_ARGUMENT, name ": not implemented yet")
extern "C" {
int spmvb_generate_csr(const spmvb_grid *, int64_t, int64_t, void *, spmvb_matrix **) { NI("generate_csr"); }
int spmvb_csr_to_ell(const spmvb_matrix *, int32_t, void *, spmvb_matrix **) { NI("csr_to_ell"); }
int spmvb_csr_compress_values(const spmvb_matrix *, const spmvb_compress_options *, int32_t, void *, spmvb_matrix **) { NI("compress_values"); }
int spmvb_csr_compress_patterns(const spmvb_matrix *, const spmvb_compress_options *, void *, spmvb_matrix **) { NI("compress_patterns"); }
int spmvb_to_csr(const spmvb_matrix *, void *, spmvb_matrix **) { NI("to_csr"); }
int spmvb_validate(const spmvb_matrix *, int64_t, void *) { NI("validate"); }
int spmvb_pattern_remap(spmvb_matrix *, int32_t, const int64_t *, const int32_t *, const int32_t *, const int32_t *, void *) { NI("remap"); }
}
