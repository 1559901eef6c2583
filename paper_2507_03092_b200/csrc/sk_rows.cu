// sk_rows.cu -- device Pauli row sets: grouping + Clifford+T pass (TEMPORARY STUBS, filled in next).
#include "sk_internal.hpp"
#define STUB(c) do { if (c) (c)->err = "not implemented yet"; return SK_EUNSUPPORTED; } while (0)
struct sk_rows { sk_ctx* ctx; };
struct sk_pbc { sk_ctx* ctx; };
extern "C" {
int32_t sk_rows_create(sk_ctx* c, uint64_t, uint64_t, sk_rows**) { STUB(c); }
void sk_rows_destroy(sk_rows*) {}
uint64_t sk_rows_count(const sk_rows*) { return 0; }
int32_t sk_rows_upload(sk_rows* r, const uint64_t*, const uint64_t*, const uint8_t*, uint64_t) { STUB(r ? r->ctx : nullptr); }
int32_t sk_rows_download(sk_rows* r, uint64_t*, uint64_t*, uint8_t*) { STUB(r ? r->ctx : nullptr); }
int32_t sk_rows_conj_layer(sk_rows* r, const sk_gate*, size_t) { STUB(r ? r->ctx : nullptr); }
int32_t sk_commutation_vector(sk_rows* r, const uint64_t*, const uint64_t*, uint64_t*) { STUB(r ? r->ctx : nullptr); }
int32_t sk_rowsum_plus_i_where_anticommuting(sk_rows* r, const uint64_t*, const uint64_t*, uint8_t, uint64_t*) { STUB(r ? r->ctx : nullptr); }
int32_t sk_find_first_duplicate(sk_rows* r, int*, uint64_t*, uint64_t*) { STUB(r ? r->ctx : nullptr); }
int32_t sk_weight_sum(sk_rows* r, uint64_t*) { STUB(r ? r->ctx : nullptr); }
int32_t sk_group_first_fit(sk_rows* r, int, uint32_t*, uint64_t*) { STUB(r ? r->ctx : nullptr); }
int32_t sk_verify_grouping(sk_rows* r, int, const uint32_t*, uint64_t*) { STUB(r ? r->ctx : nullptr); }
int32_t sk_transpile(sk_ctx* c, uint64_t, const sk_gate*, size_t, sk_pbc**) { STUB(c); }
void sk_pbc_destroy(sk_pbc*) {}
int32_t sk_pbc_stats(sk_pbc* p, uint64_t*) { STUB(p ? p->ctx : nullptr); }
uint64_t sk_pbc_layer_rows(sk_pbc*, uint64_t) { return 0; }
int32_t sk_pbc_layer_download(sk_pbc* p, uint64_t, uint64_t*, uint64_t*, uint8_t*) { STUB(p ? p->ctx : nullptr); }
int32_t sk_pbc_mtab_download(sk_pbc* p, uint64_t*, uint64_t*, uint8_t*) { STUB(p ? p->ctx : nullptr); }
}
