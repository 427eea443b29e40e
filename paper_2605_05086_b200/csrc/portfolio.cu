// portfolio.cu — multi-GPU walker portfolio: NCCL communicator and the every-K
// exchange loop of chap_run_walkers. (first build: placeholder; filled in next)
#include "host.h"

extern "C" chap_status chap_comm_unique_id(uint8_t id[128]) {
  (void)id;
  return fail(CHAP_ERR_UNSUPPORTED, "chap_comm_unique_id: not built yet");
}
extern "C" chap_status chap_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device,
                                        chap_comm** out) {
  (void)id; (void)nranks; (void)rank; (void)device; (void)out;
  return fail(CHAP_ERR_UNSUPPORTED, "chap_comm_create: not built yet");
}
extern "C" chap_status chap_comm_destroy(chap_comm* comm) {
  (void)comm;
  return CHAP_OK;
}
extern "C" chap_status chap_run_walkers(const chap_problem* p, int32_t W_local, const double* x0,
                                        const chap_params* params, chap_comm* comm, int64_t max_iters,
                                        double time_limit_s, double* best_x, chap_result* out,
                                        void* cuda_stream) {
  (void)p; (void)W_local; (void)x0; (void)params; (void)comm; (void)max_iters; (void)time_limit_s;
  (void)best_x; (void)out; (void)cuda_stream;
  return fail(CHAP_ERR_UNSUPPORTED, "chap_run_walkers: not built yet");
}
