// Placeholder; the executor lands in the next commit.
#include "runtime.h"
#include "tcb.h"
#define TCB_API extern "C" __attribute__((visibility("default")))
using namespace tcb;
TCB_API int tcb_trainer_create(const char*, tcb_trainer**) { return fail(TCB_ERR_UNSUPPORTED, "trainer not built"); }
TCB_API int tcb_trainer_destroy(tcb_trainer*) { return TCB_OK; }
TCB_API int tcb_nccl_unique_id(uint8_t*) { return fail(TCB_ERR_UNSUPPORTED, "trainer not built"); }
TCB_API int tcb_trainer_join(tcb_trainer*, int, int, const uint8_t*) { return fail(TCB_ERR_UNSUPPORTED, "x"); }
TCB_API int tcb_trainer_set_batch(tcb_trainer*, const float*, const int32_t*, void*) { return fail(TCB_ERR_UNSUPPORTED, "x"); }
TCB_API int tcb_trainer_step(tcb_trainer*, void*) { return fail(TCB_ERR_UNSUPPORTED, "x"); }
TCB_API int tcb_trainer_loss(tcb_trainer*, float*, void*) { return fail(TCB_ERR_UNSUPPORTED, "x"); }
TCB_API int tcb_trainer_phase_times(tcb_trainer*, float*) { return fail(TCB_ERR_UNSUPPORTED, "x"); }
TCB_API int tcb_trainer_enable_timing(tcb_trainer*, int) { return fail(TCB_ERR_UNSUPPORTED, "x"); }
TCB_API int tcb_trainer_describe(tcb_trainer*, char**) { return fail(TCB_ERR_UNSUPPORTED, "x"); }
TCB_API int tcb_trainer_tensor(tcb_trainer*, const char*, void**, size_t*) { return fail(TCB_ERR_UNSUPPORTED, "x"); }
TCB_API int tcb_trainer_launch_count(tcb_trainer*, int*) { return fail(TCB_ERR_UNSUPPORTED, "x"); }
