/*
 * tcb_planner.h — C-ABI of the traincap planner (libtraincap.so).
 *
 * One JSON request in, one JSON reply out. The request's "op" selects a
 * function of the reference's C++ API, which this library re-implements with
 * identical semantics (csrc/host/*.cpp):
 *
 *   op                        reference interface replaced
 *   propagate_shapes          traincap::propagate_shapes      src/net_model.cpp:80
 *   validate_network          traincap::validate_network      src/net_model.cpp:36
 *   memory_bound              traincap::memory_bound          src/mem_model.cpp:83
 *   feature_map_memory        traincap::feature_map_memory    src/mem_model.cpp:30
 *   model_param_memory        traincap::model_param_memory    src/mem_model.cpp:43
 *   classifier_memory         traincap::classifier_memory     src/mem_model.cpp:61
 *   parameter_bits            traincap::parameter_bits        src/mem_model.cpp:97
 *   load_catalog              traincap::load_catalog/save_catalog src/catalog.cpp:205,224
 *   catalog_options           traincap::catalog_options       src/conv_select.cpp:173
 *   solve / solve_catalog     traincap::solve_selection / brute_force_selection
 *                                                             src/conv_select.cpp:182,199
 *   plan_batch_size           traincap::plan_batch_size       src/batch_plan.cpp:54
 *   default_batch_candidates  traincap::default_batch_candidates src/batch_plan.cpp:17
 *   efficiency, scaling_table, max_overhead_ratio, recommend_gpus,
 *   estimate_overhead_ratio, min_parameter_servers
 *                             traincap Lemma 1 / 2            src/scale_plan.cpp:30-112
 *   load_step_trace           traincap::load_step_trace       src/io.cpp:103
 *   run_plan, render_scale, render_ps
 *                             traincap::run_plan + renderers  src/report.cpp:57-358
 *   parse_bytes, parse_bandwidth, human_bytes, to_shortest_string, parse_number
 *                             traincap units/util             src/units.cpp, src/util.cpp
 *
 * (paths relative to /root/reference/proj). Errors come back as
 * {"error": {"type": "<traincap exception class>", "message": ..., "line": n}}.
 * The returned string is malloc'ed; release it with tcb_planner_free.
 */
#ifndef TCB_PLANNER_H_
#define TCB_PLANNER_H_

#ifdef __cplusplus
extern "C" {
#endif

char* tcb_planner_call(const char* request_json);
void tcb_planner_free(char* reply);

#ifdef __cplusplus
}
#endif
#endif /* TCB_PLANNER_H_ */
