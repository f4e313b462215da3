/* ppd_engine.h — C entry point of the host C++ engine (libppd_engine.so), for
 * callers that are not C++ (the Python tests and bench.py use it via ctypes).
 * C++ callers use the ppd:: headers (include/ppd/ headers) directly.
 *
 * One JSON job in, one JSON result out. The job schema is the one the
 * reference-side driver oracle/ref_tool.cpp accepts for op=simulate (cluster,
 * x | policy+table_json, conversations | workload+seed, calib_overrides |
 * calib_json, qps_replay, think_time_s, max_decode_batch, request_timeout_s),
 * plus "clock": "virtual" (default; the reference's cost model) or "device"
 * (every prefill, decode step and KV hop executes on the GPUs). */
#ifndef PPD_ENGINE_H
#define PPD_ENGINE_H
#ifdef __cplusplus
extern "C" {
#endif

/* returns 0 on success; *out_json must be released with ppd_engine_free */
int ppd_engine_run_json(const char* job_json, char** out_json);
void ppd_engine_free(char* p);
const char* ppd_engine_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
