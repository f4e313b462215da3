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

/* Routing gateway (reference proj/include/ppd/gateway.hpp).
 * Replaces ppd::gateway::Gateway (gateway.hpp:72-108) for non-C++ callers:
 * the same framed-JSON messages (register / heartbeat / route / stats,
 * gateway.cpp:204-255), handled in process or over loopback TCP
 * (serve_tcp, gateway.cpp:316-342). A backend may register with "gpu": i, and
 * route replies then name decode_gpu / prefill_gpu. Status: 0 ok, -1 invalid
 * argument (the reference's std::invalid_argument), -2 other failure. */
typedef struct ppd_gateway ppd_gateway;
/* policy_json: {"x": 0..1} (static) or {"policy": "dynamic", "table_json": "..."},
 * optional "session_ttl_s" (3600), "backend_timeout_s" (30) */
int ppd_gateway_create(const char* policy_json, ppd_gateway** out);
/* one JSON payload in (no length prefix), reply payload out (free with
 * ppd_engine_free); `now` in seconds, the caller's clock */
int ppd_gateway_handle(ppd_gateway* gw, const char* payload, double now, char** reply);
/* start the TCP server on 127.0.0.1:port (0 = ephemeral) on a background
 * thread; *bound_port receives the port. One server per gateway. */
int ppd_gateway_serve(ppd_gateway* gw, int port, int* bound_port);
/* stop the server (joins its threads); no-op when not serving */
int ppd_gateway_stop(ppd_gateway* gw);
void ppd_gateway_destroy(ppd_gateway* gw);

#ifdef __cplusplus
}
#endif
#endif
