"""§8f-3 widening: the routing gateway fronting GPU workers
(include/ppd/gateway.hpp, engine/gateway.cpp). Every scripted case mirrors a
reference test (proj/tests/test_gateway.cpp) and is also replayed through the
UNMODIFIED reference gateway (oracle/_ref/ref_tool op=gateway): results must
be identical item for item (the wall-clock decision-latency field excepted).
The TCP cases run the real loopback server with GPU workers registering and
heartbeating over the wire."""
import json
import os
import random

from oracle import oracle as O
from paper_2603_13358_b200 import engine as E


def both(job):
    ours = E.run(dict(job, op="gateway"))
    if not os.path.exists(O.REF_TOOL):  # reference checker not built: properties only
        return ours["results"]
    ref = O.ref_tool(dict(job, op="gateway"))
    assert "error" not in ref, ref
    assert ours["results"] == ref["results"]
    return ours["results"]


def q(conv, turn, now, ctx=1000):
    return {"do": "route", "conv": conv, "turn": turn, "n_in": 256, "n_ctx": 0 if turn == 1 else ctx, "n_out": 256,
            "now": now}


def test_registry_heartbeat_boundary():
    # test_gateway.cpp:40-64: staleness is strictly greater than 30 s
    s = [{"do": "add", "role": "P", "address": "p:1"}, {"do": "add", "role": "D", "address": "d:1"},
         {"do": "add", "role": "Q", "address": "q:1"},
         {"do": "heartbeat", "id": 0, "now": 10.0},
         {"do": "prune", "now": 29.0}, {"do": "prune", "now": 30.0}, {"do": "prune", "now": 30.5},
         {"do": "heartbeat", "id": 1, "now": 31.0}, {"do": "find", "id": 0}, {"do": "find", "id": 1},
         {"do": "stats"}]
    r = both({"script": s})
    assert r[0] == {"id": 0} and r[1] == {"id": 1}
    assert r[2] == {"invalid_argument": True}
    assert r[4]["removed"] == [] and r[5]["removed"] == [] and r[6]["removed"] == [1]
    assert r[7] == {"ok": False}
    assert r[8]["found"] and r[8]["last_heartbeat"] == 10.0 and not r[9]["found"]
    assert r[10]["backends"] == 1


def _affinity_script(tail):
    s = [{"do": "add", "role": "P", "address": "p:1"}, {"do": "add", "role": "D", "address": "d:1"},
         {"do": "add", "role": "D", "address": "d:2"}, q("conv-a", 1, 1.0)]
    for i in range(5):
        t = 2.0 + i
        s += [{"do": "heartbeat", "id": b, "now": t} for b in (0, 1, 2)]
        s.append(q("conv-a", 2 + i, t))
    return s + tail


def test_route_session_affinity():
    # test_gateway.cpp:78-99 + "a second conversation gets its own pin"
    r = both({"x": 1.0, "script": _affinity_script([q("conv-b", 1, 8.0), {"do": "stats"}])})
    first = r[3]
    assert first["ok"] and first["target"] == "P_path" and first["prefill_backend"] == 0
    pinned = first["decode_backend"]
    routes = [x for x in r[4:-2] if "target" in x]
    assert len(routes) == 5 and all(x["target"] == "D_local" and x["decode_backend"] == pinned for x in routes)
    assert r[-2]["decode_backend"] != pinned
    assert r[-1]["queries"] == 7 and r[-1]["p_path"] == 2 and r[-1]["d_local"] == 5


def test_pruned_backend_invalidates_sessions():
    # test_gateway.cpp:107-119 (pinned D is d:1 = id 1 by round robin)
    r = both({"x": 1.0, "script": _affinity_script([{"do": "heartbeat", "id": 0, "now": 45.0},
                                                    {"do": "heartbeat", "id": 2, "now": 45.0},
                                                    q("conv-a", 8, 45.0)])})
    pinned, last = r[3]["decode_backend"], r[-1]
    assert last["ok"] and last["session_missing"] and last["target"] == "P_path" and last["decode_backend"] != pinned


def test_session_ttl():
    # test_gateway.cpp:121-129
    t = 3700.0
    r = both({"x": 1.0, "script": _affinity_script([{"do": "heartbeat", "id": b, "now": t} for b in (0, 1, 2)]
                                                   + [q("conv-a", 3, t)])})
    assert r[-1]["session_missing"] and r[-1]["target"] == "P_path"


def test_capacity_and_replicas():
    # test_gateway.cpp:132-163
    none = both({"x": 0.0, "script": [q("c", 1, 0.0)]})[0]
    assert not none["ok"] and none["error"] == "no_capacity"
    rep = both({"x": 0.0, "script": [{"do": "add", "role": "R", "address": "r:1"},
                                     {"do": "add", "role": "R", "address": "r:2"}, q("conv-a", 1, 1.0),
                                     {"do": "heartbeat", "id": 0, "now": 2.0},
                                     {"do": "heartbeat", "id": 1, "now": 2.0}, q("conv-a", 2, 2.0),
                                     q("conv-z", 2, 2.0)]})
    assert rep[2]["target"] == "R_local" and rep[5]["decode_backend"] == rep[2]["decode_backend"]
    assert rep[6]["session_missing"]  # turn 2 of an unknown conversation
    stand_in = both({"x": 0.0, "script": [{"do": "add", "role": "P", "address": "p:1"},
                                          {"do": "add", "role": "R", "address": "r:1"}, q("c", 1, 0.0)]})
    assert stand_in[2]["ok"]
    only_p = both({"x": 0.0, "script": [{"do": "add", "role": "P", "address": "p:1"}, q("c", 1, 0.0)]})
    assert only_p[1]["error"] == "no_capacity"


def test_affinity_under_churn():
    # test_gateway.cpp:165-207, 10k queries with backend kills and re-adds
    rnd = random.Random(99)
    s, pin, ds, next_id, t = [{"do": "add", "role": "P", "address": "p:1"}], {}, [], 1, 0.0
    for i in range(4):
        s.append({"do": "add", "role": "D", "address": f"d:{i}"})
        ds.append(next_id)
        next_id += 1
    route_idx = []
    for i in range(10000):
        t += 0.01
        s += [{"do": "heartbeat", "id": b, "now": t} for b in [0] + ds]
        conv = f"conv-{rnd.randrange(64)}"
        turn = 2 if conv in pin else 1
        s.append(q(conv, turn, t))
        route_idx.append((len(s) - 1, conv, turn))
        pin.setdefault(conv, None)
        if i % 2500 == 2499:
            victim = ds[rnd.randrange(len(ds))]
            s += [{"do": "remove", "id": victim}, {"do": "invalidate", "id": victim}]
            route_idx.append(("kill", victim, None))
            ds.remove(victim)
            s.append({"do": "add", "role": "D", "address": f"d:new{i}", "now": t})
            ds.append(next_id)
            next_id += 1
    s.append({"do": "stats"})
    r = both({"x": 1.0, "script": s})
    pinned = {}
    for k, conv, turn in route_idx:
        if k == "kill":
            pinned = {c: b for c, b in pinned.items() if b != conv}
            continue
        x = r[k]
        assert x["ok"]
        if conv in pinned:
            assert x["target"] == "D_local" and x["decode_backend"] == pinned[conv]
        else:
            pinned[conv] = x["decode_backend"]
    st = r[-1]
    assert st["queries"] == 10000 and st["errors"] == 0 and st["d_local"] > 0 and st["p_path"] > 0


def test_wire_messages():
    # test_gateway.cpp:209-246, byte-equal replies
    msgs = [('{"kind":"register","role":"P","address":"p:1"}', 0.0),
            ('{"kind":"register","role":"D","address":"d:1"}', 0.0),
            ('{"kind":"register","role":"PD","address":"x"}', 0.0),
            (json.dumps({"kind": "heartbeat", "id": 1}), 5.0),
            (json.dumps({"kind": "route", "conv_first_message": "hello", "turn_index": 1, "new_input_tokens": 128,
                         "target_output_tokens": 128}), 5.0),
            (json.dumps({"kind": "route", "conv_first_message": "hello", "turn_index": 2, "new_input_tokens": 64,
                         "cached_context_tokens": 256, "target_output_tokens": 16}), 5.5),
            ('{"kind":"route","turn_index":1}', 5.5),
            ('{"kind":"stats"}', 6.0), ('{"kind":"warp"}', 0.0), ("not json", 0.0)]
    r = both({"x": 1.0, "script": [{"do": "message", "payload": p, "now": t} for p, t in msgs]})
    rep = [json.loads(x["reply"]) for x in r]
    assert rep[0]["kind"] == "register_reply" and rep[2]["kind"] == "error"
    assert rep[3] == {"kind": "heartbeat_reply", "ok": True}
    assert rep[4]["target"] == "P_path" and rep[5]["target"] == "D_local"
    assert rep[6]["kind"] == "error"
    assert rep[7]["queries"] == 2 and rep[7]["p_path"] == 1 and rep[7]["backends"] == 2 and rep[7]["sessions"] == 1
    assert rep[8] == {"kind": "error", "error": "unknown_kind"} and rep[9]["kind"] == "error"


def test_dynamic_policy_matches_reference():
    # Phase-2 decisions through the gateway with a Phase-1 table (routing.cpp:340-387)
    s = [{"do": "add", "role": "P", "address": "p:1"}, {"do": "add", "role": "D", "address": "d:1"},
         {"do": "add", "role": "D", "address": "d:2"}]
    rnd = random.Random(5)
    t = 0.0
    for i in range(300):
        t += 0.05
        s += [{"do": "heartbeat", "id": b, "now": t} for b in (0, 1, 2)]
        s.append({"do": "route", "conv": f"c{rnd.randrange(40)}", "turn": rnd.choice([1, 2, 3]),
                  "n_in": rnd.choice([64, 512, 4096]), "n_ctx": rnd.choice([0, 1000, 9000, 20000]),
                  "n_out": rnd.choice([16, 256, 1024]), "now": t})
    for x in (1.0 / 3, 0.5, 2.0 / 3):
        both({"x": x, "script": s})
    table = {"header": {"weights": {"w_ttft": 1.0, "w_tpot": 1.0}, "calibration_hash": "h", "built_at": "t"},
             "entries": {}}
    for ci, cls in enumerate(("small", "medium", "large")):
        for typ in ("balanced", "prefill_heavy", "decode_heavy"):
            for qi, qps in enumerate((0.5, 1, 2, 4, 6, 8, 10, 12, 16, 20)):
                x1 = (ci + qi) % 3 != 0
                table["entries"][f"{cls}|{typ}|{qps}"] = {
                    "ttft_x0": 1.0, "ttft_x1": 0.5, "tpot_x0": 0.01, "tpot_x1": 0.0101, "delta_ttft": 0.5,
                    "delta_tpot": 0.01, "score": 0.49 if x1 else -0.1, "x_star": int(x1), "available": qi != 3}
    r = both({"policy": "dynamic", "table_json": json.dumps(table), "script": s})
    assert {x["x_used"] for x in r if "x_used" in x} == {0, 1}


def test_gpu_workers_over_tcp():
    # loopback server; four GPU workers (1P_3D on GPUs 0-3) register + heartbeat
    # on their own threads; a client routes over split frames
    workers = [{"role": "P", "gpu": 0, "address": "gpu0"}] + [
        {"role": "D", "gpu": g, "address": f"gpu{g}"} for g in (1, 2, 3)]
    msgs = [json.dumps({"kind": "route", "conv_first_message": f"conv-{i % 5}", "turn_index": 1 + (i >= 5),
                        "new_input_tokens": 256, "cached_context_tokens": 0 if i < 5 else 512,
                        "target_output_tokens": 64}) for i in range(10)] + ['{"kind":"stats"}']
    out = E.run({"op": "gateway_tcp", "x": 1.0, "workers": workers, "messages": msgs, "split": 3,
                 "heartbeat_s": 0.02, "hold_s": 0.3})
    assert out["port"] > 0 and out["worker_ids"] == [0, 1, 2, 3]
    rep = [json.loads(x) for x in out["replies"]]
    gpu_of = {0: 0, 1: 1, 2: 2, 3: 3}
    pins = {}
    for i, r in enumerate(rep[:10]):
        assert r["ok"] and r["decode_gpu"] == gpu_of[r["decode_backend"]]
        if i < 5:
            assert r["target"] == "P_path" and r["prefill_gpu"] == 0
            pins[i] = r["decode_backend"]
        else:
            assert r["target"] == "D_local" and r["decode_backend"] == pins[i - 5] and "prefill_gpu" not in r
    assert len(set(pins.values())) == 3  # round robin over the three D GPUs
    assert rep[10]["kind"] == "stats_reply" and rep[10]["backends"] == 4 and rep[10]["queries"] == 10
    assert out["heartbeats"] >= 4


def test_frame_split_delivery_over_tcp():
    # test_gateway.cpp:11-38 over a real socket: 1-byte pieces, an empty-ish
    # payload, a garbled payload
    out = E.run({"op": "gateway_tcp", "x": 0.0, "messages": ['{"kind":"stats"}', "x", '{"kind":"register","role":"R"}'],
                 "split": 1})
    rep = [json.loads(x) for x in out["replies"]]
    assert rep[0]["kind"] == "stats_reply" and rep[0]["backends"] == 0
    assert rep[1]["kind"] == "error"
    assert rep[2] == {"kind": "register_reply", "id": 0}


def test_gateway_c_abi_symbols():
    import re
    import subprocess
    hdr = open(os.path.join(os.path.dirname(E.ENGINE_PATH), "..", "include", "ppd_engine.h")).read()
    names = re.findall(r"^\w[\w\s\*]*?\b(ppd_\w+)\s*\(", hdr, re.M)
    assert {"ppd_engine_run_json", "ppd_gateway_create", "ppd_gateway_handle", "ppd_gateway_serve",
            "ppd_gateway_stop", "ppd_gateway_destroy"} <= set(names)
    out = subprocess.run(["nm", "-D", "--defined-only", E.ENGINE_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(names) <= exported


def test_gateway_c_abi_in_process_and_python_client():
    import socket
    import struct
    import pytest
    with pytest.raises(ValueError):
        E.Gateway({"x": 1.5})  # RoutingPolicy::validate (routing.cpp) rejects x outside [0, 1]
    gw = E.Gateway({"x": 1.0})
    assert json.loads(gw.handle('{"kind":"register","role":"P","gpu":0}', 0.0)) == {"kind": "register_reply", "id": 0}
    assert json.loads(gw.handle('{"kind":"register","role":"D","gpu":1}', 0.0))["id"] == 1
    port = gw.serve(0)
    with pytest.raises(ValueError):
        gw.serve(0)  # one server per gateway

    def call(sock, payload):
        b = payload.encode()
        sock.sendall(struct.pack(">I", len(b)) + b)
        hdr = b""
        while len(hdr) < 4:
            hdr += sock.recv(4 - len(hdr))
        n, body = struct.unpack(">I", hdr)[0], b""
        while len(body) < n:
            body += sock.recv(n - len(body))
        return json.loads(body)

    with socket.create_connection(("127.0.0.1", port)) as s:
        # the in-process registrations above used clock 0; the server's wall
        # clock prunes them (> 30 s without a heartbeat), so workers re-register
        assert call(s, '{"kind":"register","role":"P","gpu":0}')["id"] == 2
        assert call(s, '{"kind":"register","role":"D","gpu":1}')["id"] == 3
        r = call(s, json.dumps({"kind": "route", "conv_first_message": "hi", "turn_index": 1,
                                "new_input_tokens": 100, "target_output_tokens": 10}))
        assert r["target"] == "P_path" and r["prefill_gpu"] == 0 and r["decode_gpu"] == 1
        st = call(s, '{"kind":"stats"}')
        assert st["queries"] == 1 and st["backends"] == 2 and st["decision_latency_p99_us"] > 0
    gw.stop()
    gw.stop()
    gw.close()


def test_gateway_threadsanitizer(tmp_path):
    """SURVEY §5 race detection: the gateway under concurrent TCP clients,
    heartbeating workers and in-process admin calls, built with
    -fsanitize=thread (tests/native/gateway_tsan.cpp)."""
    import shutil
    import subprocess
    import pytest
    if not shutil.which("g++"):
        pytest.skip("g++ absent")
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    eng = os.path.join(repo, "paper_2603_13358_b200", "engine")
    json_inc = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
    if not os.path.isdir(json_inc):
        pytest.skip("nlohmann json headers absent")
    exe = str(tmp_path / "gateway_tsan")
    srcs = [os.path.join(repo, "tests", "native", "gateway_tsan.cpp")] + [
        os.path.join(eng, f) for f in ("gateway.cpp", "routing.cpp", "md5.cpp", "metrics.cpp", "util.cpp",
                                       "workload.cpp", "costmodel.cpp")]
    subprocess.run(["g++", "-std=c++20", "-O1", "-g", "-fsanitize=thread", "-pthread", "-I" + os.path.join(repo, "include"),
                    "-I" + json_inc, *srcs, "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, TSAN_OPTIONS="halt_on_error=1 second_deadlock_stack=1"))
    assert "ThreadSanitizer" not in r.stderr, r.stderr[-4000:]
    assert r.returncode == 0, (r.stdout, r.stderr[-2000:])
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["bad"] == 0 and out["queries"] == 2400 and out["backends"] == 6


def test_worker_heartbeats_survive_gateway_shutdown():
    """the gateway stops under live GPU-worker agents; their
    heartbeat threads record the closed connection and stop (no
    std::terminate from an exception escaping the thread)."""
    workers = [{"role": "D", "gpu": g, "address": f"gpu{g}"} for g in (0, 1)]
    out = E.run({"op": "gateway_tcp", "x": 1.0, "workers": workers, "messages": ['{"kind":"stats"}'],
                 "heartbeat_s": 0.01, "hold_s": 0.05, "stop_server_first": True, "after_stop_s": 0.2})
    assert len(out["after_stop"]) == 2
    assert all(w["failed"] and "closed" in w["error"] for w in out["after_stop"])
