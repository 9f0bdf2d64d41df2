"""The B200 task server over loopback TCP, driven by the REFERENCE client
(client::submit compiled from /root/reference/proj/src/client.cpp into
oracle/_ref) -- the client a user of the reference already has.

Mirrors proj/tests/test_server.cpp:190-386 (ephemeral port, concurrent
clients, idle timeout, abandoned connection, port in use) and
acceptance.cpp:446-523 (served bytes == direct kernel bytes), with the
reference server (same registry, CPU-restated tasks) as the comparison.
"""
from __future__ import annotations

import socket
import threading
import time

import numpy as np
import pytest

import paper_1505_05655_b200 as G
import wire_util as W


@pytest.fixture(scope="module")
def server():
    with G.Server(max_tasks=4, idle_timeout_ms=300) as s:
        yield s


def test_ephemeral_port_and_early_errors_match_reference(server, refl):
    assert server.port != 0
    with refl.RefServer() as rs:
        for flag, params in [("NOPE", "rows=4,cols=4"), ("LUT_CORRECT", "rows=4"),
                             ("LUT_CORRECT", "rows=q,cols=4"), ("MATMUL", "m=1,k=1,n=1,prec=x"),
                             ("LUT_CORRECT", "rows=32768,cols=32768")]:
            ours = refl.ref_submit(server.port, flag, params, b"\x01\x02", "x.bin")
            ref = refl.ref_submit(rs.port, flag, params, b"\x01\x02", "x.bin")
            assert ours == ref
            assert ours[0].startswith("ERR:")


def test_raw_bad_header_gets_error_and_salvaged_name(server, refl):
    req = W.header("\x07AD", "", name="keep.me")
    resp = W.parse_response(W.roundtrip(server.port, req))
    assert resp["status"] == "ERR:BAD_HEADER" and resp["name"] == "keep.me"
    with refl.RefServer() as rs:
        assert W.roundtrip(server.port, req) == W.roundtrip(rs.port, req)


def test_early_reject_without_payload(server):
    """Header promising 2 GiB: the answer comes before any payload is sent."""
    with socket.create_connection(("127.0.0.1", server.port), timeout=10) as s:
        s.sendall(W.header("LUT_CORRECT", "rows=32768,cols=32768", has_payload=True))
        data = s.recv(4096)
    assert W.parse_response(data)["status"] == "ERR:TOO_LARGE"


def test_idle_connection_is_dropped_without_response(server):
    with socket.create_connection(("127.0.0.1", server.port), timeout=10) as s:
        s.sendall(W.header("LUT_CORRECT", "rows=64,cols=64", has_payload=True) + b"\0" * 100)
        t0 = time.time()
        data = s.recv(4096)  # server closes after its 300 ms idle timeout
        assert data == b"" and time.time() - t0 < 5


def test_abandoned_connection_does_not_wedge_server(server, refl):
    s = socket.create_connection(("127.0.0.1", server.port))
    s.sendall(b"LUT")
    s.close()
    status, _, _, _ = refl.ref_submit(server.port, "NOPE", "", b"", "a")
    assert status == "ERR:UNKNOWN_TASK"


def test_port_in_use_fails_with_bind_failed(server):
    with pytest.raises(G.GpcxError) as e:
        G.Server(port=server.port).start()
    assert e.value.code == "BindFailed"


def test_concurrent_clients(server, refl):
    results = []

    def worker(i):
        results.append(refl.ref_submit(server.port, "NOPE", f"i={i}", b"", f"n{i}"))

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(16)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert len(results) == 16 and all(r[0] == "ERR:UNKNOWN_TASK" for r in results)
    assert sorted(r[3] for r in results) == sorted(f"n{i}" for i in range(16))


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["equalize", "stretch"])
def test_loopback_lut_correct_equals_reference_server(gpu, server, refl, mode):
    from oracle import oracle as O
    rows, cols = 1024, 1536
    img = O.synth_image(O.IMG_RAMP12, 0x5EED, rows, cols)
    params = f"rows={rows},cols={cols},mode={mode}"
    ours = refl.ref_submit(server.port, "LUT_CORRECT", params, img.tobytes(), "c.raw")
    with refl.RefServer() as rs:
        ref = refl.ref_submit(rs.port, "LUT_CORRECT", params, img.tobytes(), "c.raw")
    assert ours[0] == "OK" and ours == ref
    direct_out, _, _ = O.lut_correct(img, O.LUT_EQUALIZE if mode == "equalize" else O.LUT_STRETCH)
    assert ours[2] == direct_out.tobytes()


@pytest.mark.gpu
def test_loopback_matmul_tensor_core(gpu, server, refl):
    from oracle import oracle as O
    m, k, n = 96, 200, 128
    A = O.synth_matrix(O.MAT_UNIFORM32, 2, m, k)
    B = O.synth_matrix(O.MAT_UNIFORM32, O.seed_b(2), k, n)
    payload = A.tobytes() + B.tobytes()
    status, params, data, name = refl.ref_submit(server.port, "MATMUL", f"m={m},k={k},n={n},prec=bf16",
                                                 payload, "c.f32")
    assert status == "OK" and name == "c.f32"
    assert G.parse_params(params) == {"m": str(m), "n": str(n), "k": str(k), "prec": "bf16",
                                      "bytes": str(m * n * 4)}
    Cg = np.frombuffer(data, dtype=np.float32).reshape(m, n)
    Cref, ab = O.matmul_f64(O.round_matrix(O.PREC_BF16, A), O.round_matrix(O.PREC_BF16, B))
    assert np.all(np.abs(Cg - Cref) <= 1e-5 * ab)


@pytest.mark.gpu
def test_many_concurrent_gpu_requests(gpu, server, refl):
    """The config-C5 shape in miniature: 16 concurrent clients, each a
    LUT_GEN -> LUT_APPLY -> MATMUL chain, against the 4-worker server."""
    from oracle import oracle as O
    errors = []

    def chain(i):
        try:
            img = O.synth_image(O.IMG_UNIFORM16, i, 128, 128)
            st, p, lut, _ = refl.ref_submit(server.port, "LUT_GEN", "rows=128,cols=128", img.tobytes())
            assert st == "OK"
            st, p, out, _ = refl.ref_submit(server.port, "LUT_APPLY", "rows=128,cols=128", lut + img.tobytes())
            assert st == "OK"
            r_out, _, _ = O.lut_correct(img, O.LUT_EQUALIZE)
            assert out == r_out.tobytes()
            x = np.frombuffer(out, dtype=np.uint16).astype(np.float32).reshape(128, 128) / 65535
            st, p, c, _ = refl.ref_submit(server.port, "MATMUL", "m=128,k=128,n=128",
                                          x.tobytes() + x.tobytes())
            assert st == "OK"
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    ts = [threading.Thread(target=chain, args=(i,)) for i in range(16)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert not errors, errors


def test_native_client_round_trips_errors_like_reference_client(server, refl):
    from paper_1505_05655_b200.client import submit_native
    for flag, params in [("NOPE", "a=1"), ("LUT_CORRECT", "rows=4"), ("MATMUL", "m=1,k=1,n=1,prec=q")]:
        ours = submit_native("127.0.0.1", server.port, flag, params, [b"\x01\x02"], 0, "n.bin")
        st, p, _, _ = refl.ref_submit(server.port, flag, params, b"\x01\x02", "n.bin")
        assert ours.status == st and ours.params == G.parse_params(p)
    with pytest.raises(G.GpcxError) as e:
        submit_native("127.0.0.1", 1, "NOPE", "", [], 0)
    assert e.value.code == "ConnectFailed"


def test_large_payload_cut_short_drops_connection(server):
    """A >= 8 MiB payload is handed to the task while it arrives; if the
    client stops early the request is dropped (no response), like the
    reference's read_exact failure, and the server keeps serving."""
    with socket.create_connection(("127.0.0.1", server.port), timeout=10) as s:
        s.sendall(W.header("LUT_CORRECT", "rows=2048,cols=4096", has_payload=True))
        s.sendall(b"\0" * (5 << 20))  # 5 of 16 MiB, then half-close
        s.shutdown(socket.SHUT_WR)
        t0 = time.time()
        data = s.recv(4096)
        assert data == b"" and time.time() - t0 < 10
    with socket.create_connection(("127.0.0.1", server.port), timeout=10) as s:
        s.sendall(W.header("NOPE", "", name="after"))
        assert W.parse_response(s.recv(4096))["status"] == "ERR:UNKNOWN_TASK"


@pytest.mark.gpu
def test_large_requests_overlap_receive_and_match(gpu, server):
    """>= 8 MiB payloads take the receive-overlapped path (rt::Arrival):
    LUT_CORRECT 4096^2 (32 MiB) and MATMUL 1536^3 f32 (18 MiB) served
    results equal the oracle."""
    from oracle import oracle as O
    from paper_1505_05655_b200.client import submit_native
    img = O.synth_image(O.IMG_RAMP12, 77, 4096, 4096)
    out = np.empty(img.size, dtype=np.uint16)
    r = submit_native("127.0.0.1", server.port, "LUT_CORRECT", "rows=4096,cols=4096",
                      [img], img.nbytes, "big.raw", out=out.view(np.uint8))
    assert r.ok, r.status
    ref_out, _, _ = O.lut_correct(img, O.LUT_EQUALIZE)
    assert np.array_equal(out, ref_out)
    n = 1536
    A = O.synth_matrix(O.MAT_UNIFORM32, 5, n, n)
    B = O.synth_matrix(O.MAT_UNIFORM32, O.seed_b(5), n, n)
    cm = np.empty(n * n, dtype=np.float32)
    r = submit_native("127.0.0.1", server.port, "MATMUL", f"m={n},k={n},n={n}", [A, B],
                      cm.nbytes, "c.f32", out=cm.view(np.uint8))
    assert r.ok, r.status
    rows = np.arange(0, n, 97).astype(np.uint64)
    Cref, ab = O.matmul_f64(A, B, rows)
    got = cm.reshape(n, n)[rows.astype(np.int64)].astype(np.float64)
    assert np.all(np.abs(got - Cref) <= 1e-5 * ab + 1e-30)


@pytest.mark.gpu
@pytest.mark.slow
def test_c5_chains_match_reference_server(gpu, server, refl):
    """Config C5's chain at its full sizes (LUT_GEN -> LUT_APPLY of a 4096^2
    u16 image, then MATMUL prec=bf16 4096^3 of the corrected image with B),
    4 chains in flight, sent by the reference client to the B200 server and
    to the reference server (acceptance.cpp:446-523: served bytes are the
    same bytes): LUT_GEN / LUT_APPLY responses byte-identical, MATMUL
    params identical and C within 1e-5 * sum|a||b| of the f64 oracle on the
    bf16-rounded operands, for both servers."""
    from oracle import oracle as O
    side = 4096
    dims = f"rows={side},cols={side}"
    B = O.synth_matrix(O.MAT_UNIFORM32, O.seed_b(0x5EED), side, side)
    imgs = [O.synth_image(O.IMG_RAMP12, 0x5EED + i, side, side) for i in range(4)]

    def chain(port, img):
        g = refl.ref_submit(port, "LUT_GEN", dims, img.tobytes(), "lut.bin")
        a = refl.ref_submit(port, "LUT_APPLY", dims, g[2] + img.tobytes(), "img.raw")
        A = np.frombuffer(a[2], dtype=np.uint16).reshape(side, side).astype(np.float32)
        A *= np.float32(1.0 / 65535.0)
        m = refl.ref_submit(port, "MATMUL", f"m={side},k={side},n={side},prec=bf16",
                            A.tobytes() + B.tobytes(), "c.f32")
        return g, a, m, A

    def run_all(port):
        import concurrent.futures as cf
        with cf.ThreadPoolExecutor(max_workers=len(imgs)) as ex:
            return list(ex.map(lambda im: chain(port, im), imgs))

    ours = run_all(server.port)
    with refl.RefServer(max_tasks=4) as rs:
        theirs = run_all(rs.port)
    rows = np.array([0, 1, 2047, 4095], dtype=np.uint64)
    Br = O.round_matrix(O.PREC_BF16, B)
    for img, (g, a, m, A), (g2, a2, m2, _) in zip(imgs, ours, theirs):
        assert g[0] == "OK" and g == g2
        assert a[0] == "OK" and a == a2
        r_out, _, _ = O.lut_correct(img, O.LUT_EQUALIZE)
        assert a[2] == r_out.tobytes()
        assert m[0] == m2[0] == "OK" and m[1] == m2[1] and m[3] == m2[3] == "c.f32"
        Cref, ab = O.matmul_f64(O.round_matrix(O.PREC_BF16, A), Br, rows)
        for resp in (m, m2):
            got = np.frombuffer(resp[2], dtype=np.float32).reshape(side, side)[rows.astype(np.int64)]
            assert np.all(np.abs(got.astype(np.float64) - Cref) <= 1e-5 * ab + 1e-30)


@pytest.mark.gpu
def test_worker_and_device_count_invariance(gpu, refl):
    """acceptance.cpp:278-315 pattern (results independent of the worker
    count), carried to the B200 server: the same requests served with
    max_tasks 1 and 8, and with the planner splitting large requests into 1
    or 2 row bands (G.init([0]) / [0, 0]), return byte-identical responses."""
    from oracle import oracle as O
    rows, cols = 4096, 4096  # 2^24 px / 2^37 flop: the planner's band thresholds
    img = O.synth_image(O.IMG_UNIFORM16, 11, rows, cols)
    m = k = n = 4096
    A = O.synth_matrix(O.MAT_UNIFORM32, 5, m, k)
    B = O.synth_matrix(O.MAT_UNIFORM32, O.seed_b(5), k, n)
    reqs = [("LUT_CORRECT", f"rows={rows},cols={cols}", img.tobytes()),
            ("LUT_GEN", f"rows={rows},cols={cols},mode=stretch", img.tobytes()),
            ("MATMUL", f"m={m},k={k},n={n}", A.tobytes() + B.tobytes()),
            ("MATMUL", f"m={m},k={k},n={n},prec=bf16", A.tobytes() + B.tobytes())]
    seen = {}
    try:
        for devices in ([0], [0, 0]):
            G.init(devices)
            for max_tasks in (1, 8):
                with G.Server(max_tasks=max_tasks) as s:
                    for flag, params, payload in reqs:
                        got = refl.ref_submit(s.port, flag, params, payload, "o.bin")
                        assert got[0] == "OK", got[:2]
                        key = (flag, params)
                        assert seen.setdefault(key, got) == got, (key, devices, max_tasks)
    finally:
        G.init([0])


def _raw_exchange(port: int, request: bytes) -> bytes:
    with socket.create_connection(("127.0.0.1", port), timeout=10) as s:
        s.sendall(request)
        s.shutdown(socket.SHUT_WR)
        chunks = []
        while True:
            b = s.recv(65536)
            if not b:
                break
            chunks.append(b)
    return b"".join(chunks)


def _malformed(i: int, rng) -> bytes:
    """acceptance.cpp:529-627's ten malformed-request classes (plus the
    B200 flags for the classes that apply to them)."""
    flag = ["BAYER_BILINEAR", "LUT_CORRECT", "MATMUL"][i // 10 % 3]
    case = i % 10
    if case == 0:
        return W.header("DEVINFO", "", "out.bin", marker=0x5A)
    if case == 1:
        return W.header("DEVINFO", "", "", marker=W.MARK_DATA)
    if case == 2:
        return W.header(flag, "rows=64,cols=64" if flag != "MATMUL" else "m=4,k=4,n=4", "x.raw",
                        marker=W.MARK_NONE)
    if case == 3:
        return W.header(f"NO_SUCH_TASK_{rng.randrange(1000)}", "", "", marker=W.MARK_NONE)
    if case == 4:
        return W.header(flag, "rows=1048576,cols=1048576" if flag != "MATMUL"
                        else "m=1048576,k=1048576,n=1048576", "", marker=W.MARK_DATA)
    if case == 5:
        h = bytearray(W.header(flag, "", "", marker=W.MARK_NONE))
        h[20] = ord("X")
        return bytes(h)
    if case == 6:
        h = bytearray(W.header("DEVINFO", "a=b", "", marker=W.MARK_NONE))
        h[31] = 0x01
        return bytes(h)
    if case == 7:
        return W.header(flag, "rows=8,rows=9,cols=8", "", marker=W.MARK_DATA)
    if case == 8:
        return W.header(flag, "==,,", "", marker=W.MARK_DATA)
    return W.header(flag, "rows=abc,cols=8" if flag != "MATMUL" else "m=abc,k=2,n=2", "",
                    marker=W.MARK_DATA)


def test_malformed_request_fuzz_over_tcp(server, refl):
    """acceptance.cpp:529-627 over loopback TCP: every malformed request gets
    a well-formed ERR frame -- byte-identical to the reference server's for
    the reference's own flags -- and the server keeps serving."""
    import random
    rng = random.Random(0xBADF00D5)
    with refl.RefServer() as rs:
        for i in range(300):
            req = _malformed(i, rng)
            ours = _raw_exchange(server.port, req)
            r = W.parse_response(ours)
            assert r["status"].startswith("ERR:"), (i, r["status"])
            flag = req[:29].split(b"\0", 1)[0]
            if not flag.startswith((b"LUT_", b"MATMUL")):
                assert ours == _raw_exchange(rs.port, req), (i, r["status"])
    status, _, _, _ = refl.ref_submit(server.port, "NOPE", "", b"", "a")
    assert status == "ERR:UNKNOWN_TASK"


def test_server_phase_stats_count_answered_requests(refl):
    """gpcx_server_stats_get: every answered request (here ERR frames, no
    GPU needed) adds one request and non-negative phase times."""
    with G.Server(max_tasks=2) as s:
        assert s.stats()["requests"] == 0
        for i in range(5):
            status, _, _, _ = refl.ref_submit(s.port, "NOPE", f"i={i}", b"", "a")
            assert status == "ERR:UNKNOWN_TASK"
        st = s.stats()
        assert st["requests"] == 5
        assert all(st[k] >= 0.0 for k in ("recv_ms", "task_ms", "send_ms"))


def test_admission_control_answers_busy_early(monkeypatch, refl):
    """The bounded pipeline: with GPCX_MAX_PENDING=1, a request admitted and
    still receiving its payload holds the only place; the next valid request
    is answered ERR:TASK_FAILED ("server busy") at once, before any payload
    byte (the reference queues it in an unbounded deque, server.hpp:81).
    Once the first one is answered the server admits again."""
    monkeypatch.setenv("GPCX_MAX_PENDING", "1")
    with G.Server(max_tasks=2, idle_timeout_ms=5000) as s:
        hold = socket.create_connection(("127.0.0.1", s.port), timeout=10)
        hold.sendall(W.header("LUT_CORRECT", "rows=64,cols=64", has_payload=True) + b"\0" * 100)
        time.sleep(0.3)  # admitted, receiving
        status, params, _, name = refl.ref_submit(s.port, "LUT_CORRECT", "rows=64,cols=64",
                                                  b"\0" * 8192, "busy.raw")
        assert status == "ERR:TASK_FAILED" and name == "busy.raw"
        assert G.parse_params(params)["msg"].startswith("server busy")
        hold.sendall(b"\0" * (8192 - 100))  # completes: answered (TASK_FAILED without a GPU)
        hold.settimeout(30)
        assert W.parse_response(hold.recv(4096))["status"].startswith(("OK", "ERR:"))
        hold.close()
        status, _, _, _ = refl.ref_submit(s.port, "NOPE", "", b"", "a")
        assert status == "ERR:UNKNOWN_TASK"
        st = s.stats()
        assert st["busy"] == 1


def test_dropped_connections_are_counted(server):
    before = server.stats()["dropped"]
    with socket.create_connection(("127.0.0.1", server.port), timeout=10) as c:
        c.sendall(b"LUT_")
        assert c.recv(16) == b""  # dropped at the 300 ms idle timeout, no response
    time.sleep(0.1)
    assert server.stats()["dropped"] >= before + 1


def test_stop_drains_admitted_requests(refl):
    """Server.stop() first stops accepting, then lets every admitted request
    finish: a request whose payload is still arriving when stop() is called
    is received, run and answered before stop() returns."""
    s = G.Server(max_tasks=2, idle_timeout_ms=5000).start()
    c = socket.create_connection(("127.0.0.1", s.port), timeout=30)
    c.sendall(W.header("LUT_CORRECT", "rows=64,cols=64", has_payload=True) + b"\0" * 1000)
    time.sleep(0.3)  # admitted, receiving
    stopper = threading.Thread(target=s.stop)
    stopper.start()
    time.sleep(0.3)
    assert stopper.is_alive()  # waiting for the in-flight request
    c.sendall(b"\0" * (8192 - 1000))
    resp = W.parse_response(c.recv(4096))
    assert resp["status"].startswith(("OK", "ERR:TASK_FAILED"))  # TASK_FAILED without a GPU
    stopper.join(timeout=30)
    assert not stopper.is_alive()
    c.close()
    with pytest.raises(OSError):  # no longer listening
        socket.create_connection(("127.0.0.1", s.port), timeout=2).close()


def test_synth_request_is_header_only(server):
    """A header-only synthetic request (synth=, no payload, marker 0x00) is
    admitted without reading a payload byte; a payload marker on it is a
    PAYLOAD_MISMATCH, like any task whose rule says 0 bytes."""
    resp = W.parse_response(W.roundtrip(server.port, W.header(
        "LUT_CORRECT", "rows=32768,cols=32768,synth=ramp12", name="d.bin")))
    # OK with a GPU (8-byte digest), TASK_FAILED without one -- never a read
    assert resp["status"] in ("OK", "ERR:TASK_FAILED") and resp["name"] == "d.bin"
    if resp["status"] == "OK":
        assert len(resp["payload"]) == 8
    with socket.create_connection(("127.0.0.1", server.port), timeout=30) as c:
        c.sendall(W.header("LUT_CORRECT", "rows=4,cols=4,synth=ramp12", has_payload=True))
        assert W.parse_response(c.recv(4096))["status"] == "ERR:PAYLOAD_MISMATCH"
