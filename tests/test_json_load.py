"""The graph / device JSON loaders (json_load.cu: host code in libdagplace_b200.so, no GPU
needed) against the reference's graph_from_json / devices_from_json (json_io.cpp, compiled
with nlohmann/json 3.11.3 into oracle/_ref): identical SoA arrays on valid documents,
identical error kind + message on schema errors, the same kind (ParseError) on syntax
errors (whose wording is nlohmann's own)."""
import json
import os

import numpy as np
import pytest

from paper_2208_00184_b200 import HERE as PKG
from paper_2208_00184_b200._abi import DagError, devices_from_json, graph_from_json

LIB = os.path.join(PKG, "libdagplace_b200.so")


@pytest.fixture(scope="module")
def libs():
    import ctypes as C
    from oracle.bind import reference_available
    if not os.path.exists(LIB):
        pytest.skip("libdagplace_b200.so not built")
    if not reference_available():
        pytest.skip("oracle/_ref not built")
    from oracle.bind import reference_backend
    return C.CDLL(LIB), reference_backend().lib


def _outcome(fn, lib, text, prefix):
    try:
        return "ok", fn(lib, text, prefix)
    except DagError as e:
        return "err", (e.kind, str(e))


def _same(a, b, text, syntax_kind_only=False):
    assert a[0] == b[0], (text[:200], a, b)
    if a[0] == "err":
        assert a[1][0] == b[1][0], (text[:200], a[1], b[1])
        if not syntax_kind_only and "invalid JSON" not in b[1][1]:
            assert a[1][1] == b[1][1], (text[:200], a[1], b[1])
        return
    x, y = a[1], b[1]
    if isinstance(x, tuple):  # devices
        assert x == y
        return
    for f in ("node_id", "compute_us", "memory_bytes", "edge_src", "edge_dst", "edge_bytes", "group"):
        assert np.array_equal(getattr(x, f), getattr(y, f)), (f, text[:200])


def _graph_doc(rng, n, groups=False, extras=False):
    nodes = []
    for i in range(n):
        nd = {"id": int(rng.integers(-5, 10 ** 9)) if i % 7 == 3 else i, "name": f"opé{i}\\\"q\"",
              "compute_us": int(rng.integers(0, 1000)), "memory_bytes": int(rng.integers(0, 1 << 40))}
        if groups and i % 3 == 0:
            nd["colocation_group"] = f"g{int(rng.integers(0, 4))}☃"
        elif groups and i % 3 == 1:
            nd["colocation_group"] = None
        if extras:
            nd["extra"] = {"a": [1, 2.5, {"b": None}], "t": True}
        nodes.append(nd)
    edges = [{"src": i - 1, "dst": i, "tensor_bytes": int(rng.integers(0, 1 << 20))} for i in range(1, n)]
    doc = {"schema_version": 1, "nodes": nodes, "edges": edges}
    if extras:
        doc["meta"] = {"x": "y"}
    return doc


VALID = [
    '{"nodes":[],"edges":[]}',
    '{"nodes":[{"id":1,"compute_us":2,"memory_bytes":3}],"edges":[]}',
    # floats truncate, exponents, negative zero, big unsigned wraps, duplicate keys (last wins)
    '{"nodes":[{"id":1.9,"compute_us":2e2,"memory_bytes":-0.0},{"id":18446744073709551615,'
    '"compute_us":5,"memory_bytes":7,"id":3}],"edges":[{"src":1,"dst":3,"tensor_bytes":1.5E1}]}',
    ' \n\t{"edges":[{"tensor_bytes":4,"dst":2,"src":1}],"nodes":[{"memory_bytes":1,"compute_us":1,"id":1},'
    '{"id":2,"compute_us":1,"memory_bytes":1,"colocation_group":"a\\u00e9\\ud83d\\ude00"},'
    '{"id":3,"compute_us":1,"memory_bytes":1,"colocation_group":"aé\U0001F600"}]} ',
    '{"schema_version":1,"nodes":[{"id":-9223372036854775808,"compute_us":1,"memory_bytes":1}],"edges":[]}',
    '{"nodes":[{"id":9223372036854775808,"compute_us":1,"memory_bytes":1}],"edges":[]}',
]

SCHEMA_ERRORS = [
    '[]', '3', '"x"', 'null',
    '{"schema_version":2,"nodes":[],"edges":[]}',
    '{"schema_version":1.0,"nodes":[],"edges":[]}',
    '{"schema_version":"1","nodes":[],"edges":[]}',
    '{"edges":[]}', '{"nodes":{},"edges":[]}', '{"nodes":[]}', '{"nodes":[],"edges":3}',
    '{"nodes":[{"compute_us":1,"memory_bytes":1}],"edges":[]}',
    '{"nodes":[{"id":"1","compute_us":1,"memory_bytes":1}],"edges":[]}',
    '{"nodes":[{"id":1,"memory_bytes":1}],"edges":[]}',
    '{"nodes":[{"id":1,"compute_us":true,"memory_bytes":1}],"edges":[]}',
    '{"nodes":[{"id":1,"compute_us":1}],"edges":[]}',
    '{"nodes":[{"id":1,"compute_us":1,"memory_bytes":null}],"edges":[]}',
    '{"nodes":[{"id":1,"compute_us":1,"memory_bytes":1,"colocation_group":5}],"edges":[]}',
    '{"nodes":[5],"edges":[]}',
    '{"nodes":[],"edges":[{"src":1,"dst":2}]}',
    '{"nodes":[],"edges":[{"src":1,"tensor_bytes":2}]}',
    '{"nodes":[],"edges":[[1,2,3]]}',
    '{"nodes":[{"id":1}],"edges":[{"bad":1}]}',  # node error reported first
]

SYNTAX_ERRORS = [
    '', ' ', '{', '{"nodes":[]', '{"nodes":[],}', '{"nodes":[1,]}', '{nodes:[]}', "{'nodes':[]}",
    '{"nodes":[01]}', '{"nodes":[1.]}', '{"nodes":[.5]}', '{"nodes":[-]}', '{"nodes":[1e]}',
    '{"nodes":[tru]}', '{"nodes":[nul]}', '{"a":"\\x"}', '{"a":"\\ud800"}', '{"a":"\\udc00"}',
    '{"a":"\x01"}', '{"a":"\xff"}', '{"nodes":[],"edges":[]} x', '{"a" 1}', '[1 2]',
    '{"nodes":[],"edges":[]}{}', '{"a":"\\u12"}',
    b'{"a":"\xff"}', b'{"a":"\xc0\xaf"}', b'{"a":"\xed\xa0\x80"}', b'{"a":"\xe2\x82"}',
]


def test_valid_documents(libs):
    dp, ref = libs
    for t in VALID:
        _same(_outcome(graph_from_json, dp, t, "dp_"), _outcome(graph_from_json, ref, t, "dpr_"), t)


def test_generated_documents(libs):
    dp, ref = libs
    rng = np.random.default_rng(5)
    for n, groups, extras in [(1, False, False), (30, True, False), (200, True, True), (5000, False, True)]:
        t = json.dumps(_graph_doc(rng, n, groups, extras), ensure_ascii=bool(n % 2))
        a = _outcome(graph_from_json, dp, t, "dp_")
        assert a[0] == "ok"
        _same(a, _outcome(graph_from_json, ref, t, "dpr_"), t)


@pytest.mark.parametrize("i", range(len(SCHEMA_ERRORS)))
def test_schema_errors(libs, i):
    dp, ref = libs
    t = SCHEMA_ERRORS[i]
    a, b = _outcome(graph_from_json, dp, t, "dp_"), _outcome(graph_from_json, ref, t, "dpr_")
    assert b[0] == "err"
    _same(a, b, t)


@pytest.mark.parametrize("i", range(len(SYNTAX_ERRORS)))
def test_syntax_errors(libs, i):
    dp, ref = libs
    t = SYNTAX_ERRORS[i]
    a, b = _outcome(graph_from_json, dp, t, "dp_"), _outcome(graph_from_json, ref, t, "dpr_")
    assert b[0] == "err" and b[1][0] == "ParseError", b
    _same(a, b, t, syntax_kind_only=True)


def test_devices(libs):
    dp, ref = libs
    docs = [
        '{"devices":[{"id":3,"memory_bytes":100},{"id":1,"memory_bytes":5e3}],"comm":{"k_us_per_byte":0.001,"b_us":10}}',
        '{"schema_version":1,"devices":[{"id":1,"memory_bytes":1}],"comm":{"k_us_per_byte":0,"b_us":0}}',
        '{"devices":[],"comm":{"k_us_per_byte":1,"b_us":1}}',
        '{"devices":[{"id":1,"memory_bytes":0}],"comm":{"k_us_per_byte":1,"b_us":1}}',
        '{"devices":[{"id":1,"memory_bytes":1}]}',
        '{"devices":[{"id":1,"memory_bytes":1}],"comm":{"k_us_per_byte":-1,"b_us":1}}',
        '{"devices":[{"id":1,"memory_bytes":1}],"comm":{"b_us":1}}',
        '{"devices":[{"memory_bytes":1}],"comm":{"k_us_per_byte":1,"b_us":1}}',
        '{"devices":{},"comm":{}}', '[]', '{"devices":[1],"comm":{}}', '{"devices":[{"id":1,',
    ]
    for t in docs:
        _same(_outcome(devices_from_json, dp, t, "dp_"), _outcome(devices_from_json, ref, t, "dpr_"), t)


def test_deep_nesting(libs):
    """json::parse has no nesting limit; neither does the loader (iterative validation)."""
    dp, ref = libs
    for depth in (600, 5000):
        deep = "[" * depth + "]" * depth
        obj = '{"a":' * depth + "1" + "}" * depth
        for t in ('{"nodes":[],"edges":[],"meta":%s,"x":%s}' % (deep, obj),
                  '{"nodes":[{"id":1,"compute_us":2,"memory_bytes":3,"extra":%s}],"edges":[]}' % deep):
            a = _outcome(graph_from_json, dp, t, "dp_")
            assert a[0] == "ok", a
            _same(a, _outcome(graph_from_json, ref, t, "dpr_"), t)
        bad = '{"nodes":[],"edges":[],"meta":' + "[" * depth + "]" * (depth - 1) + "}"
        a, b = _outcome(graph_from_json, dp, bad, "dp_"), _outcome(graph_from_json, ref, bad, "dpr_")
        assert b[0] == "err"
        _same(a, b, bad, syntax_kind_only=True)
