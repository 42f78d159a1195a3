"""Trace files (JSON Lines, include/moesim/trace.hpp load/save_token_trace):
byte-identical to the reference writer (verbatim build, oracle/_ref), each
side reads the other's files, the same error texts for malformed or invalid
traces, and the same load matrix.  CPU only."""
import json

import numpy as np
import pytest

from oracle import native as N
from paper_2303_06182_b200.traces import save_synthetic_trace, trace_loads, trace_roundtrip

pytestmark = pytest.mark.skipif(not N.ref_available(), reason="oracle/_ref not built")

SPECS = [(128, 2, 4, 96, 1.2, 0.9, 1.0, 42), (16, 1, 3, 50, 0.0, 0.0, 0.5, 1), (512, 2, 2, 300, 2.0, 0.5, 0.25, 7)]


@pytest.mark.parametrize("spec", SPECS)
def test_saved_bytes_equal_reference(tmp_path, spec):
    ours, ref = tmp_path / "ours.jsonl", tmp_path / "ref.jsonl"
    save_synthetic_trace(ours, *spec)
    N.ref_save_synthetic_trace(ref, *spec)
    assert ours.read_bytes() == ref.read_bytes()
    head = json.loads(ours.read_text().splitlines()[0])
    assert head == {"num_experts": spec[0], "top_k": spec[1], "version": 1}


@pytest.mark.parametrize("spec", SPECS)
def test_cross_read_and_load_matrix(tmp_path, spec):
    E, k, B = spec[0], spec[1], spec[2]
    ref = tmp_path / "ref.jsonl"
    N.ref_save_synthetic_trace(ref, *spec)
    assert trace_roundtrip(ref, tmp_path / "again.jsonl") == (E, k, B)
    assert (tmp_path / "again.jsonl").read_bytes() == ref.read_bytes()
    assert N.ref_trace_roundtrip(tmp_path / "again.jsonl") == (E, k, B)
    ours, theirs = trace_loads(ref, E, B), N.ref_trace_loads(ref, E, B)
    assert np.array_equal(ours, theirs)
    assert np.allclose(ours.sum(0), 1.0)


BAD = {
    "version": '{"num_experts":4,"top_k":1,"version":2}\n',
    "empty": "",
    "parse": '{"num_experts":4,"top_k":1,"version":1}\n{"batch_id":0,"tokens":[\n',
    "range": '{"num_experts":4,"top_k":1,"version":1}\n{"batch_id":0,"tokens":[{"e":[4],"w":[1.0]}]}\n',
    "dup": '{"num_experts":4,"top_k":2,"version":1}\n{"batch_id":0,"tokens":[{"e":[1,1],"w":[0.5,0.5]}]}\n',
    "sum": '{"num_experts":4,"top_k":1,"version":1}\n{"batch_id":0,"tokens":[{"e":[1],"w":[0.9]}]}\n',
    "neg": '{"num_experts":4,"top_k":2,"version":1}\n{"batch_id":0,"tokens":[{"e":[0,1],"w":[-0.5,1.5]}]}\n',
    "order": ('{"num_experts":4,"top_k":1,"version":1}\n{"batch_id":1,"tokens":[{"e":[1],"w":[1.0]}]}\n'
              '{"batch_id":1,"tokens":[{"e":[2],"w":[1.0]}]}\n'),
    "notok": '{"num_experts":4,"top_k":1,"version":1}\n{"batch_id":0,"tokens":[]}\n',
    "k": '{"num_experts":4,"top_k":2,"version":1}\n{"batch_id":0,"tokens":[{"e":[1],"w":[1.0]}]}\n',
    "record": '{"num_experts":4,"top_k":1,"version":1}\n{"tokens":[]}\n',
    "missing": None,
}


@pytest.mark.parametrize("case", sorted(BAD))
def test_errors_match_reference(tmp_path, case):
    path = tmp_path / f"{case}.jsonl"
    if BAD[case] is not None:
        path.write_text(BAD[case])

    def outcome(fn):
        try:
            fn(path)
        except (RuntimeError, N.OracleError) as e:  # OracleError: the reference's non-invalid_argument
            return "runtime_error", str(e)
        except ValueError as e:
            return "invalid_argument", str(e)
        return "ok", ""

    ours, ref = outcome(trace_roundtrip), outcome(N.ref_trace_roundtrip)
    assert ours[0] == ref[0] != "ok"
    if case != "parse":  # parse errors embed the json library's message: compare the prefix
        assert ours[1] == ref[1]
    else:
        assert ours[1].split("parse error")[0] == ref[1].split("parse error")[0]
