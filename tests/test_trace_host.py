"""Host logic of the schedule trace (no GPU): Lamport clocks / global order built by
spava.trace_events from program-order records, checked with the reference's own
seqpar::validate_trace (oracle/_ref/libseqpar_trace.so), including a violating schedule."""
import ctypes as C
import os

import pytest

from paper_2601_21444_b200 import spava

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TRACE_LIB = os.path.join(ROOT, "oracle", "_ref", "libseqpar_trace.so")

CI, CW, CC, CB, CE = range(5)


def ref_validate(jsonl):
    if not os.path.exists(TRACE_LIB):
        pytest.skip("oracle/_ref/libseqpar_trace.so not built")
    L = C.CDLL(TRACE_LIB)
    L.ref_validate_trace_jsonl.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
    buf = C.create_string_buffer(1 << 16)
    return L.ref_validate_trace_jsonl(jsonl.encode(), buf, len(buf)), buf.value.decode()


def run_host_records(layers, swap_stage2_wait=False):
    """run_host's overlapped program order (simhost.cpp:343-426) for one host."""
    recs = []
    for L in range(layers):
        t = lambda r: f"{r}.L{L}"
        seq = [(CB, "score", ""), (CE, "score", ""), (CI, "pass1", t("pass1")), (CI, "pass2", t("pass2")),
               (CB, "query_attn", ""), (CE, "query_attn", ""), (CI, "qpartial", t("qpartial")),
               (CW, "pass1", t("pass1")), (CC, "pass1", t("pass1")), (CB, "stage1", ""), (CE, "stage1", ""),
               (CW, "pass2", t("pass2")), (CC, "pass2", t("pass2")), (CB, "stage2", ""), (CE, "stage2", ""),
               (CW, "qpartial", t("qpartial")), (CC, "qpartial", t("qpartial")), (CB, "merge", ""),
               (CE, "merge", "")]
        if swap_stage2_wait:  # stage 2 begins before its pass2 wait: must be flagged
            i = seq.index((CB, "stage2", ""))
            seq[i - 2], seq[i] = seq[i], seq[i - 2]
        recs += [(k, lab, L, tag, float(j)) for j, (k, lab, tag) in enumerate(seq)]
    return recs


@pytest.mark.parametrize("hosts,layers", [(1, 1), (4, 3), (8, 2)])
def test_trace_builder_validates(hosts, layers):
    events = spava.trace_events([run_host_records(layers) for _ in range(hosts)])
    assert [e["global_index"] for e in events] == list(range(len(events)))
    # every completion sits after every contributor's issue in the global order
    for e in events:
        if e["kind"] == "comm_completed":
            issues = [x for x in events if x["kind"] == "comm_issued" and x["tag"] == e["tag"]]
            assert len(issues) == hosts and all(x["global_index"] < e["global_index"] for x in issues)
    n, msg = ref_validate(spava.trace_jsonl(events))
    assert n == 0, msg


def test_reference_validator_flags_bad_schedule():
    events = spava.trace_events([run_host_records(1, swap_stage2_wait=True) for _ in range(2)])
    n, msg = ref_validate(spava.trace_jsonl(events))
    assert n > 0 and "pass2 wait started before stage2" in msg
