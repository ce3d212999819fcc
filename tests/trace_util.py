"""The device RunTrace checked twice: by libperseus (perseus_trace_analyze, the
drop-in restatements in csrc/planner.cpp) and by the UNMODIFIED reference
checkers (oracle/_ref via ref_analyze_records) on the very same records.
Test infrastructure."""
import numpy as np

EV_DTYPE = np.dtype([("t", np.uint64), ("kind", np.int32), ("pe", np.int32), ("peer", np.int32),
                     ("tile", np.int32), ("group", np.int32), ("bytes", np.uint32), ("aux", np.uint32),
                     ("pad", np.uint32)])


def compare_checkers(pb, ref, events, protocol, transfers):
    """Returns libperseus' report; asserts the reference's checkers agree field
    for field in both directions (fence markers, flagged signals, proxy stops,
    NIC stalls, ordering violations, conservation verdict and its first failure)."""
    ours = pb.analyze_trace(events, protocol, transfers)
    for d, key in ((0, "dispatch"), (1, "combine")):
        recs, n, sub, dlv = pb.trace_records(events, protocol, d)
        theirs = ref.analyze_records(recs, n, sub, dlv, transfers, swap=(d == 1))
        mine = ours[key]
        assert theirs["fence_count"] == mine["fence_count"], (key, theirs, mine)
        assert theirs["flagged_signal_count"] == mine["flagged_signal_count"], (key, theirs, mine)
        assert theirs["n_violations"] == mine["ordering_violations"], (key, theirs, mine)
        assert bool(theirs["conservation_pass"]) == mine["conservation_ok"], (key, theirs, mine)
        assert theirs["proxy_stop_episodes"] == 0 and theirs["nic_stall_episodes"] == 0
        if not mine["conservation_ok"] and ours["conservation_error"].startswith(key):
            first = ours["conservation_error"].split(": ", 1)[1]
            assert theirs["failures"] and theirs["failures"][0].startswith(first[:200]), (first, theirs["failures"])
    return ours
