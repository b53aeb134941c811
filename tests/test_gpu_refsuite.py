"""The reference's own unit suites for the hot path's two classes, run
unmodified through the drop-in: proj/tests/test_photon_map.cpp (PhotonGrid:
brute-force ball parity, closed-ball boundary, visit order, deterministic
rebuilds, the invalid_argument cases) and proj/tests/test_gather.cpp
(sector_index layout, hold/reject semantics, the power-law floor, forced
rejection == fixed schedule bitwise, monotone radius, t counting, F and
chi-squared policies, rgb channels, constructor validation).

They are compiled (oracle/Makefile, in the container that holds the
reference) against include/compat/fppm/{photon_map,gather}.hpp -- PhotonGrid
and GatherRegion re-expressed over the C ABI -- and linked to
libfppm_gpu.so, so every grid build, ball query, accumulate and
end-of-iteration decision in them runs on the B200.  The prebuilt binaries
travel in oracle/_ref; nothing here reads the reference tree."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")


@pytest.mark.parametrize("suite", ["test_photon_map_gpu", "test_gather_gpu"])
def test_reference_suite_through_the_drop_in(suite):
    exe = os.path.join(REF, suite)
    if not os.path.exists(exe):
        pytest.fail(f"{exe} missing: build it with __graft_entry__.build() where /root/reference exists")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(p.stdout)
    print(p.stderr)
    assert p.returncode == 0, p.stderr[-4000:]
    assert "failed: 0 assertions" in p.stdout
