"""pytest plugin (-p ref_suite_plugin): swap the reference's VGICP path for the drop-in before
the reference's own test modules import it.

Used by tests/test_gpu_reference_suite.py, which runs the UNMODIFIED reference test suite
(/root/reference/pkg/tests, copied next to the reference install in baseline/_ref by
tools/install_reference.sh) against ``integrate.patch(limapper)`` on the GPU: the reference's
FactorGraph, LM, IMU factors and odometry stay its own; registration / preprocess /
MatchingCostFactor calls land on libvgicp.  VGICP_REF_SUITE_UNPATCHED=1 runs the suite
against the reference itself (control run)."""

import os


def pytest_configure(config):
    if os.environ.get("VGICP_REF_SUITE_UNPATCHED"):
        return
    from paper_2202_00242_b200 import integrate

    integrate.patch("limapper")
    config._vgicp_patched = True


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    if os.environ.get("VGICP_REF_SUITE_UNPATCHED"):
        terminalreporter.write_line("limapper VGICP path: reference (unpatched)")
        return
    from paper_2202_00242_b200 import _lib

    launches = sum(c.launch_count() for c in _lib._contexts.values())
    terminalreporter.write_line("limapper VGICP path: paper_2202_00242_b200 drop-in "
                                f"(integrate.patch); libvgicp kernel launches: {launches}")
