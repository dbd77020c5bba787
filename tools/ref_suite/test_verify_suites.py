"""verify.SUITES (the reference's oracle and property suites, verify.py:293-299)
run unchanged against the drop-in."""
import pytest

import adp.verify as V


@pytest.mark.parametrize("name", sorted(V.SUITES))
def test_suite_passes(name):
    res = V.SUITES[name]()
    print(res.line())
    assert res.passed, res.line()


def test_fd_suite_detects_mutation():
    res = V.fd_suite(mutate="mixed_second_transpose")
    print(res.line())
    assert not res.passed
