"""pytest plugin: install the B200 binding into tnkit before the reference's own tests are
collected, and write the routing counters (engine contract_pair calls, GPU permutes, libtnb
kernel launches) to $TNKIT_B200_COUNTERS at the end of the session.

    python -m pytest -p integration.pytest_tnkit_b200 tests/...   (cwd = the staged suite)
"""
import json
import os


def pytest_configure(config):
    import tnkit

    from integration import tnkit_b200
    tnkit_b200.install(tnkit)


def pytest_sessionfinish(session, exitstatus):
    from integration import tnkit_b200
    path = os.environ.get("TNKIT_B200_COUNTERS")
    if path:
        with open(path, "w") as f:
            json.dump(tnkit_b200.counters(), f)
