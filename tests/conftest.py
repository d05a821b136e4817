import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture(scope="session")
def lex_min():
    import oracle
    return oracle.Lexicon.from_file(os.path.join(ROOT, "data", "lexicon_min.txt"))


@pytest.fixture(scope="session")
def lex_v1():
    import oracle
    return oracle.Lexicon.from_file(os.path.join(ROOT, "data", "lexicon_v1.txt"))


@pytest.fixture(scope="session")
def golden():
    import json

    def load(name):
        with open(os.path.join(ROOT, "tests", "golden", name)) as f:
            return json.load(f)
    return load
