"""Loader for tests/golden/replay_cases.json (reference-generated fixtures)."""
import json
import os

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "replay_cases.json")


def load():
    with open(PATH) as f:
        return json.load(f)["cases"]


def ids():
    return [c["case"]["name"] for c in load()]
