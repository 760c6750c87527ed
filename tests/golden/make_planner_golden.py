"""Regenerate tests/golden/planner_golden.json.gz from the REFERENCE planner.

Runs every request in tests/planner_cases.py through oracle/_ref/
libtraincap_ref.so (the unmodified reference sources, built by
oracle/Makefile) and stores request/reply pairs, so the parity suite can
check this build's planner on machines without /root/reference (the GPU box).

    make -C oracle ref && python tests/golden/make_planner_golden.py
"""
import ctypes
import gzip
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from paper_1709_06622_b200.planner import Planner  # noqa: E402
import planner_cases  # noqa: E402

FIXTURE_TOKEN = "@FIXTURES@"


def main():
    ref = Planner(ctypes.CDLL(os.path.join(ROOT, "oracle", "_ref", "libtraincap_ref.so")),
                  prefix="tcref_")
    fixture_dir = planner_cases.FIXTURES
    records = []
    for req in planner_cases.build_cases():
        records.append({"request": req, "reply": ref.raw(**req)})
    for req in planner_cases.build_plan_cases(fixture_dir):
        reply = ref.raw(**req)
        text = json.dumps({"request": req, "reply": reply}).replace(fixture_dir, FIXTURE_TOKEN)
        records.append(json.loads(text))
    out = os.path.join(HERE, "planner_golden.json.gz")
    with gzip.open(out, "wt") as f:
        json.dump({"generator": "oracle/_ref/libtraincap_ref.so (reference planner)",
                   "records": records}, f)
    print(f"wrote {len(records)} records to {out}")


if __name__ == "__main__":
    main()
