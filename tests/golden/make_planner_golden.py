"""Regenerate tests/golden/planner_golden.json.gz from the REFERENCE planner.

Runs every request in tests/planner_cases.py through oracle/_ref/
libtraincap_ref.so (the unmodified reference sources, built by
oracle/Makefile) and stores request/reply pairs, so the parity suite can
check this build's planner on machines without /root/reference (the GPU box).
B200-catalog cases run in a child process with a time limit: the reference's
branch-and-bound is exponential under binding bounds, and a case
it cannot finish is recorded as such instead of stalling the generator.

    make -C oracle ref && python tests/golden/make_planner_golden.py
"""
import ctypes
import gzip
import json
import multiprocessing as mp
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from paper_1709_06622_b200.planner import Planner  # noqa: E402
import planner_cases  # noqa: E402

FIXTURE_TOKEN = "@FIXTURES@"
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libtraincap_ref.so")
TIME_LIMIT_S = 60


def _ref():
    return Planner(ctypes.CDLL(REF_LIB), prefix="tcref_")


def _child(req, q):
    q.put(_ref().raw(**req))


def ref_with_limit(req):
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    p = ctx.Process(target=_child, args=(req, q))
    p.start()
    p.join(TIME_LIMIT_S)
    if p.is_alive():
        p.kill()
        p.join()
        return None
    return q.get()


def main():
    ref = _ref()
    fixture_dir = planner_cases.FIXTURES
    records = []
    for req in planner_cases.build_cases():
        records.append({"request": req, "reply": ref.raw(**req)})
    for req in planner_cases.build_plan_cases(fixture_dir):
        reply = ref.raw(**req)
        text = json.dumps({"request": req, "reply": reply}).replace(fixture_dir, FIXTURE_TOKEN)
        records.append(json.loads(text))
    b200, slow = [], 0
    for req in planner_cases.build_b200_cases():
        reply = ref_with_limit(req)
        if reply is None:
            slow += 1
            b200.append({"request": req, "reply": None, "reference": f"did not finish in {TIME_LIMIT_S} s"})
        else:
            b200.append({"request": req, "reply": reply})
    out = os.path.join(HERE, "planner_golden.json.gz")
    with gzip.open(out, "wt") as f:
        json.dump({"generator": "oracle/_ref/libtraincap_ref.so (reference planner)",
                   "records": records, "b200_records": b200}, f)
    print(f"wrote {len(records)} + {len(b200)} B200 records ({slow} beyond the reference's time limit)")


if __name__ == "__main__":
    main()
