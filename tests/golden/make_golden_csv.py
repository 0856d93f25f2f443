"""Golden CSV of the reference's harness writer (harness.py:447-466) for a
fixed list of RunRecords, produced by the REFERENCE itself.

    python tests/golden/make_golden_csv.py  ->  tests/golden/ref_log.csv
"""

import os
import sys

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def records(RunRecord):
    return [
        RunRecord(1, 0.000123456789, 0, 0, 0.5, 12.25, False),
        RunRecord(2, 1.5e-3, 1, 100, 0.123456789012345678, 1.0 / 3.0, True),
        RunRecord(3, 2.0, 1, 100, None, None, False),
        RunRecord(4, 2.5e-7, 2, 200, 1e-300, float("inf"), True),
        RunRecord(5, 3.0, 2, 200, 7.0, -0.0, False),
    ]


def main():
    sys.path.insert(0, REF_SRC)
    from imgskip.harness import emit_csv
    from imgskip.solvers import RunRecord
    path = os.path.join(HERE, "ref_log.csv")
    emit_csv(records(RunRecord), path)
    print(f"wrote {path}")


if __name__ == "__main__":
    main()
