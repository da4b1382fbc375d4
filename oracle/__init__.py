"""CPU oracle (TEST INFRASTRUCTURE ONLY): see corrvol_oracle.py.

Importable only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
leg.  oracle/_ref/ (built by oracle/build.sh, git-ignored) holds the real
reference package for validation and for the CPU baseline.
"""

from pathlib import Path

REF_DIR = Path(__file__).resolve().parent / "_ref"


def import_reference():
    """Import the reference corrvol package from oracle/_ref (None if absent)."""
    import sys

    if not (REF_DIR / "corrvol").exists():
        return None
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import corrvol  # noqa: E402

    return corrvol
