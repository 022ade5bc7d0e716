"""Install the B200 LU backend into a COPY of an installed reference package.

    python integration/install_backend.py <dir containing rlra/>

Copies integration/_lu_b200.py to <dir>/rlra/_lu_b200.py and adds one branch to
<dir>/rlra/backend.py (rlra/backend.py:12-30):

    elif _choice == "b200":
        from . import _lu_b200 as _impl
        BACKEND = "b200"

The reference source tree itself is never modified; tests install into a
temporary copy of oracle/_ref (tests/test_reference_suite_gpu.py).
"""

import os
import shutil
import sys

BRANCH = '''elif _choice == "b200":
    from . import _lu_b200 as _impl

    BACKEND = "b200"
'''


def install(root):
    pkg = os.path.join(root, "rlra")
    shutil.copy(os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lu_b200.py"),
                os.path.join(pkg, "_lu_b200.py"))
    path = os.path.join(pkg, "backend.py")
    src = open(path).read()
    if '_choice == "b200"' in src:
        return path
    anchor = 'elif _choice == "python":'
    if anchor not in src:
        raise RuntimeError(f"unexpected reference backend.py: no {anchor!r} branch")
    src = src.replace(anchor, BRANCH + anchor, 1)
    src = src.replace("RLRA_BACKEND must be auto, compiled, or python", "RLRA_BACKEND must be auto, compiled, python, or b200")
    with open(path, "w") as fh:
        fh.write(src)
    return path


if __name__ == "__main__":
    print(install(sys.argv[1]))
