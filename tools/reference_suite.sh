# The reference's own test suite against the drop-in.
#   stage (build container, where /root/reference exists):  bash tools/reference_suite.sh stage
#       copies the reference's pkg/tests for the hot path into baseline/_ref/tests (git-ignored,
#       never committed; it travels to the GPU box with the snapshot) and writes
#       baseline/_ref/conftest.py, which registers this package under the name `hsewald`
#       (compat.install_as_hsewald) before the reference's conftest imports it.
#   run (GPU box):  bash tools/reference_suite.sh run OUTDIR
# Out of scope and not staged: test_cli.py (the reference CLI).  Acceptance criterion 9
# (complexity timing sweep, ~hours on the reference) is deselected.
set -u
mode=${1:-run}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
DST=$ROOT/baseline/_ref
if [ "$mode" = stage ]; then
  mkdir -p $DST/tests
  for f in conftest.py test_ewald_fourier.py test_ewald_real.py test_acceptance.py test_kernels_direct.py \
           test_system.py test_estimates.py; do
    cp /root/reference/pkg/tests/$f $DST/tests/$f
  done
  cat > $DST/conftest.py <<'PY'
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_1802_07844_b200 import compat  # noqa: E402

compat.install_as_hsewald()
PY
  echo "staged $(ls $DST/tests | wc -l) files into $DST"
  exit 0
fi
out=${2:-gpurun_out/refsuite}
mkdir -p $out
cd $DST && python -m pytest tests -q -p no:cacheprovider -k "not criterion_9" -rs --durations=15 \
    > $ROOT/$out/reference_suite.log 2>&1
echo "rc=$?" >> $ROOT/$out/reference_suite.log
