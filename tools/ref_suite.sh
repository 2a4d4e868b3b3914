#!/bin/bash
# the reference's unit tests through the import shim (tests/shim), per file, bounded
cd baseline/_ref_tests || exit 1
for f in test_rope.py test_core.py test_attention.py test_clustering.py test_pipeline.py; do
  echo "=== $f"
  PYTHONPATH=../../tests/shim:../..:$PYTHONPATH timeout 600 python -m pytest -q -p no:cacheprovider $f 2>&1 | grep -E "passed|failed|Error|assert|^FAILED|^E " | head -25
done
