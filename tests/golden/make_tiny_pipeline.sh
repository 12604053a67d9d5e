#!/usr/bin/env bash
# Regenerate tests/golden/tiny_pipeline/ with the REFERENCE's own default
# pipeline (src/specexit/pipeline.py:28-50, run_all :250-255), built from a
# writable copy of /root/reference/pkg (its Cython kernel needs an in-place
# build).  ~6 min on 8 cores.  The resulting trace.jsonl / report.json /
# similarity.json are byte-identical to the reference's shipped
# pkg/runs/default/ files (checked below); the weight/predictor/profile
# artifacts are the inputs our end-to-end parity tests replay.
set -euo pipefail
OUT="$(cd "$(dirname "$0")" && pwd)/tiny_pipeline"
rm -rf /tmp/refcopy && cp -r /root/reference/pkg /tmp/refcopy && chmod -R u+w /tmp/refcopy
cd /tmp/refcopy && python setup.py build_ext --inplace >/dev/null
rm -rf /tmp/refrun
python -c "
import sys; sys.path.insert(0, 'src')
from specexit.pipeline import Pipeline, load_config
Pipeline(load_config(out_dir='/tmp/refrun')).run_all()"
for f in trace.jsonl report.json similarity.json; do
  cmp /tmp/refrun/$f /root/reference/pkg/runs/default/$f
done
cp /tmp/refrun/{target.spxw,draft.spxw,predictors.spxp,profile.spxs,trace.jsonl,report.json,similarity.json} "$OUT/"
cp /root/reference/pkg/data/fixture_corpus.txt "$OUT/"
echo "tiny pipeline fixtures refreshed in $OUT"
