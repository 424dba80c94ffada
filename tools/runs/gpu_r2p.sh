#!/bin/bash
# Round-2 evidence pass: smoke, the -m gpu suite, the bench line + reference arm, and the
# profile set (launch list + full captures) via tools/profile_round.sh.
OUT=gpurun_out/r2p
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo rc=$? >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
bash tools/profile_round.sh r2p
