#!/bin/bash
# time the fused fine pass with phases disabled (TMG_FFP4_DBG bits: 2 no A, 4 no B, 8 no C, 16 no D); results are wrong by design
python -m paper_1903_10367_b200.build > gpurun_out/build.log 2>&1 || exit 1
bash tools/ab.sh config5 "TMG_FFP=4 TMG_FFP4_DBG=2" "TMG_FFP=4 TMG_FFP4_DBG=18" "TMG_FFP=4 TMG_FFP4_DBG=26" "TMG_FFP=4 TMG_FFP4_DBG=30" "TMG_FFP=4 TMG_FFP4_DBG=31"
