#!/bin/bash
# Attribution of the concurrent pass time to tensor-core operand loads
# (outputs invalid under the knobs; token counts show the work is unchanged)
for v in "" "AMUN_DEBUG_LOGIT_FLAGS=2" "AMUN_DEBUG_LOGIT_FLAGS=1" "AMUN_DEBUG_LOGIT_FLAGS=3" "AMUN_DEBUG_SK_FLAGS=2" "AMUN_DEBUG_SK_FLAGS=1" "AMUN_DEBUG_SK_FLAGS=3 AMUN_DEBUG_LOGIT_FLAGS=3" "AMUN_DEBUG_LOGIT_FLAGS=8" "AMUN_DEBUG_LOGIT_FLAGS=4"; do
  echo "== $v"; env $v python tools/decode_probe.py cfg2 2 2>&1 | tail -1
done
