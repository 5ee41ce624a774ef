#!/bin/bash
# Grid sweep at C3 in the bench's default mode (two concurrent parts of 21 groups).
run() {
  echo "== $*"
  env "$@" python tools/profile_step.py --config C3 --steps 2 | tail -1
}
run UQG_NONE=1
run UQG_UPDATE_B=56
run UQG_UPDATE_B=112
run UQG_UPDATE_B=225
run UQG_UPDATE_B=112 UQG_DIR_B=225 UQG_FLUSH_B=225
run UQG_UPDATE_B=112 UQG_DIR_B=56 UQG_FLUSH_B=56
echo C2
run2() {
  echo "== $*"
  env "$@" python tools/profile_step.py --config C2 --steps 2 | tail -1
}
run2 UQG_NONE=1
run2 UQG_UPDATE_B=16
run2 UQG_UPDATE_B=32
run2 UQG_UPDATE_B=64
