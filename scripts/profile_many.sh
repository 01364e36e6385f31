#!/bin/bash
# several full ncu captures in one GPU session: profile_many.sh "NAME WORKLOAD REGEX" ...
cd "$(dirname "$0")/.." || exit 1
for spec in "$@"; do
  set -- $spec
  bash scripts/profile_one.sh $1 $2 "$3" > /dev/null 2>&1
  echo "$1 done"
done
