#!/usr/bin/env bash
# Regenerates tests/golden/*.json from the unmodified reference (this
# container only: needs /root/reference).  TEST INFRASTRUCTURE.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
make -s -C "$HERE" ref
"$HERE/_ref/ref_dump" "$HERE/../tests/golden"
