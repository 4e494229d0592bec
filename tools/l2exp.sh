#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.smoke()"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1; echo smoke-launches=$?
