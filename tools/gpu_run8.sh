timeout 600 python tools/nsplit_sweep.py c3 1,2,4,8 2>&1 | grep nsplit=
TLS_CLUSTER=1 timeout 600 python tools/nsplit_sweep.py c3 1,2,4 2>&1 | grep nsplit=
TLS_NOPRIO=1 timeout 600 python tools/nsplit_sweep.py c3 2,4 2>&1 | grep nsplit=
