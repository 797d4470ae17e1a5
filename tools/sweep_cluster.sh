# attention cluster size sweep (TLS_CLUSTER) for one config: bash tools/sweep_cluster.sh c4 "2 4 8 16"
c=${1:-c3}; for cs in ${2:-1 2 4}; do echo "cs=$cs"; TLS_CLUSTER=$cs timeout 300 python tools/kernel_times.py $c 2>&1 | tail -1; done
