for pb in 24 8 64; do echo "pipeline_bytes=$pb MB"; timeout 300 python scratch/e2e_diag.py $pb; done
