for c in bicycle mcmc; do timeout 600 python tools/time_raster_ab.py $c 0 2>&1 | grep -E "records"; done
