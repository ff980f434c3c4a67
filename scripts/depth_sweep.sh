for d in ${DEPTHS:-9 10 11 12}; do timeout 300 python scripts/model_time.py resnet20 $d 128 3 | tail -1 | cut -c1-60; done
