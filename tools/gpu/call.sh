for i in 1 2; do
echo "== r1 tree"; (cd _r1tree && MS=1024,2048 timeout 600 python tools/gemm_micro.py 148)
echo "== now"; MS=1024,2048 timeout 600 python tools/gemm_micro.py 148
done
