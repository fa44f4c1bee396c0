for f in -1 0 1 2 3 4 5; do echo "== force $f"; NF_GEMM_FORCE=$f ONLY=70r MS=512,1024,2048 timeout 600 python tools/gemm_micro.py 148 132 2>&1 | grep -E "kqv|ocol|70r.o "; done
