for rep in 1 2; do for lib in abtest/A.so abtest/B.so; do echo "== $lib"; 
TFHE_B200_LIB=$PWD/$lib timeout 300 python tools/prof_hmult.py 4096 set_a 2>&1 | tail -1
TFHE_B200_LIB=$PWD/$lib timeout 300 python tools/prof_hmult.py 32 2>&1 | tail -1
done; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
