"""Run the alpha=9 -> 54 base conversion with a TFHE_BC_TRACE build (TFHE_B200_LIB)."""
import sys
sys.argv = [sys.argv[0], sys.argv[1] if len(sys.argv) > 1 else "32"]
exec(open("tools/prof_bconv.py").read())
