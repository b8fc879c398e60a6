for v in base "" base "" base ""; do
  echo "variant=$v $(CITO_LIB_VARIANT=$v KNEE_B=29,29,29,199 python tools/knee.py | tr '\n' ' ')"
done
