for i in 1 2; do python tools/variants.py run rmat24 3 ur2 ur1 ur0; done
python tools/variants.py run rmat22 3 ur2 ur1 ur0
