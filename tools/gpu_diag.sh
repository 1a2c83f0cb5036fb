timeout 60 ./tools/ubench/ex2_rate
