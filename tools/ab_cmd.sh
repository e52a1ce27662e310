LIBS="ab/lib_old.so ab/lib_new.so" bash tools/ab_sample.sh
