python tools/time_encode.py c4 20
