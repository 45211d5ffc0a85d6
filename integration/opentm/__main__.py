import sys

from paper_2405_19991_b200.cli import main

sys.exit(main())
