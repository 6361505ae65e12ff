from paper_2407_11488_b200.cli import main

main()
